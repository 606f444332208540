#!/bin/bash
# default bench -> gpurun_out/bench.json; then ncu launch list of a short bench and one full capture
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
cat gpurun_out/bench.json | head -c 2500; echo; tail -3 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
  B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --frames 200000"
  timeout 600 $B > gpurun_out/bench_short.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
  P="python tools/prof_one.py --config C2 --ebn0 2.0 --frames 100000 --warm 0"
  timeout 300 $P > gpurun_out/prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cbp_kernel -s 1 -c 1 -o gpurun_out/prof -f $P > gpurun_out/prof_ncu.log 2>&1; echo "full capture rc=$?"
fi
