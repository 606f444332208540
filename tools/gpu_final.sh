#!/bin/bash
# round measurement: default bench -> gpurun_out/bench.json; ncu launch list of a short
# bench; one ncu --set full capture of the C2 2 dB ber_sim launch (tools/profile_summary.py)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
head -c 1500 gpurun_out/bench.json; echo; tail -2 gpurun_out/bench.err
B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-suite --frames 200000"
timeout 600 $B > gpurun_out/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
P="python tools/prof_one.py --config C2 --ebn0 2.0 --frames 100000 --warm 0"
timeout 300 $P > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cbp_kernel -s 1 -c 1 -o gpurun_out/prof_final -f $P > gpurun_out/prof_ncu.log 2>&1; echo "full capture rc=$?"
