#!/bin/bash
# round 2, first call: default bench on the C5 headline (baseline of the round-1 kernel) + ncu of the C5 launch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo "bench rc=$?" >> gpurun_out/r02a_bench.err
timeout 600 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --reps 3 > gpurun_out/r02a_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_kernel -o gpurun_out/r02a_c5 -f \
   python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --warm 0 > gpurun_out/r02a_ncu.log 2>&1
tail -c 2500 gpurun_out/r02a_bench.json; tail -3 gpurun_out/r02a_bench.err; tail -3 gpurun_out/r02a_plain.log
