#!/bin/bash
# parity suite + ncu of the producer-side kernel (C5 and C2)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r02c_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02c_parity.log
timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --reps 3 > gpurun_out/r02c_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_kernel -o gpurun_out/r02c_c5 -f \
   python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --warm 0 > gpurun_out/r02c_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_kernel -o gpurun_out/r02c_c2 -f \
   python tools/prof_one.py --config C2 --ebn0 2.0 --frames 100000 --warm 0 > gpurun_out/r02c_ncu2.log 2>&1
tail -5 gpurun_out/r02c_parity.log; tail -3 gpurun_out/r02c_plain.log
