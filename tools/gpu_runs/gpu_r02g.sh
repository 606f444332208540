#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_kernel -o gpurun_out/r02g_c2 -f \
   python tools/prof_one.py --config C2 --ebn0 2.0 --frames 50000 --warm 0 > gpurun_out/r02g_ncu2.log 2>&1
CBP_SPLIT_R=0 timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_kernel -o gpurun_out/r02g_c5s -f \
   python tools/prof_one.py --config C5 --ebn0 2.5 --frames 30000 --warm 0 > gpurun_out/r02g_ncu5.log 2>&1
ls -la gpurun_out
