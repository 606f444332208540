#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_warp -o gpurun_out/r02i_c5 -f \
   python tools/prof_one.py --config C5 --ebn0 2.5 --frames 30000 --warm 0 > gpurun_out/r02i_ncu.log 2>&1
tail -3 gpurun_out/r02i_ncu.log
