#!/bin/bash
# ncu --set full of the C5 ber_sim launch (current kernel)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
P="python tools/prof_one.py --config C5 --ebn0 2.5 --frames 50000 --warm 0"
timeout 300 $P > gpurun_out/r02bl_plain.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cbp_warp -s 1 -c 1 -o gpurun_out/r02bl_c5 -f $P > gpurun_out/r02bl_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r02bl_plain.log
