#!/bin/bash
# plain run, then ncu --set full on the measured launch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CMD="python tools/prof_one.py --warm 0 $*"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:cbp_kernel -s 1 -c 1 -o gpurun_out/prof -f $CMD > gpurun_out/prof_ncu.log 2>&1
echo "rc=$?"; cat gpurun_out/prof_plain.log; tail -5 gpurun_out/prof_ncu.log
