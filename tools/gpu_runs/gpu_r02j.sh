#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in "C5 2.5 100000" "C2 2.0 200000" "C3b 4.0 100000" "P2048 2.0 100000"; do
  set -- $c; echo "== $1" >> gpurun_out/r02j_t.log
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|threads|Error|error" >> gpurun_out/r02j_t.log
done
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_warp -o gpurun_out/r02j_c5 -f \
   python tools/prof_one.py --config C5 --ebn0 2.5 --frames 30000 --warm 0 > gpurun_out/r02j_ncu.log 2>&1
cat gpurun_out/r02j_t.log
