#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in "CBP_WARP_TEX=2" "CBP_WARP_TEX=1" "X=1"; do
for c in "C5 2.5 100000" "C2 2.0 200000"; do
  set -- $c; echo "== $v $1" >> gpurun_out/r02q_t.log
  env $v timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|Error|error" >> gpurun_out/r02q_t.log
done; done
grep -E "==|best" gpurun_out/r02q_t.log
