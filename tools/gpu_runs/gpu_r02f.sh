#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in "X=1" "CBP_MULTI_MAXT=512" "CBP_SPLIT_R=0" "CBP_SPLIT_R=0 CBP_MULTI_MAXT=1024" "CBP_MULTI_MAXT=1024"; do
  echo "== $v" >> gpurun_out/r02f_ab.log
  env $v timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --reps 3 2>&1 | grep -E "best|threads" >> gpurun_out/r02f_ab.log
done
cat gpurun_out/r02f_ab.log
