#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
O=gpurun_out/r02ad_t.log
for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000" "C3b 4.0 100000" "C3a 2.0 100000" "C1 2.0 400000"; do
  set -- $c; echo "== $1" >> $O
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "threads|best|rror" >> $O
done
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 1200 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02ad_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02ad_gpu.log
grep -E "==|best" $O; tail -3 gpurun_out/r02ad_gpu.log
