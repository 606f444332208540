#!/bin/bash
# A/B: warps per SM on C5 (L1 left for the TEX phi rows vs frames in flight)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for w in 0 10 9 8 7; do
  echo "== warps $w" >> gpurun_out/r02z_t.log
  CBP_WARPS=$w timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --reps 3 2>&1 | grep -E "threads|best|rror" >> gpurun_out/r02z_t.log
done
for t in 1 2; do
  for w in 0 9; do
  echo "== tex $t warps $w" >> gpurun_out/r02z_t.log
  CBP_WARP_TEX=$t CBP_WARPS=$w timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --reps 3 2>&1 | grep -E "threads|best|rror" >> gpurun_out/r02z_t.log
  done
done
cat gpurun_out/r02z_t.log
