#!/bin/bash
# A/B: warps per SM (L1 left for the TEX phi rows) and phi-row paths on C5, env knobs only
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() { echo "== $*"; env "$@" timeout 200 python tools/prof_one.py --config C5 --ebn0 2.5 --reps 5 --frames 100000 2>&1 | grep -E "best|launch|threads" | tail -2; }
{
run CBP_NONE=1
for w in 19 18 17 16; do run CBP_WARPS=$w; done
for t in 1 2; do run CBP_WARP_TEX=$t; run CBP_WARP_TEX=$t CBP_WARPS=19; run CBP_WARP_TEX=$t CBP_WARPS=18; done
} > gpurun_out/r02bb_ab.log 2>&1
cat gpurun_out/r02bb_ab.log
