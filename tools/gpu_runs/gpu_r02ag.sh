#!/bin/bash
# team frames (one frame per CTA) for C4 / P8192: parity + A/B timing vs cbp_kernel teams
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
O=gpurun_out/r02ag_t.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 600 -p no:cacheprovider -k "team_frames or c4" > gpurun_out/r02ag_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02ag_parity.log
tail -30 gpurun_out/r02ag_parity.log
for env in "" "CBP_WARP_TEAM=0"; do
  for c in "C4 1.5 3000 2" "P8192 2.0 10000 0"; do
    set -- $c; echo "== $1 $env" >> $O
    env $env timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --rule $4 --reps 3 2>&1 | grep -E "threads|best|rror|frames'" | tail -3 >> $O
  done
done
cat $O
