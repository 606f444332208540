#!/bin/bash
# A/B: after the per-frame code compaction, one max-dc body (libcbp.so) vs one body per dc (libcbp_nomerge.so)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ab() { for lib in "$@"; do for c in "C5 2.5" "C3a 1.5"; do set -- $c
  echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done; }
{ ab libcbp.so libcbp_nomerge.so libcbp.so libcbp_nomerge.so
  for lib in libcbp.so libcbp_nomerge.so; do CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 300 python tools/split_ber.py --config C5 --ebn0 2.5 --frames 200000 | head -1; done
} > gpurun_out/r02bq_ab.log 2>&1
cat gpurun_out/r02bq_ab.log
