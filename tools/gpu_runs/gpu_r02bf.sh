#!/bin/bash
# A/B: phi-row pipe balance (C2B rows of some edges from shared memory / B2V rows of some edges through TEX)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ab() { for lib in "$@"; do for c in "C5 2.5" "C2 2.0" "P2048 2.5"; do set -- $c
  echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done; }
{
ab libcbp.so libcbp_mt512.so libcbp_c2b01b2v40.so libcbp_c2b01.so libcbp_b2v40.so libcbp.so libcbp_mt512.so libcbp_c2b01b2v40.so
} > gpurun_out/r02bf_ab.log 2>&1
cat gpurun_out/r02bf_ab.log
