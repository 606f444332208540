#!/bin/bash
# A/B: max-dc body shared by dc-1 rows (libcbp.so) vs one body per dc (libcbp_nomerge.so); parity subset on the new lib
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ab() { for lib in "$@"; do for c in "C5 2.5" "C2 2.0" "C3b 4.0" "P2048 2.5"; do set -- $c
  echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done; }
{
ab libcbp_nomerge.so libcbp.so libcbp_nomerge.so libcbp.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not all_frames" 2>&1 | tail -3
} > gpurun_out/r02bd_ab.log 2>&1
cat gpurun_out/r02bd_ab.log
