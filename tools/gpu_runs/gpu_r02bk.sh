#!/bin/bash
# A/B: compact channel code (libcbp.so) vs round-2 state before the footprint work (libcbp_nomerge.so);
# merged max-dc body for K = 1 codes too (libcbp_mk1.so)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ab() { for lib in "$@"; do for c in "C5 2.5" "C2 2.0" "C2 3.0" "P2048 2.5" "C1 2.0"; do set -- $c
  echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done; }
{
ab libcbp_nomerge.so libcbp.so libcbp_mk1.so libcbp.so libcbp_mk1.so
timeout 300 python tools/split_ber.py --config C5 --ebn0 2.5 --frames 200000 | head -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "ber_sim or channel or stop" 2>&1 | tail -2
} > gpurun_out/r02bk_ab.log 2>&1
cat gpurun_out/r02bk_ab.log
