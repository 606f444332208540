#!/bin/bash
# A/B: phi rows of the parked (long-row) path through TEX for some chunk edges (C3b; libcbp_pk1/2/3.so) and a second
# B2V row through TEX in the register rows (libcbp_m1.so, CBP_B2V_TEX_MASK=0x60); parity subset under the best candidates
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() { CBP_LIB=$PWD/paper_2305_05286_b200/$1 timeout 200 python tools/prof_one.py --config $2 --ebn0 $3 --reps 5 --frames 100000 2>&1 | grep best; }
{ for rep in 1 2; do
    for lib in libcbp.so libcbp_pk1.so libcbp_pk2.so libcbp_pk3.so; do echo "== $lib C3b 4.0 $(run $lib C3b 4.0)"; done
    for lib in libcbp.so libcbp_m1.so; do for c in "C5 2.5" "C3a 1.5"; do set -- $c; echo "== $lib $1 $2 $(run $lib $1 $2)"; done; done
  done
  for lib in libcbp_pk1.so libcbp_pk3.so; do
    CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "C3b or layouts or extreme" 2>&1 | tail -2; done
} > gpurun_out/r02ca_ab.log 2>&1
cat gpurun_out/r02ca_ab.log
