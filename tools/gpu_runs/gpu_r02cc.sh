#!/bin/bash
# A/B on the parked rows: chunks of 6 edges (libcbp_u6.so) and one B2V row of a chunk through TEX as well (libcbp_b1.so)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() { CBP_LIB=$PWD/paper_2305_05286_b200/$1 timeout 300 python tools/prof_one.py --config $2 --ebn0 $3 --reps 5 --frames $4 2>&1 | grep best; }
{ for rep in 1 2; do for lib in libcbp.so libcbp_u6.so libcbp_b1.so; do
    echo "== $lib C3b 4.0 $(run $lib C3b 4.0 100000)"; echo "== $lib C3b 3.0 $(run $lib C3b 3.0 100000)"; echo "== $lib C4 1.5 $(run $lib C4 1.5 3000)"; done; done
  for lib in libcbp_u6.so; do
    CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "C3b or layouts or extreme or C4" 2>&1 | tail -2; done
} > gpurun_out/r02cc_ab.log 2>&1
cat gpurun_out/r02cc_ab.log
