#!/bin/bash
# B2V lookups of a row issued before its stores: timings + parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
O=gpurun_out/r02aa_t.log
for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000" "C3b 4.0 100000" "C1 2.0 400000" "P8192 2.0 10000"; do
  set -- $c; echo "== $1" >> $O
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|rror" >> $O
done
for t in 1 2; do echo "== C5 tex $t" >> $O
  CBP_WARP_TEX=$t timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --reps 3 2>&1 | grep -E "best|rror" >> $O
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02aa_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02aa_parity.log
cat $O; tail -2 gpurun_out/r02aa_parity.log
