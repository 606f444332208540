#!/bin/bash
# H as bytes (5N bytes per frame): warps per SM A/B (launch bounds 384 / 512 / 640) + parity
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
O=gpurun_out/r02ab_t.log
for lib in "" build/libcbp_m512.so build/libcbp_m640.so; do
 for t in 0 2; do
  for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000" "C3b 4.0 100000"; do
   set -- $c; echo "== $1 lib=$lib tex=$t" >> $O
   CBP_LIB=$lib CBP_WARP_TEX=$t timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "threads|best|rror" >> $O
  done
 done
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02ab_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02ab_parity.log
grep -E "==|best|rror" $O; tail -2 gpurun_out/r02ab_parity.log
