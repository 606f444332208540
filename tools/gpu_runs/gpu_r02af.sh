#!/bin/bash
# A/B: part of the B2V phi rows through TEX (balances the LSU and TEX data pipes)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
O=gpurun_out/r02af_t.log
for lib in "" build/libcbp_t11.so build/libcbp_t49.so build/libcbp_t55.so; do
  for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000"; do
   set -- $c; echo "== $1 lib=$lib" >> $O
   CBP_LIB=$lib timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|rror" >> $O
  done
done
cat $O
