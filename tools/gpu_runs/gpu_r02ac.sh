#!/bin/bash
# launch-bound A/B for the byte-H layout
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
O=gpurun_out/r02ac_t.log
for lib in build/libcbp_m640.so build/libcbp_a.so build/libcbp_b.so; do
  for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000" "C3b 4.0 100000" "C3a 2.0 100000"; do
   set -- $c; echo "== $1 lib=$lib" >> $O
   CBP_LIB=$lib timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "threads|best|rror" >> $O
  done
done
cat $O
