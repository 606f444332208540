#!/bin/bash
# A/B: R words with an L2 persisting access property (libcbp_evl.so) vs ld/st.cg (libcbp.so); DRAM bytes of each
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ab() { for lib in "$@"; do for c in "C5 2.5" "C3b 4.0"; do set -- $c
  echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done; }
{
ab libcbp.so libcbp_evl.so libcbp.so libcbp_evl.so
for lib in libcbp.so libcbp_evl.so; do
  CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum -k regex:cbp_warp -s 1 -c 1 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 50000 --warm 0 2>&1 | grep -E "dram__|lts__|gpu__time"
done
} > gpurun_out/r02bp_ab.log 2>&1
cat gpurun_out/r02bp_ab.log
