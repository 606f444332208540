#!/bin/bash
# A/B: R words L2-only (libcbp.so) vs L2-only + L2 evict_last policy descriptor (libcbp_el.so, CBP_R_CG=2):
# time (prof_one, best of 5), DRAM bytes of the decode launch (ncu metrics pass), parity subset under the variant
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ab() { for lib in "$@"; do for c in "C5 2.5" "C3a 1.5" "C3b 4.0" "P2048 2.5"; do set -- $c
  echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done; }
{ ab libcbp_el.so libcbp.so libcbp_el.so libcbp.so
  for lib in libcbp.so libcbp_el.so; do
    CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -s 3 -c 1 -k regex:cbp_warp --csv python tools/prof_one.py --config C5 --ebn0 2.5 --frames 50000 --warm 0 2>&1 | grep -i "dram__\|gpu__time\|lts__" | sed "s/^/$lib /"
  done
  CBP_LIB=$PWD/paper_2305_05286_b200/libcbp_el.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not all_frames" 2>&1 | tail -2
} > gpurun_out/r02bv_ab.log 2>&1
cat gpurun_out/r02bv_ab.log
