#!/bin/bash
# A/B: batched LLR loads at a frame's start (libcbp.so vs libcbp_chan.so) and the next row's slot-0 R words requested
# in the row's last slot (libcbp_rpre.so, CBP_RPRE=1); parity subsets; ncu --set full of one channel launch
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
ab() { for lib in "$@"; do for c in "C5 2.5" "C3a 1.5" "C3b 4.0" "P2048 2.5" "C2 2.0"; do set -- $c
  echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done; }
{ ab libcbp_chan.so libcbp.so libcbp_rpre.so libcbp_chan.so libcbp.so libcbp_rpre.so
  for lib in libcbp_chan.so libcbp.so libcbp_rpre.so; do echo "== $lib decode $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --mode decode --reps 5 --frames 200000 2>&1 | grep best)"; done
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "not all_frames" 2>&1 | tail -2
  CBP_LIB=$PWD/paper_2305_05286_b200/libcbp_rpre.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peg.py -m gpu -x -q -p no:cacheprovider -k "not all_frames" 2>&1 | tail -2
} > gpurun_out/r02bx_ab.log 2>&1
cat gpurun_out/r02bx_ab.log
timeout 600 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_warp -o gpurun_out/r02bx_chan -f \
   python tools/time_channel.py --config C5 --frames 100000 --reps 1 > gpurun_out/r02bx_ncu.log 2>&1
tail -3 gpurun_out/r02bx_ncu.log
