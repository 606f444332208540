#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
O=gpurun_out/r02ah_t.log
for c in "C4 1.5 3000 2" "P8192 2.0 10000 0" "C5 2.5 100000 0" "C2 2.0 200000 2"; do
  set -- $c; echo "== $1 rule $4" >> $O
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --rule $4 --reps 3 2>&1 | grep -E "best|rror" >> $O
done
timeout 600 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_warp -o gpurun_out/r02ah_c4 -f \
   python tools/prof_one.py --config C4 --ebn0 1.5 --frames 1000 --rule 2 --warm 0 > gpurun_out/r02ah_ncu.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02ah_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02ah_parity.log
cat $O; tail -3 gpurun_out/r02ah_parity.log
