#!/bin/bash
# producer-side CBP kernel + phi contract v3: parity suite, smoke, C5 timings per geometry
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python __graft_entry__.py smoke > gpurun_out/r02b_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02b_smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider > gpurun_out/r02b_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02b_parity.log
for v in "" "CBP_MULTI_MAXT=512" "CBP_SPLIT_R=0"; do
  echo "== $v" >> gpurun_out/r02b_c5.log
  env $v timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 200000 --reps 3 >> gpurun_out/r02b_c5.log 2>&1
done
for c in "C2 2.0" "C1 2.0" "C3b 4.0" "C4 1.5" "P2048 2.0"; do
  set -- $c; echo "== $1" >> gpurun_out/r02b_other.log
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $([ $1 = C4 ] && echo 3000 || echo 200000) --reps 2 --rule $([ $1 = C4 ] && echo 2 || echo 0) >> gpurun_out/r02b_other.log 2>&1
done
tail -3 gpurun_out/r02b_smoke.log; tail -5 gpurun_out/r02b_parity.log; grep -E "==|best|launch|threads" gpurun_out/r02b_c5.log gpurun_out/r02b_other.log
