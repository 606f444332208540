#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in "X=1" "CBP_WARP_TEX=2"; do
for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000" "C3b 4.0 100000"; do
  set -- $c; echo "== $v $1" >> gpurun_out/r02l_t.log
  env $v timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|Error|error" >> gpurun_out/r02l_t.log
done; done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02l_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02l_parity.log
cat gpurun_out/r02l_t.log; tail -3 gpurun_out/r02l_parity.log
