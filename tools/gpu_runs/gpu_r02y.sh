#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000" "C3b 4.0 100000"; do
  set -- $c; echo "== $1" >> gpurun_out/r02y_t.log
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|Error|error" >> gpurun_out/r02y_t.log
done
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02y_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02y_parity.log
grep -E "==|best" gpurun_out/r02y_t.log; tail -2 gpurun_out/r02y_parity.log
