#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for c in "C3b 4.0 100000 0" "C5 2.5 100000 0" "P8192 1.5 10000 0" "C4 1.5 3000 2"; do
  set -- $c; echo "== $1" >> gpurun_out/r02u_t.log
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 2 --rule $4 2>&1 | grep -E "best|Error|error|threads" >> gpurun_out/r02u_t.log
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peg.py -x -q --timeout 900 -p no:cacheprovider -k "C3b or c3b or P8192 or size_limits or degree_one" > gpurun_out/r02u_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02u_parity.log
grep -E "==|best|threads" gpurun_out/r02u_t.log; tail -2 gpurun_out/r02u_parity.log
