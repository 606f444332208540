#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in "X=1" "CBP_WARP_KERNEL=0"; do
for c in "C4 1.5 3000 2" "P8192 1.5 10000 0" "C3b 4.0 100000 0" "C1 2.0 1000000 0"; do
  set -- $c; echo "== $v $1" >> gpurun_out/r02t_t.log
  env $v timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 2 --rule $4 2>&1 | grep -E "best|Error|error|threads" >> gpurun_out/r02t_t.log
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peg.py -x -q --timeout 900 -p no:cacheprovider -k "c4 or C4 or P8192 or layouts or size_limits" > gpurun_out/r02t_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02t_parity.log
grep -E "==|best|threads" gpurun_out/r02t_t.log; tail -3 gpurun_out/r02t_parity.log
