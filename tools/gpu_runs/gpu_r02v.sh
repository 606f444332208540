#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in "X=1" "CBP_WARP_KERNEL=0"; do
for c in "C4 1.5 3000 2" "C3b 4.0 100000 0"; do
  set -- $c; echo "== $v $1" >> gpurun_out/r02v_t.log
  env $v timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 2 --rule $4 2>&1 | grep -E "best|Error|error" >> gpurun_out/r02v_t.log
done; done
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider -k "c4 or C4 or size_limits or degree_one or layouts" > gpurun_out/r02v_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02v_parity.log
grep -E "==|best" gpurun_out/r02v_t.log; tail -2 gpurun_out/r02v_parity.log
