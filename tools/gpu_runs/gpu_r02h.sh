#!/bin/bash
# cbp_warp_kernel: parity suite + timings
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r02h_smoke.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 900 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02h_parity.log 2>&1; echo "rc=$?" >> gpurun_out/r02h_parity.log
for c in "C5 2.5 100000" "C2 2.0 200000" "C3b 4.0 100000" "P2048 2.0 100000" "P8192 1.5 10000"; do
  set -- $c; echo "== $1" >> gpurun_out/r02h_t.log
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|threads|Error|error" >> gpurun_out/r02h_t.log
done
echo "== C5 old kernel" >> gpurun_out/r02h_t.log
CBP_WARP_KERNEL=0 timeout 300 python tools/prof_one.py --config C5 --ebn0 2.5 --frames 100000 --reps 3 2>&1 | grep -E "best|threads" >> gpurun_out/r02h_t.log
tail -3 gpurun_out/r02h_smoke.log; tail -4 gpurun_out/r02h_parity.log; cat gpurun_out/r02h_t.log
