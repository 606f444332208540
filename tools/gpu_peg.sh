#!/bin/bash
# The paper's own code families (QC-PEG) on the GPU: parity tests, schedule
# comparison -> gpurun_out/schedules_P*.jsonl, min-sum alpha sweep -> gpurun_out/alpha_P*.jsonl
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peg.py -q -p no:cacheprovider > gpurun_out/pytest_peg.log 2>&1; tail -1 gpurun_out/pytest_peg.log
[ -n "$SKIP_SCHED" ] && exit 0
for c in P2048 P8192; do
  timeout 1200 python tools/alpha_sweep.py --config $c --frames ${FA:-20000} > gpurun_out/alpha_$c.jsonl 2> gpurun_out/alpha_$c.err; echo "alpha $c rc=$?"
done
timeout 1200 python tools/compare_schedules.py --config P2048 --frames ${F2048:-100000} --alphas 0.75,0.8 > gpurun_out/schedules_P2048.jsonl 2> gpurun_out/schedules_P2048.err; echo "P2048 rc=$?"
timeout 1500 python tools/compare_schedules.py --config P8192 --frames ${F8192:-100000} --alphas 0.75,0.9 > gpurun_out/schedules_P8192.jsonl 2> gpurun_out/schedules_P8192.err; echo "P8192 rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
