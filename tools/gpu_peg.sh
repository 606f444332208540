#!/bin/bash
# Schedule comparison on the paper's own code families (QC-PEG) ->
# gpurun_out/schedules_P*.jsonl, plus the ABI error-path test.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k abi_error > gpurun_out/pytest_abi.log 2>&1; tail -1 gpurun_out/pytest_abi.log
timeout 1200 python tools/compare_schedules.py --config P2048 --frames ${F2048:-100000} > gpurun_out/schedules_P2048.jsonl 2> gpurun_out/schedules_P2048.err; echo "P2048 rc=$?"
timeout 1500 python tools/compare_schedules.py --config P8192 --frames ${F8192:-20000} > gpurun_out/schedules_P8192.jsonl 2> gpurun_out/schedules_P8192.err; echo "P8192 rc=$?"
