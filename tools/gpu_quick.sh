#!/bin/bash
# gpu tests (optionally -k filter) + quick perf lines
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider $PYTEST_ARGS > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
for c in ${CONFIGS:-C2 C3a C3b C1}; do timeout 120 python tools/prof_one.py --config $c --reps 2 --frames ${FRAMES:-100000} 2>&1 | tail -2 | cut -c1-220; done
