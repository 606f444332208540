#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 1200 -p no:cacheprovider -k "not all_frames" > gpurun_out/r02ai_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/r02ai_gpu.log
tail -3 gpurun_out/r02ai_gpu.log
