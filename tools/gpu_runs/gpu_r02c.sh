#!/bin/bash
# time split of the fused ber_sim on C5 and C2: ber_sim vs channel + decode
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/split_ber.py --config C5 --ebn0 2.5 --frames 400000
timeout 300 python tools/split_ber.py --config C5 --ebn0 2.5 --frames 400000
timeout 300 python tools/split_ber.py --config C2 --ebn0 2.0 --frames 400000
} > gpurun_out/r02c_split.log 2>&1
cat gpurun_out/r02c_split.log
