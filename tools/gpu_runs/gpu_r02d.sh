#!/bin/bash
# split ber_sim A/B (fused vs channel + decode) and the ber_sim / channel parity tests
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{
timeout 600 python tools/ab_split.py --config C5 --ebn0 2.5 --frames 400000
timeout 600 python tools/ab_split.py --config C5 --ebn0 2.5 --frames 2000000 --reps 3
timeout 600 python tools/ab_split.py --config C2 --ebn0 2.0 --frames 400000
timeout 600 python tools/ab_split.py --config C3b --ebn0 4.0 --frames 400000
timeout 900 python -m pytest tests -m gpu -q -x -k "ber or channel or counts" -p no:cacheprovider 2>&1 | tail -5
} > gpurun_out/r02d.log 2>&1
cat gpurun_out/r02d.log
