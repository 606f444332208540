#!/bin/bash
# time split: fused ber_sim vs channel + decode on the same frames
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{ for c in "C5 2.5" "C3a 1.5" "C2 2.0" "P2048 2.5"; do set -- $c; timeout 300 python tools/split_ber.py --config $1 --ebn0 $2 --frames 200000; done; } > gpurun_out/r02bh_split.log 2>&1
cat gpurun_out/r02bh_split.log
