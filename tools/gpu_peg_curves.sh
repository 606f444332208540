#!/bin/bash
# Denser schedule comparison on the paper's code families (QC-PEG, Fig. 6/7):
# CBP / LBP / FBP / min-sum CBP at the family's best alpha -> gpurun_out/curves_P*.jsonl
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python tools/compare_schedules.py --config P2048 --frames 1000000 --ebn0 1.0,1.25,1.5,1.75,2.0,2.25,2.5 \
  --alphas 0.8 > gpurun_out/curves_P2048.jsonl 2> gpurun_out/curves_P2048.err; echo "P2048 rc=$?"
timeout 2000 python tools/compare_schedules.py --config P8192 --frames 200000 --ebn0 0.75,0.875,1.0,1.125,1.25,1.375,1.5,1.625 \
  --alphas 0.95 > gpurun_out/curves_P8192.jsonl 2> gpurun_out/curves_P8192.err; echo "P8192 rc=$?"
