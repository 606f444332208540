#!/bin/bash
# BASELINE C5 at full size on one GPU: 10^9 frames at 2.5 dB, fp32 and int8 channel LLRs
# (resumable JSONL checkpoints via paper_2305_05286_b200.sweep) -> gpurun_out/c5_full_*.jsonl
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for m in 0 1; do
  SECONDS=0
  timeout 900 python -m paper_2305_05286_b200.sweep --config C5 --frames 1e9 --chunk 5e7 \
    --llr-mode $m --out gpurun_out/c5_full_llr$m.jsonl > gpurun_out/c5_full_llr$m.log 2>&1
  rc=$?; echo "wall ${SECONDS} s rc=$rc" >> gpurun_out/c5_full_llr$m.log
  echo "llr_mode $m"; tail -2 gpurun_out/c5_full_llr$m.log
done
