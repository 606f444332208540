#!/bin/bash
# frame-level parity audit at the BASELINE sizes on the final kernel of round 2, at a quarter of the full ranges
# (CBP_AUDIT_SCALE=0.25: C3a / C3b 2.5e6 frames at 7 points each, C5 2.5e8 frames fp32 + int8; per point every
# flagged frame up to 5000 and 25000 uniform samples re-decoded by the oracle)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
CBP_AUDIT=1 CBP_AUDIT_SCALE=0.25 CBP_AUDIT_OUT=gpurun_out/r02ce_parity_audit.json timeout 1500 python -m pytest tests/test_gpu_audit.py -m gpu -q -x -p no:cacheprovider --timeout 1500 > gpurun_out/r02ce_audit.log 2>&1
echo "rc=$?" >> gpurun_out/r02ce_audit.log; tail -4 gpurun_out/r02ce_audit.log
