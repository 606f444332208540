#!/bin/bash
# GPU tests, then frames-per-lane A/B timing (ber_sim, best of 3) per config and algorithm
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q --timeout 900 -p no:cacheprovider $PYTEST_ARGS > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  tail -15 gpurun_out/pytest_gpu.log
fi
for c in ${CONFIGS:-C2 C3a C3b C1}; do
  for alg in ${ALGS:-0 1}; do
    for fpl in 1 2; do
      echo "== $c alg=$alg fpl=$fpl"
      timeout 150 python tools/prof_one.py --config $c --ebn0 ${EB:-2.0} --reps 3 --alg $alg --fpl $fpl --frames ${FRAMES:-100000} 2>&1 | grep -E "best|Error|error" | cut -c1-200
    done
  done
done
