#!/bin/bash
# min-sum vs log-tanh timing lines (ber_sim, C2/C3a, best of 3)
cd "$GRAFT_REPO_ROOT" || exit 1
for c in ${CONFIGS:-C2 C3a}; do
  for alg in 0 1; do
    for eb in ${EBS:-2.0 3.0}; do
      echo "== $c alg=$alg eb=$eb"
      timeout 150 python tools/prof_one.py --config $c --ebn0 $eb --reps 3 --alg $alg --frames ${FRAMES:-100000} 2>&1 | tail -2 | cut -c1-240
    done
  done
done
