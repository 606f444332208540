#!/bin/bash
# A/B timing of library variants: bash tools/gpu_ab.sh lib1 lib2 ...   (each: 3 reps of prof_one, best)
cd "$GRAFT_REPO_ROOT" || exit 1
for lib in "$@"; do
  for c in ${CONFIGS:-C2 C3a}; do
    echo "== $lib $c"
    CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $c --ebn0 2.0 --reps 5 --frames ${FRAMES:-100000} 2>&1 | grep best
  done
done
