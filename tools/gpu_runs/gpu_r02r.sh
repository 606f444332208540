#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for lib in "" "build/var/libcbp_full.so" "build/var/libcbp_full320.so"; do
for c in "C5 2.5 100000" "C2 2.0 200000" "P2048 2.0 100000"; do
  set -- $c; echo "== $lib $1" >> gpurun_out/r02r_t.log
  CBP_LIB=$lib timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|Error|error" >> gpurun_out/r02r_t.log
done; done
grep -E "==|best" gpurun_out/r02r_t.log
