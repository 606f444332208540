#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for lib in "" "build/var/libcbp_m416.so" "build/var/libcbp_lean448.so"; do
for c in "C5 2.5 100000" "C2 2.0 200000"; do
  set -- $c; echo "== $lib $1" >> gpurun_out/r02o_t.log
  CBP_LIB=$lib timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|Error|error|threads" >> gpurun_out/r02o_t.log
done; done
for c in "C3b 4.0 100000" "P2048 2.0 100000"; do
  set -- $c; echo "== $1" >> gpurun_out/r02o_t.log
  timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|Error|error" >> gpurun_out/r02o_t.log
done
echo "== C4" >> gpurun_out/r02o_t.log
timeout 300 python tools/prof_one.py --config C4 --ebn0 1.5 --frames 3000 --reps 2 --rule 2 2>&1 | grep -E "best|threads" >> gpurun_out/r02o_t.log
grep -E "==|best|threads" gpurun_out/r02o_t.log
