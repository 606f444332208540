#!/bin/bash
# A/B: register-resident rows (default) vs all rows through the parked path; ncu of the default on C5
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for lib in "" "build/var/libcbp_dc0.so"; do
  for c in "C5 2.5 100000" "C2 2.0 200000"; do
    set -- $c; echo "== lib=$lib $1" >> gpurun_out/r02d_ab.log
    CBP_LIB=$lib timeout 300 python tools/prof_one.py --config $1 --ebn0 $2 --frames $3 --reps 3 2>&1 | grep -E "best|threads" >> gpurun_out/r02d_ab.log
  done
done
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_kernel -o gpurun_out/r02d_c5 -f \
   python tools/prof_one.py --config C5 --ebn0 2.5 --frames 50000 --warm 0 > gpurun_out/r02d_ncu.log 2>&1
cat gpurun_out/r02d_ab.log
