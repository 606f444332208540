#!/bin/bash
# ncu --set full (with source) of C2 ber_sim launches; VARIANTS="alg:fpl ..." -> gpurun_out/prof_a<alg>_p<fpl>.ncu-rep
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for v in ${VARIANTS:-0:1 0:2}; do
  alg=${v%%:*}; fpl=${v##*:}
  CMD="python tools/prof_one.py --warm 0 --config ${CFG:-C2} --ebn0 2.0 --frames ${FRAMES:-100000} --alg $alg --fpl $fpl"
  timeout 300 $CMD > gpurun_out/prof_plain_a${alg}_p${fpl}.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:cbp_kernel -s 1 -c 1 -o gpurun_out/prof_a${alg}_p${fpl} -f $CMD > gpurun_out/prof_ncu_a${alg}_p${fpl}.log 2>&1
  echo "variant $v rc=$?"; grep -E "best|threads" gpurun_out/prof_plain_a${alg}_p${fpl}.log | cut -c1-200
done
