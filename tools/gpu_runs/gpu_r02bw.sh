#!/bin/bash
# channel-only launch: throughput form (two Philox blocks per step, inline Box-Muller, 128-bit LLR stores) and the
# sign-word encoder -- A/B against the previous build (libcbp_old.so), parity subset, bench without the suite
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{ for lib in libcbp_old.so libcbp.so libcbp_old.so libcbp.so; do for c in "C5 2.5" "C2 2.0" "C3b 4.0" "P2048 2.5"; do set -- $c
    echo "== $lib $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/time_channel.py --config $1 --ebn0 $2 --frames 524288 2>&1 | tail -1)"; done; done
  for lib in libcbp_old.so libcbp.so; do echo "== $lib int8 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/time_channel.py --config C5 --mode 1 --frames 524288 2>&1 | tail -1)"; done
  for lib in libcbp_old.so libcbp.so; do for c in "C5 2.5" "C2 2.0"; do set -- $c
    echo "== $lib $1 $2 $(CBP_LIB=$PWD/paper_2305_05286_b200/$lib timeout 200 python tools/prof_one.py --config $1 --ebn0 $2 --reps 5 --frames 100000 2>&1 | grep best)"; done; done
  timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peg.py -m gpu -x -q -p no:cacheprovider -k "channel or ber_sim or ber_count or split or symmetry" 2>&1 | tail -3
} > gpurun_out/r02bw_ab.log 2>&1
cat gpurun_out/r02bw_ab.log
timeout 900 python bench.py --no-suite > gpurun_out/r02bw_bench.json 2> gpurun_out/r02bw_bench.err; echo "bench rc=$?" >> gpurun_out/r02bw_bench.err
tail -2 gpurun_out/r02bw_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r02bw_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['frames_per_s'], d['ms_per_step']); r=d['roofline']; print(r['frac'], r['step_frac'], r['channel_ms_per_step'], r['launch_ms'], r['share_of_step']); print(d['int8_stream']['value'], d['clocks'])"
