#!/bin/bash
# split-step bench on C5 + the new parity tests
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ber_count or fused_equals_split or channel_parity or ber_sim_parity" -p no:cacheprovider > gpurun_out/r02e_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02e_pytest.log
timeout 900 python bench.py --no-suite > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err; echo "bench rc=$?" >> gpurun_out/r02e_bench.err
tail -3 gpurun_out/r02e_pytest.log; tail -3 gpurun_out/r02e_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/r02e_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['frames_per_s'], d['ms_per_step']); print(json.dumps(d['roofline'])[:900]); print(d['int8_stream']['value'], d['int8_stream']['roofline_frac'], d['roofline_decode']['frac'], d['gpu_launches'], d['clocks'])"
