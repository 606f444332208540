#!/bin/bash
# last call of round 2: the committed tree as the driver will run it -- build(), GPU suite, smoke, the reference arm, bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); print('build ok')" > gpurun_out/r02cd_build.log 2>&1; tail -1 gpurun_out/r02cd_build.log
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 1500 -p no:cacheprovider > gpurun_out/r02cd_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02cd_pytest.log
tail -3 gpurun_out/r02cd_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02cd_smoke.log 2>&1; tail -1 gpurun_out/r02cd_smoke.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02cd_ref.json 2> gpurun_out/r02cd_ref.err; echo "ref rc=$?"; tail -c 700 gpurun_out/r02cd_ref.json
timeout 900 python bench.py > gpurun_out/r02cd_bench.json 2> gpurun_out/r02cd_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r02cd_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['frames_per_s'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['step_frac'], d['e2e']['value'], d['clocks'])"
