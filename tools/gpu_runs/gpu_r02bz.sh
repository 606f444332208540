#!/bin/bash
# final bench of the round (suite warm-ups at full size) + the ncu launch list of the same command
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02bz_bench.json 2> gpurun_out/r02bz_bench.err; echo "bench rc=$?" >> gpurun_out/r02bz_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02bz_launches.csv \
   python bench.py --steps 2 --warmup 3 > gpurun_out/r02bz_ncu_launch.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02bz_smoke.log 2>&1
tail -c 600 gpurun_out/r02bz_bench.json; tail -2 gpurun_out/r02bz_bench.err; tail -1 gpurun_out/r02bz_smoke.log
