#!/bin/bash
# end-of-milestone measurement: bench (default), ncu launch list of the same command, ncu --set full of the
# dominant kernel on the bench workload, full GPU suite
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02ba_bench.json 2> gpurun_out/r02ba_bench.err; echo "bench rc=$?" >> gpurun_out/r02ba_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02ba_launches.csv \
   python bench.py --steps 2 --warmup 3 > gpurun_out/r02ba_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -s 1 -c 1 -k regex:cbp_warp -o gpurun_out/r02ba_c5 -f \
   python tools/prof_one.py --config C5 --ebn0 2.5 --frames 50000 --warm 0 > gpurun_out/r02ba_ncu.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/r02ba_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02ba_pytest.log
tail -c 1500 gpurun_out/r02ba_bench.json; tail -3 gpurun_out/r02ba_pytest.log
