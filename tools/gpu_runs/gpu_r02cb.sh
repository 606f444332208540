#!/bin/bash
# end of round 2: park-path C2B rows through TEX as the default (A/B against the previous build on C3b, C4, P8192),
# full GPU suite, bench (default) + ncu launch list of the same command, smoke
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() { CBP_LIB=$PWD/paper_2305_05286_b200/$1 timeout 300 python tools/prof_one.py --config $2 --ebn0 $3 --reps 5 --frames $4 2>&1 | grep best; }
{ for rep in 1 2; do for lib in libcbp_prev.so libcbp.so; do
    echo "== $lib C3b 4.0 $(run $lib C3b 4.0 100000)"; echo "== $lib C4 1.5 $(run $lib C4 1.5 3000)"; echo "== $lib P8192 1.5 $(run $lib P8192 1.5 10000)"; done; done
} > gpurun_out/r02cb_ab.log 2>&1
cat gpurun_out/r02cb_ab.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 1500 -p no:cacheprovider > gpurun_out/r02cb_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02cb_pytest.log
tail -3 gpurun_out/r02cb_pytest.log
timeout 900 python bench.py > gpurun_out/r02cb_bench.json 2> gpurun_out/r02cb_bench.err; echo "bench rc=$?" >> gpurun_out/r02cb_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02cb_launches.csv \
   python bench.py --steps 2 --warmup 3 > gpurun_out/r02cb_ncu_launch.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r02cb_smoke.log 2>&1
tail -2 gpurun_out/r02cb_bench.err; tail -1 gpurun_out/r02cb_smoke.log
