#!/bin/bash
# one gpurun call: device facts, GPU tests, smoke, short bench
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
{ nvidia-smi; nvidia-smi topo -m; nproc; lscpu | head -20;
  python -c "import torch; p=torch.cuda.get_device_properties(0); print(p); print('L2', p.L2_cache_size, 'smem/blk optin', getattr(p,'shared_memory_per_block_optin',None), 'sms', p.multi_processor_count)"; } > gpurun_out/devquery.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 2 --warmup 1 --frames 200000 --cpu-frames 50 --e2e-frames 100000 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "bench rc=$?" >> gpurun_out/bench1.err
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench1.json | head -c 3000; tail -5 gpurun_out/bench1.err
