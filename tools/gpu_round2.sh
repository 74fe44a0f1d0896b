#!/bin/bash
# Tests (all gpu incl. slow + sharded), bench, N=2 sharded smoke on one GPU, profiles.
TAG=${1:-r01c}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
TCB_BENCH_BACKEND=gloo TCB_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --points 8000000 > gpurun_out/${TAG}_bench_n2_smoke.json 2> gpurun_out/${TAG}_bench_n2_smoke.err
timeout 900 tools/profile.sh ${TAG} k_fd_main > /dev/null 2>&1
python tools/summarize_ncu.py ${TAG} gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_k_fd_main_raw.csv k_fd_main > /dev/null 2>&1
cp profiles/${TAG}_ncu_summary.md profiles/traffic.json gpurun_out/ 2>/dev/null
tail -4 gpurun_out/${TAG}_pytest_gpu.log; cat gpurun_out/${TAG}_bench.json | cut -c1-600; tail -2 gpurun_out/${TAG}_bench_n2_smoke.json | cut -c1-400; tail -3 gpurun_out/${TAG}_bench_n2_smoke.err
