#!/bin/bash
# Tests (all gpu incl. slow + sharded), bench (+ reference arm), N=2 sharded
# smoke on one GPU, launch list + ncu --set full of the main pass, summaries.
TAG=${1:-r01c}
KERNEL=${2:-k_fd_main_fof}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
TCB_BENCH_BACKEND=gloo TCB_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --points 8000000 > gpurun_out/${TAG}_bench_n2_smoke.json 2> gpurun_out/${TAG}_bench_n2_smoke.err
timeout 900 tools/profile.sh ${TAG} ${KERNEL} > /dev/null 2>&1
python tools/summarize_ncu.py ${TAG} gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_${KERNEL}_raw.csv ${KERNEL} > /dev/null 2>&1
cp profiles/${TAG}_ncu_summary.md profiles/traffic.json gpurun_out/ 2>/dev/null
tail -4 gpurun_out/${TAG}_pytest_gpu.log; cut -c1-400 gpurun_out/${TAG}_bench.json; cut -c1-300 gpurun_out/${TAG}_bench_ref.json; tail -2 gpurun_out/${TAG}_bench_n2_smoke.json | cut -c1-300; tail -3 gpurun_out/${TAG}_bench_n2_smoke.err
# the NCCL branch of the sharded path's collectives on the box's one GPU
TCB_SHARD_TIMING=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --sharded --force-exchange --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_nccl1.json 2> gpurun_out/${TAG}_bench_nccl1.err
tail -1 gpurun_out/${TAG}_bench_nccl1.json | cut -c1-300; grep "stage ms" gpurun_out/${TAG}_bench_nccl1.json gpurun_out/${TAG}_bench_nccl1.err | tail -2
