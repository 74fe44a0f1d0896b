mkdir -p gpurun_out
TAG=mg1
TCB_BENCH_BACKEND=gloo TCB_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 3 --points 8000000 > gpurun_out/${TAG}_bench_n2_smoke.json 2> gpurun_out/${TAG}_bench_n2_smoke.err
echo "n2 rc=$?"; tail -1 gpurun_out/${TAG}_bench_n2_smoke.json | cut -c1-400; tail -3 gpurun_out/${TAG}_bench_n2_smoke.err
TCB_SHARD_TIMING=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --sharded --force-exchange --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_nccl1.json 2> gpurun_out/${TAG}_bench_nccl1.err
echo "nccl1 rc=$?"; tail -1 gpurun_out/${TAG}_bench_nccl1.json | cut -c1-400
timeout 900 python -m pytest tests/test_shard.py -q -m gpu 2>&1 | tail -2
