mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "captured or async_status or massive or invalid or morton_prefix" 2>&1 | tail -25 > gpurun_out/r02n_new.log
bash tools/gpu_quick.sh r02n
cat gpurun_out/r02n_new.log
