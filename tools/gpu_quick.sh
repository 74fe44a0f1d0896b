#!/bin/bash
# Quick GPU iteration: gpu tests (fast subset unless FULL=1) + bench line.
TAG=${1:-q}
mkdir -p gpurun_out
if [ "${FULL:-0}" = "1" ]; then
  timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/${TAG}_pytest_gpu.log
else
  timeout 600 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -15 > gpurun_out/${TAG}_pytest_gpu.log
fi
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -3 gpurun_out/${TAG}_pytest_gpu.log; cat gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
