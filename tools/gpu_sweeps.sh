#!/bin/bash
# f3 sweeps with the reference column (bench.py --sweep), CSVs into gpurun_out/.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 600 python -m pytest -x -q tests/test_bench.py 2>&1 | tail -3
for s in hacc-n hacc-minpts hacc-eps taxi-minpts; do
  timeout 1500 python bench.py --sweep $s --sweep-out gpurun_out/${TAG}_sweep_$s.csv 2> gpurun_out/${TAG}_sweep_$s.log
  echo "$s rc=$?"; cat gpurun_out/${TAG}_sweep_$s.csv
done
