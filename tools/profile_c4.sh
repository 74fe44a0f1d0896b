#!/bin/bash
# DenseBox kernels on C4 (80M 2D taxi-like, eps 0.001, minpts 1000): launch
# list + one --set full capture each of the core and main passes.
TAG=${1:-r01g}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_c4_launches.csv python tools/configs.py C4 > /dev/null 2>&1
for K in k_db_core k_db_main_ranged; do
  $NCU --set full --clock-control none --import-source on -k regex:${K} -s 0 -c 1 \
       -o gpurun_out/${TAG}_c4_${K} -f python tools/configs.py C4 > /dev/null 2>&1
  $NCU -i gpurun_out/${TAG}_c4_${K}.ncu-rep --page raw --csv > gpurun_out/${TAG}_c4_${K}_raw.csv 2>&1
done
echo done
