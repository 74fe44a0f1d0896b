#!/bin/bash
# One `ncu --set full` capture of the first launch of every kernel of the C2
# bench step and of the C3 (minpts 100) step, plus the C2 launch list.
# Usage: tools/profile_all_kernels.sh <tag>
TAG=${1:-r01i}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
$NCU --set full --clock-control none --kernel-id ::regex:^k_:1 -o gpurun_out/${TAG}_c2_all -f \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
$NCU -i gpurun_out/${TAG}_c2_all.ncu-rep --page raw --csv > gpurun_out/${TAG}_c2_all_raw.csv 2>&1
$NCU --set full --clock-control none --kernel-id ::regex:^k_fd_:1 -o gpurun_out/${TAG}_c3_fd -f \
     python tools/configs.py C3 > /dev/null 2>&1
$NCU -i gpurun_out/${TAG}_c3_fd.ncu-rep --page raw --csv > gpurun_out/${TAG}_c3_fd_raw.csv 2>&1
echo done
