#!/bin/bash
# ncu --set full of the first k_fd_main_fof launch of one C2 run per library
# variant: tools/ncu_variant.sh <tag> <lib.so>...
TAG=$1; shift
NCU=/usr/local/cuda/bin/ncu
for L in "$@"; do
  v=$(basename $L .so)
  TCB_LIB_PATH=$PWD/$L $NCU --set full --clock-control none --import-source on \
    -k regex:k_fd_main_fof -s 1 -c 1 -o gpurun_out/${TAG}_${v} -f \
    python tools/configs.py C2 > /dev/null 2>&1
  $NCU -i gpurun_out/${TAG}_${v}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${v}_raw.csv 2>&1
done
