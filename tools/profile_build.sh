#!/bin/bash
# ncu --set full of the build kernels (one launch each) for the current bench config.
TAG=${1:-b1}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:"${KREG:-k_refit|k_karras}" -s 0 -c ${KCNT:-2} \
     -o gpurun_out/${TAG}_build -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_build_bench.log 2>&1
$NCU -i gpurun_out/${TAG}_build.ncu-rep --page raw --csv > gpurun_out/${TAG}_build_raw.csv 2>&1
$NCU -i gpurun_out/${TAG}_build.ncu-rep --page details --csv > gpurun_out/${TAG}_build_details.csv 2>&1
echo done
