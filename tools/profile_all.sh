#!/bin/bash
# Full profiling set for profiles/: launch list + ncu --set full of the main
# pass and of the top build kernels; summaries written by tools/summarize_ncu.py.
TAG=${1:-r01d}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
$NCU --set full --clock-control none --import-source on \
     -k regex:"k_fd_main" -s 0 -c 1 \
     -o gpurun_out/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
$NCU -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_full_raw.csv 2>/dev/null
python tools/summarize_ncu.py ${TAG} gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_full_raw.csv k_fd_main > /dev/null
cp profiles/${TAG}_ncu_summary.md profiles/traffic.json gpurun_out/
echo profiled
