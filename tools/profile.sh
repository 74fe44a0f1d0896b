#!/bin/bash
# Profiling recipe (run on the GPU box from the repo root; /opt/skills/guides/B200_PROFILING.md):
#   1. launch list of one bench invocation (per-launch device time, cold-cache, serialised)
#   2. one `ncu --set full` capture of the dominant kernel
# Usage: tools/profile.sh <tag> [kernel-regex] [extra bench args]
set -u
TAG=${1:-r01}
KREGEX=${2:-k_fd_main}
shift 2 || true
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/${TAG}_launches.csv \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${TAG}_launches_bench.log 2>&1
$NCU --set full --clock-control none --import-source on -k regex:${KREGEX} -s 0 -c 1 \
     -o gpurun_out/${TAG}_${KREGEX} -f \
     python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/${TAG}_full_bench.log 2>&1
$NCU -i gpurun_out/${TAG}_${KREGEX}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${KREGEX}_raw.csv 2>&1
$NCU -i gpurun_out/${TAG}_${KREGEX}.ncu-rep --page details --csv > gpurun_out/${TAG}_${KREGEX}_details.csv 2>&1
echo done
