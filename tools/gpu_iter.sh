#!/bin/bash
# One GPU iteration: bench (no CPU leg) summary.
TAG=${1:-it}
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stage_ms'],d['graph'],d['e2e']['ms_per_step'],d['gpu_launches'])"
tail -3 gpurun_out/${TAG}_bench.err
