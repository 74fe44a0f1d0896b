#!/bin/bash
# One GPU iteration: A/B of ab/*.so on C2, a parity subset, a bench summary.
TAG=${1:-it}
mkdir -p gpurun_out
rm -f gpurun_out/${TAG}_ab.txt
bash tools/ab_probe.sh ${TAG} C2 C2 C1 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_c_client.py -x -q -m "gpu and not slow" 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
python -c "import json;d=json.loads(open('gpurun_out/${TAG}_bench.json').read().strip().splitlines()[-1]);print(d['ms_per_step'],d['stage_ms'],d['graph'],d['e2e']['ms_per_step'],d['gpu_launches'])"
python - <<PY
import json
for l in open('gpurun_out/${TAG}_ab.txt'):
    n, j = l.split(' ', 1)
    try: d = json.loads(j)
    except Exception: print(l[:200]); continue
    print(n, d['config'], d['ms_best'], d['stage_ms'].get('sort'), d['stage_ms'].get('main'), d['digest'])
PY
