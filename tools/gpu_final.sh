#!/bin/bash
# Round-end evidence on one GPU: every GPU test (incl. the full-size reference
# parity runs), bench (+ CPU leg) and the reference arm, the config table,
# the launch list + one ncu --set full capture of the main pass, summaries.
TAG=${1:-r02q}
KERNEL=${2:-k_fd_main_fof}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/${TAG}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/${TAG}_smoke.log 2>&1; tail -2 gpurun_out/${TAG}_smoke.log
tail -3 gpurun_out/${TAG}_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
timeout 1200 python tools/configs.py C1 C2 C2db C3 C3fd C4 C4fd C5 > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err
timeout 900 tools/profile.sh ${TAG} ${KERNEL} --no-graph > /dev/null 2>&1
python tools/summarize_ncu.py ${TAG} gpurun_out/${TAG}_launches.csv gpurun_out/${TAG}_${KERNEL}_raw.csv ${KERNEL} > /dev/null 2>&1
cp profiles/${TAG}_ncu_summary.md profiles/traffic.json gpurun_out/ 2>/dev/null
cut -c1-300 gpurun_out/${TAG}_bench.json; cut -c1-300 gpurun_out/${TAG}_bench_ref.json
python -c "
import json
for l in open('gpurun_out/${TAG}_configs.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(d.get('config'), d.get('ms_best'), d.get('stage_ms',{}).get('sort'), d.get('stats',{}).get('pair_resolutions'), d.get('check', d.get('cross_check')))
"
