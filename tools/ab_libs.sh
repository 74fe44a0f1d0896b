#!/bin/bash
# A/B of library variants in paper_2103_05162_b200/ab/*.so on the given configs.
# tools/ab_libs.sh C2 C3fd
for L in paper_2103_05162_b200/ab/*.so; do
  echo "== $L"
  TCB_LIB_PATH=$PWD/$L python tools/configs.py "$@" 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(d['config'], d['ms_best'], {k: v for k, v in d['stage_ms'].items() if v > 0.05}, d['stats']['pair_resolutions'], d['stats']['distance_evaluations'], d.get('cross_check'))
"
done
