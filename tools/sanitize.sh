#!/bin/bash
# compute-sanitizer on small instances of every algorithm (memcheck, racecheck
# of shared memory, synccheck). Writes gpurun_out/sanitize_*.log.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/san_run.py <<'PY'
import sys
sys.path.insert(0, ".")
import numpy as np
import paper_2103_05162_b200 as tb
ds = tb.Dataset.blobs(4, 400, 3, 5.0, 0.4, 3)
for algo, mp in ((0, 5), (0, 2), (1, 5), (1, 2), (2, 4)):
    r = tb.cluster(ds, 0.3, mp, tb.Algorithm(algo))
    print(algo, mp, r.stats["cluster_count"], r.stats["core_count"])
ds2 = tb.Dataset.blobs(3, 300, 2, 4.0, 0.3, 5)
for algo, mp in ((0, 4), (1, 4)):
    r = tb.cluster(ds2, 0.2, mp, tb.Algorithm(algo))
    print("2d", algo, mp, r.stats["cluster_count"])
st, rep = tb.verify(ds, 0.3, 5)
print("verify", int(st))
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python /tmp/san_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log
done
