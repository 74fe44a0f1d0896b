#!/bin/bash
# Launch list only (cheap): per-kernel device times of one bench step.
TAG=${1:-l}
shift
mkdir -p gpurun_out
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > /dev/null 2>&1
python - "$TAG" <<'PY'
import csv, collections, sys
tag = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/{tag}_launches.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[h], rows[h + 1:]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.OrderedDict()
for r in data:
    name = r[ik].split("(")[0].replace("void ", "")
    if "::k_" in name: name = "k_" + name.split("::k_", 1)[1]
    agg.setdefault(name, [0, 0.0]); agg[name][0] += 1; agg[name][1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:50]:50s} n={c:4d} avg={v/c/1e3:9.1f}us share={v/tot*100:5.1f}%")
PY
