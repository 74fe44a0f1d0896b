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
# dense cells with long member runs (member trees, spatial tree, runs)
rng = np.random.default_rng(4)
g = np.stack(np.meshgrid(np.arange(60), np.arange(60)), -1).reshape(-1, 2)
lat = (g * 0.01 + rng.uniform(-0.004, 0.004, g.shape)).astype(np.float32)
lat = np.concatenate([lat, np.repeat(lat[:50], 40, axis=0)])
for mp in (2, 20, 200):
    r = tb.cluster(tb.Dataset.from_array(lat), 0.1, mp, tb.Algorithm.DENSEBOX)
    print("dense", mp, r.stats["cluster_count"], r.stats["distance_evaluations"])
# Morton prefix sort: small equal-prefix groups (fix-up) and a > 256 group (fallback)
wide = rng.uniform(-5, 5, (3000, 3))
for pts in (np.concatenate([wide, wide[:500] + 1e-6]), np.concatenate([wide, np.repeat(wide[:1], 400, axis=0)])):
    r = tb.cluster(tb.Dataset.from_array(pts.astype(np.float32)), 0.3, 3, tb.Algorithm.FDBSCAN)
    print("prefix", r.stats["cluster_count"], r.stats["pair_resolutions"])
# keyed run, local context, binary load to the device
import torch
from paper_2103_05162_b200.shard import DeviceEngine
eng = DeviceEngine("cuda:0")
x = torch.from_numpy(ds.coords()).cuda()
keys = torch.arange(5000, 5000 + x.shape[0], dtype=torch.int32, device="cuda")
lab, core = eng.cluster_keyed(x, keys, 0.3, 2)
ctx = eng.local(x, keys, 0.3)
cf = ctx.core_flags(5)
lab2 = ctx.cluster(cf)
ctx.close()
torch.cuda.synchronize()
print("keyed", int((lab >= 0).sum()), int((lab2 >= 0).sum()))
ds.save("/tmp/san.bin")
y = tb.load_device("/tmp/san.bin")
print("load", bool(torch.equal(y, x)))
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python /tmp/san_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log
done
