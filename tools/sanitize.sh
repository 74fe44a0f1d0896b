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
# eps near the extent (every child a contained run: full action queues) and tiny eps
from oracle import oracle
h = oracle.hacc_like(20000)
hd = tb.Dataset.from_array(h)
for eps in (0.3, 1.0, 1e-4):
    for algo, mp in ((0, 2), (0, 5), (1, 2), (1, 50)):
        r = tb.cluster(hd, eps, mp, tb.Algorithm(algo))
        print("eps", eps, algo, mp, r.stats["cluster_count"])
# the fused shard stages
hx = torch.from_numpy(h).cuda()
gid = torch.arange(h.shape[0], dtype=torch.int64, device="cuda")
codes = eng.morton(hx, hx.min(0).values, hx.max(0).values)
spl = torch.sort(codes[torch.randint(0, h.shape[0], (3,), device="cuda")]).values
rows, counts = eng.route(hx, gid, codes, spl)
ux, ug, uc = eng.unpack(rows, 3, True)
bx = eng.region_boxes(ux, uc)
own = torch.zeros(bx.shape[0], dtype=torch.int32, device="cuda") + 3
pm = eng.near_peers(hx, 0.05, bx[:, :3], bx[:, 3:], own)
torch.cuda.synchronize()
print("shard", counts, int(bx.shape[0]), int((pm != 0).sum()))
# device generators and the device checker
gz = tb.generate_device("hacc_like", 5000)
gt = tb.generate_device("taxi_like", 5000)
a = tb.cluster(hd, 0.042, 5, tb.Algorithm.FDBSCAN)
b = tb.cluster(hd, 0.042, 5, tb.Algorithm.DENSEBOX)
chk = tb.api.check_equivalence_device(hx, 0.042, *(torch.from_numpy(np.ascontiguousarray(v)).cuda()
                                       for v in (a.labels, a.core_flags, b.labels, b.core_flags)))
print("check", chk[0], int(gz.shape[0]), int(gt.shape[0]))
PY
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python /tmp/san_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log
done
