"""Randomized stress of tcg_cluster_multi (the sharded path behind the C ABI)
against tc_cluster on the same points, 1-6 shards on the box's device(s)
(developer tool). python tools/stress_multi.py [seconds]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
import paper_2103_05162_b200 as tb  # noqa: E402
from stress import cloud  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(777)
t0 = time.time()
runs = bad = 0
while time.time() - t0 < budget:
    kind, pts = cloud(rng)
    n = len(pts)
    ext = float(np.max(pts.max(0) - pts.min(0))) if n > 1 else 1.0
    eps = float(np.float32(max(ext, 1e-3) * 10 ** rng.uniform(-4, 0.3)))
    minpts = int(rng.choice([2, 3, 5, 20]))
    algo = tb.Algorithm(int(rng.choice([0, 1])))
    shards = int(rng.integers(1, 7))
    ds = tb.Dataset.from_array(pts)
    want = tb.cluster(ds, eps, minpts, algo)
    try:
        got = tb.cluster_multi(ds, eps, minpts, [0] * shards, algo)
    except Exception as e:  # noqa: BLE001
        print("EXC", kind, n, eps, minpts, int(algo), shards, repr(e), flush=True)
        bad += 1
        break
    cm = want.core_flags == 1
    ok = (np.array_equal(got.core_flags, want.core_flags)
          and np.array_equal(got.labels == -1, want.labels == -1)
          and np.array_equal(got.labels[cm], want.labels[cm]))
    runs += 1
    if not ok:
        bad += 1
        print("BAD", kind, n, pts.shape[1], eps, minpts, int(algo), shards, flush=True)
print(f"runs {runs} bad {bad}", flush=True)
