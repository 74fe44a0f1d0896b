"""Randomized stress on larger clouds (20K-150K points, blobs / heavy
duplicates, 2D/3D, minpts 2..100, FDBSCAN and DenseBox) against the oracle,
counters included (developer tool; 5 minutes: 972 cases, 0 differences).

  python tools/stress_big.py
"""
import sys, time
import numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tools")
from oracle import oracle
import paper_2103_05162_b200 as tb
import torch
rng = np.random.default_rng(99)
t0 = time.time(); runs = bad = 0
while time.time() - t0 < 300:
    d = int(rng.choice([2, 3])); n = int(rng.integers(20000, 150000))
    kind = rng.choice(["blobs", "dups"])
    if kind == "blobs":
        k = int(rng.integers(1, 20)); c = rng.normal(0, 1, (k, d)) * 5
        pts = c[rng.integers(0, k, n)] + rng.normal(0, rng.uniform(0.05, 1), (n, d))
    else:
        base = rng.uniform(-1, 1, (max(1, n // 100), d)); pts = base[rng.integers(0, len(base), n)]
    pts = pts.astype(np.float32)
    ext = float(np.max(pts.max(0) - pts.min(0)))
    eps = float(np.float32(ext * 10 ** rng.uniform(-4, -1.3)))
    minpts = int(rng.choice([2, 5, 20, 100]))
    algo = int(rng.choice([0, 1]))
    want = oracle.dbscan(pts, eps, minpts, algo)
    got = tb.cluster(tb.Dataset.from_array(pts), eps, minpts, tb.Algorithm(algo))
    cm = want["core"] == 1
    ok = (np.array_equal(got.core_flags, want["core"]) and np.array_equal(got.labels == -1, want["labels"] == -1)
          and np.array_equal(got.labels[cm], want["labels"][cm]) and got.stats["pair_resolutions"] == want["stats"]["pair_resolutions"]
          and got.stats["distance_evaluations"] == want["stats"]["distance_evaluations"])
    runs += 1
    if not ok:
        bad += 1; print("BAD", kind, n, d, eps, minpts, algo, flush=True)
print("runs", runs, "bad", bad)
