"""Randomized stress against the C oracle (test infrastructure / developer
tool): random clouds (blobs / uniform / duplicates / lattice-like), eps from
far below the spacing to beyond the extent, minpts 2..64, 2D/3D, FDBSCAN /
DenseBox / brute force, through tc_cluster and the device entry.

  python tools/stress.py [seconds]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2103_05162_b200 as tb  # noqa: E402
from oracle import oracle  # noqa: E402


def cloud(rng):
    d = int(rng.choice([2, 3]))
    n = int(rng.integers(1, 6000))
    kind = str(rng.choice(["blobs", "uniform", "dups", "lattice"]))
    if kind == "blobs":
        k = int(rng.integers(1, 8))
        c = rng.normal(0, 1, (k, d)) * 5
        pts = c[rng.integers(0, k, n)] + rng.normal(0, rng.uniform(0.05, 1), (n, d))
    elif kind == "uniform":
        pts = rng.uniform(-1, 1, (n, d)) * rng.uniform(0.1, 100)
    elif kind == "dups":  # ~50 copies per point, or ~1000 (Morton groups > 256: fallback sort)
        base = rng.uniform(-1, 1, (max(1, n // int(rng.choice([50, 1000]))), d))
        pts = base[rng.integers(0, len(base), n)]
    else:
        s = int(round(n ** (1 / d))) + 1
        g = np.stack(np.meshgrid(*[np.arange(s)] * d), -1).reshape(-1, d)[:n]
        pts = g * 0.1 + rng.uniform(-1e-3, 1e-3, g.shape)
    return kind, pts.astype(np.float32)


def one(rng):
    """One random case: (description, ok)."""
    kind, pts = cloud(rng)
    n, d = pts.shape
    ext = float(np.max(pts.max(0) - pts.min(0))) if n > 1 else 1.0
    eps = float(np.float32(max(ext, 1e-3) * 10 ** rng.uniform(-4, 0.5)))
    minpts = int(rng.choice([2, 2, 3, 5, 10, 64]))
    algo = int(rng.choice([0, 1, 1, 2])) if n <= 3000 else int(rng.choice([0, 1]))
    desc = f"{kind} n={n} d={d} eps={eps:.4g} minpts={minpts} algo={algo}"
    want = oracle.dbscan(pts, eps, minpts, algo)
    got = tb.cluster(tb.Dataset.from_array(pts), eps, minpts, tb.Algorithm(algo))
    _, core, _ = tb.cluster_device(torch.from_numpy(pts).cuda(), eps, minpts, tb.Algorithm(algo),
                                   stats=True)
    if algo == 0:  # the stream-ordered entry too (device status word)
        alab, acore, ast = tb.cluster_device_async(torch.from_numpy(pts).cuda(), eps, minpts)
        torch.cuda.synchronize()
        wcm = want["core"] == 1
        alab = alab.cpu().numpy()
        if (int(ast.item()) != 0 or not np.array_equal(acore.cpu().numpy(), want["core"])
                or not np.array_equal(alab[wcm], want["labels"][wcm])
                or not np.array_equal(alab == -1, want["labels"] == -1)):
            return desc + " (async)", False
    torch.cuda.synchronize()
    cm = want["core"] == 1
    ok = (np.array_equal(got.core_flags, want["core"])
          and np.array_equal(got.labels == -1, want["labels"] == -1)
          and np.array_equal(got.labels[cm], want["labels"][cm])
          and np.array_equal(core.cpu().numpy(), want["core"])
          and (algo == 2 or got.stats["pair_resolutions"] == want["stats"]["pair_resolutions"]))
    if ok:
        ok, _ = oracle.check_equivalence(pts, eps, got.labels, got.core_flags, want["labels"],
                                         want["core"])
    return desc, ok


def run(budget_s, max_runs=None, seed=12345, verbose=True):
    rng = np.random.default_rng(seed)
    t0 = time.time()
    runs, bad = 0, []
    while time.time() - t0 < budget_s and (max_runs is None or runs < max_runs):
        desc, ok = one(rng)
        runs += 1
        if not ok:
            bad.append(desc)
            if verbose:
                print("BAD", desc, flush=True)
    if verbose:
        print(f"runs {runs} bad {len(bad)}", flush=True)
    return runs, bad


if __name__ == "__main__":
    run(float(sys.argv[1]) if len(sys.argv) > 1 else 120.0,
        seed=int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
