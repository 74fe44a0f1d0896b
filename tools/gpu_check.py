"""Quick GPU parity + timing probe (developer tool; tests/ hold the real gates)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2103_05162_b200 as tb  # noqa: E402
from oracle import ref  # noqa: E402


def compare(coords, eps, minpts, algo, tag):
    ds = tb.Dataset.from_array(coords)
    g = tb.cluster(ds, eps, minpts, tb.Algorithm(algo))
    r = ref.dbscan(coords, eps, minpts, algo, threads=1)
    ok = True
    msgs = []
    if not np.array_equal(g.core_flags, r["core"]):
        ok = False
        msgs.append("core flags differ (%d)" % int((g.core_flags != r["core"]).sum()))
    if not np.array_equal(g.labels == -1, r["labels"] == -1):
        ok = False
        msgs.append("noise differs")
    cm = r["core"] == 1
    if not np.array_equal(g.labels[cm], r["labels"][cm]):
        ok = False
        msgs.append("core labels differ (%d)" % int((g.labels[cm] != r["labels"][cm]).sum()))
    eq, m = ref.check_equivalence(coords, eps, minpts, g.labels, g.core_flags, r["labels"], r["core"])
    if not eq:
        ok = False
        msgs.append("equivalence: " + m)
    for key in ("pair_resolutions", "distance_evaluations", "cluster_count", "core_count",
                "noise_count", "preprocess_skipped"):
        if algo == 2 and key in ("pair_resolutions", "distance_evaluations"):
            continue
        if g.stats[key] != r["stats"][key]:
            ok = False
            msgs.append("%s %s vs ref %s" % (key, g.stats[key], r["stats"][key]))
    if algo == 1 and abs(g.stats["dense_point_fraction"] - r["stats"]["dense_point_fraction"]) > 0:
        ok = False
        msgs.append("dense fraction %r vs %r" % (g.stats["dense_point_fraction"],
                                                 r["stats"]["dense_point_fraction"]))
    print(("OK  " if ok else "BAD ") + tag, "; ".join(msgs), flush=True)
    return ok


def main():
    bad = 0
    for seed in list(range(1, 41)):
        c, eps, mp = ref.random_instance(seed, 50, 2000)
        for algo in (0, 1, 2):
            bad += not compare(c, eps, mp, algo, f"seed={seed} n={len(c)} d={c.shape[1]} eps={eps:.3f} minpts={mp} algo={algo}")
    # C1-like 1M blobs
    ds = tb.Dataset.blobs(100, 10000, 2, 0.8333333, 0.08333333, 7)
    c = ds.coords()
    for algo in (0, 1):
        t = time.time()
        bad += not compare(c, 0.01, 5, algo, f"C1 algo={algo}")
        print("  took %.1fs" % (time.time() - t))
    print("FAILURES:", bad)

    import torch
    for n, algo, mp in ((37_000_000, 0, 2), (37_000_000, 1, 2), (37_000_000, 1, 100), (37_000_000, 0, 100)):
        h = tb.Dataset.hacc_like(n)
        x = torch.from_numpy(h.coords()).cuda()
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            lab, core, st = tb.cluster_device(x, 0.042, mp, tb.Algorithm(algo), stats=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
        print(f"n={n} algo={algo} minpts={mp}: {dt*1e3:.1f} ms wall; stages {tb.last_stage_ms()}; stats {st}", flush=True)


if __name__ == "__main__":
    main()
