"""Times every BASELINE config on the device (tcg_cluster_device, points resident
in HBM) and cross-checks FDBSCAN against DenseBox on the same points (core
flags, noise and core labels must agree exactly). Developer tool; the bench
contract lives in bench.py.

  python tools/configs.py [C1 C2 C3 C4 ...]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2103_05162_b200 as tb  # noqa: E402

# inputs from the device generators (byte-identical to the host ones)
CONFIGS = {
    "C1": dict(gen=lambda: tb.generate_device("blobs", 100, 10000, 2, 0.8333333, 0.08333333, 7),
               eps=0.01, minpts=5, algo=tb.Algorithm.FDBSCAN),
    "C2": dict(gen=lambda: tb.generate_device("hacc_like", 37_000_000), eps=0.042, minpts=2,
               algo=tb.Algorithm.FDBSCAN),
    "C2db": dict(gen=lambda: tb.generate_device("hacc_like", 37_000_000), eps=0.042, minpts=2,
                 algo=tb.Algorithm.DENSEBOX),
    "C3": dict(gen=lambda: tb.generate_device("hacc_like", 37_000_000), eps=0.042, minpts=100,
               algo=tb.Algorithm.DENSEBOX),
    "C3fd": dict(gen=lambda: tb.generate_device("hacc_like", 37_000_000), eps=0.042, minpts=100,
                 algo=tb.Algorithm.FDBSCAN),
    "C5": dict(gen=lambda: tb.generate_device("hacc_like", 497_000_000,
                                              36.8 * (497 / 37) ** (1 / 3)),
               eps=0.042, minpts=2, algo=tb.Algorithm.FDBSCAN),
    "C4": dict(gen=lambda: tb.generate_device("taxi_like", 80_000_000), eps=0.001, minpts=1000,
               algo=tb.Algorithm.DENSEBOX),
    "C4fd": dict(gen=lambda: tb.generate_device("taxi_like", 80_000_000), eps=0.001, minpts=1000,
                 algo=tb.Algorithm.FDBSCAN),
}


def run(name, reps=3, check=True):
    cfg = CONFIGS[name]
    if name == "C5":  # keep C5's ~80 GB of scratch between the repetitions
        tb.set_pool_release_threshold(160 << 30)
    t0 = time.time()
    x = cfg["gen"]()
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    ms = []
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        lab, core, st = tb.cluster_device(x, cfg["eps"], cfg["minpts"], cfg["algo"], stats=True)
        ev1.record()
        torch.cuda.synchronize()
        ms.append(ev0.elapsed_time(ev1))
    stages = tb.last_stage_ms()
    out = {"config": name, "n": int(x.shape[0]), "algo": cfg["algo"].name, "minpts": cfg["minpts"],
           "ms_best": round(min(ms[1:]), 3), "mpts_s": round(x.shape[0] / min(ms[1:]) / 1e3, 2),
           "stage_ms": {k: round(v, 3) for k, v in stages.items()},
           "stats": {k: st[k] for k in ("pair_resolutions", "distance_evaluations", "cluster_count",
                                        "core_count", "noise_count", "dense_point_fraction")},
           "gen_s": round(gen_s, 1)}
    if check:
        other = tb.Algorithm.FDBSCAN if cfg["algo"] == tb.Algorithm.DENSEBOX else tb.Algorithm.DENSEBOX
        lab2, core2, _ = tb.cluster_device(x, cfg["eps"], cfg["minpts"], other, stats=True)
        m = core.bool()
        out["cross_check"] = bool(torch.equal(core, core2) and torch.equal(lab == -1, lab2 == -1)
                                  and torch.equal(lab[m], lab2[m]))
    print(json.dumps(out), flush=True)
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or ["C1", "C2", "C2db", "C3", "C3fd", "C4", "C4fd"]  # C5: 497M, on request
    for n in names:
        run(n, check=not n.endswith(("fd", "db")))
