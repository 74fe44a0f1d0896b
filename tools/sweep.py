"""Parameter sweeps through the C ABI — the GPU counterpart of the reference's
`treeclust bench` (REF tools/treeclust_cli.cpp:146-198): same CSV columns,
one `tc_cluster` call per (n, eps, minpts, algorithm), phase seconds from
`tc_cluster_stats`. Adds the device-resident time of the same call
(`tcg_cluster_device`, best of --reps) and Mpoints/s.

  python tools/sweep.py --input points.bin --eps-list 0.042 --minpts-list 2,5,100
  python tools/sweep.py --gen hacc:37000000 --eps-list 0.042 --minpts-list 2,5,10,50,100 \
      --algos fdbscan,densebox --out profiles/sweep.csv

--gen takes hacc:N, taxi:N or blobs:K:PER:DIM; --n-list takes prefixes of
the input (like the reference's --n-list).
"""
import argparse
import csv
import io
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_05162_b200 as tb  # noqa: E402

ALGOS = {"fdbscan": tb.Algorithm.FDBSCAN, "densebox": tb.Algorithm.DENSEBOX,
         "bruteforce": tb.Algorithm.BRUTEFORCE}
COLUMNS = ["algorithm", "n", "eps", "minpts", "build_s", "preprocess_s", "main_s", "finalize_s",
           "total_s", "clusters", "cores", "noise", "dense_fraction",
           # additions
           "device_ms", "mpts_per_s", "pair_resolutions", "distance_evaluations"]


def load(args):
    if args.input:
        return tb.Dataset.load(args.input)
    kind, *rest = args.gen.split(":")
    if kind == "hacc":
        return tb.Dataset.hacc_like(int(rest[0]))
    if kind == "taxi":
        return tb.Dataset.taxi_like(int(rest[0]))
    if kind == "blobs":
        k, per, dim = (int(v) for v in rest)
        return tb.Dataset.blobs(k, per, dim, 0.8333333, 0.08333333, 7)
    raise SystemExit(f"unknown --gen {args.gen}")


def device_ms(x, eps, minpts, algo, reps):
    import torch

    best = float("inf")
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tb.cluster_device(x, eps, minpts, algo)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    ap = argparse.ArgumentParser()
    src = ap.add_mutually_exclusive_group(required=True)
    src.add_argument("--input")
    src.add_argument("--gen")
    ap.add_argument("--out")
    ap.add_argument("--algos", default="fdbscan,densebox")
    ap.add_argument("--eps-list", required=True)
    ap.add_argument("--minpts-list", required=True)
    ap.add_argument("--n-list", default="")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()

    import torch

    full = load(args)
    coords = full.coords()
    n_list = [int(v) for v in args.n_list.split(",") if v] or [coords.shape[0]]
    rows = []
    for n in n_list:
        sub = coords[:n]
        ds = tb.Dataset.from_array(sub) if n < coords.shape[0] else full
        x = torch.from_numpy(np.ascontiguousarray(sub)).cuda()
        for eps in (float(v) for v in args.eps_list.split(",")):
            for minpts in (int(v) for v in args.minpts_list.split(",")):
                for name in args.algos.split(","):
                    algo = ALGOS[name]
                    res = tb.cluster(ds, eps, minpts, algo)
                    s = res.stats
                    total = s["build_seconds"] + s["preprocess_seconds"] + s["main_seconds"] + \
                        s["finalize_seconds"]
                    dms = device_ms(x, eps, minpts, algo, args.reps)
                    rows.append([name, n, eps, minpts, s["build_seconds"], s["preprocess_seconds"],
                                 s["main_seconds"], s["finalize_seconds"], total,
                                 s["cluster_count"], s["core_count"], s["noise_count"],
                                 s["dense_point_fraction"], round(dms, 3),
                                 round(n / dms / 1e3, 2), s["pair_resolutions"],
                                 s["distance_evaluations"]])
                    print(",".join(str(v) for v in rows[-1]), file=sys.stderr, flush=True)
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(COLUMNS)
    w.writerows(rows)
    if args.out:
        with open(args.out, "w") as f:
            f.write(buf.getvalue())
    else:
        sys.stdout.write(buf.getvalue())


if __name__ == "__main__":
    t0 = time.time()
    main()
    print(f"sweep done in {time.time() - t0:.1f} s", file=sys.stderr)
