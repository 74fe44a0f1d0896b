#!/usr/bin/env python3
"""CPU baseline plan of BASELINE.md §3: the unmodified reference (oracle/_ref)
through its own C ABI (inputs written as .bin by the oracle's generators and
loaded with the reference's tc_dataset_load), per config at threads=0 (all host
cores) and threads=1, with the host's CPU model; per-phase seconds from
tc_cluster_stats. One JSON line per run on stdout.

  python tools/ref_baseline.py [--configs C1,C2,C3,C4] [--threads 0,1] [--reps 3]
"""
import argparse
import json
import os
import shutil
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle, ref  # noqa: E402

CONFIGS = {
    # name: (generator, eps, minpts, algo)
    "C1": (lambda: None, 0.01, 5, 0),
    "C2": (lambda: oracle.hacc_like(37_000_000), 0.042, 2, 0),
    "C2db": (lambda: oracle.hacc_like(37_000_000), 0.042, 2, 1),
    "C3": (lambda: oracle.hacc_like(37_000_000), 0.042, 100, 1),
    "C3fd": (lambda: oracle.hacc_like(37_000_000), 0.042, 100, 0),
    "C4": (lambda: oracle.taxi_like(80_000_000), 0.001, 1000, 1),
}


def load(name, tmp):
    if name == "C1":  # reference generator, acceptance crit. 9 rescaled
        import ctypes as C
        L = ref._capi()
        L.tc_generate_blobs.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_float, C.c_float,
                                        C.c_uint64, C.POINTER(C.c_void_p)]
        h = C.c_void_p()
        assert L.tc_generate_blobs(100, 10000, 2, C.c_float(0.8333333), C.c_float(0.08333333),
                                   7, C.byref(h)) == 0
        return ref.RefDataset(h)
    path = os.path.join(tmp, f"{name}.bin")
    oracle.write_bin(path, CONFIGS[name][0]())
    ds = ref.RefDataset.load(path)
    os.remove(path)
    return ds


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2,C3")
    ap.add_argument("--threads", default="0,1")
    ap.add_argument("--reps", type=int, default=1)
    args = ap.parse_args()
    tmp = tempfile.mkdtemp(prefix="tcb_refbase_")
    model = ref.host_cpu_model()
    try:
        for name in args.configs.split(","):
            _, eps, minpts, algo = CONFIGS[name]
            ds = load(name, tmp)
            for th in (int(t) for t in args.threads.split(",")):
                reps = args.reps if name == "C1" else 1
                best = None
                for _ in range(reps):
                    dt, st, _, _ = ds.cluster(eps, minpts, algo, th)
                    if best is None or dt < best[0]:
                        best = (dt, st)
                dt, st = best
                print(json.dumps({
                    "config": name, "n": ds.size, "eps": eps, "minpts": minpts,
                    "algo": ["FDBSCAN", "DenseBox"][algo], "threads": th,
                    "threads_used": os.cpu_count() if th == 0 else th, "cpu_model": model,
                    "wall_s": round(dt, 3), "mpts_s": round(ds.size / dt / 1e6, 4),
                    "reps": reps, "stats": st}), flush=True)
            ds.close()
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


if __name__ == "__main__":
    main()
