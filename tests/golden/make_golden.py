"""Generates the golden fixtures in tests/golden/ by RUNNING THE REFERENCE.

Source of truth: oracle/_ref/libtreeclust_ref.so = /root/reference/proj
compiled unmodified (oracle/Makefile) + oracle/ref_shim.cpp. Run here (where
/root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed):
  generators.json  sha256 of the reference generators' coordinates
                   (tc_generate_blobs/uniform/lattice, testutil::random_instance)
  morton.npz       random points + bounds -> reference morton_encode codes
  bvh.npz          point sets -> reference Bvh accessors (leaf ids, left,
                   right, max_rank, boxes)
  grid.npz         build_grid perm / cell ids / ranges / dense flags
  dbscan.npz       random_instance seeds 1..24 -> dbscan_run (threads = 1)
                   labels, core flags and RunStats counters for FDBSCAN,
                   DenseBox and dbscan_bruteforce
"""
import ctypes as C
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

SEEDS = list(range(1, 25))
MIN_N, MAX_N = 50, 1500


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def ref_dataset(fn, *args):
    L = ref.lib()
    out = C.c_void_p()
    getattr(L, fn).restype = C.c_int
    st = getattr(L, fn)(*args, C.byref(out))
    assert st == 0, (fn, st)
    L.tc_dataset_size.restype = C.c_int64
    L.tc_dataset_size.argtypes = [C.c_void_p]
    L.tc_dataset_dim.argtypes = [C.c_void_p]
    L.tc_dataset_coords.restype = C.POINTER(C.c_float)
    L.tc_dataset_coords.argtypes = [C.c_void_p]
    n, d = L.tc_dataset_size(out), L.tc_dataset_dim(out)
    arr = np.ctypeslib.as_array(L.tc_dataset_coords(out), shape=(n, d)).copy()
    L.tc_dataset_free.argtypes = [C.c_void_p]
    L.tc_dataset_free(out)
    return arr


def main():
    gens = {}
    f = C.c_float
    gens["blobs(3,80,2,20,0.5,21)"] = sha(ref_dataset(
        "tc_generate_blobs", C.c_int(3), C.c_int64(80), C.c_int(2), f(20.0), f(0.5), C.c_uint64(21)))
    gens["blobs(3,40,3,6,0.4,11)"] = sha(ref_dataset(
        "tc_generate_blobs", C.c_int(3), C.c_int64(40), C.c_int(3), f(6.0), f(0.4), C.c_uint64(11)))
    gens["blobs(100,10000,2,0.8333333,0.08333333,7)"] = sha(ref_dataset(
        "tc_generate_blobs", C.c_int(100), C.c_int64(10000), C.c_int(2), f(0.8333333),
        f(0.08333333), C.c_uint64(7)))
    lo = (C.c_float * 3)(0.0, -1.0, 2.0)
    hi = (C.c_float * 3)(1.0, 1.0, 5.0)
    gens["uniform(1000,3,[0,-1,2],[1,1,5],3)"] = sha(ref_dataset(
        "tc_generate_uniform", C.c_int64(1000), C.c_int(3), lo, hi, C.c_uint64(3)))
    gens["lattice(40,2,0.1)"] = sha(ref_dataset("tc_generate_lattice", C.c_int64(40), C.c_int(2),
                                                f(0.1)))
    gens["lattice(12,3,0.1)"] = sha(ref_dataset("tc_generate_lattice", C.c_int64(12), C.c_int(3),
                                                f(0.1)))
    for s in SEEDS:
        c, eps, mp = ref.random_instance(s, MIN_N, MAX_N)
        gens[f"random_instance({s},{MIN_N},{MAX_N})"] = {"sha256": sha(c), "n": len(c),
                                                         "dim": int(c.shape[1]), "eps": eps,
                                                         "minpts": mp}
    with open(os.path.join(HERE, "generators.json"), "w") as fh:
        json.dump(gens, fh, indent=1, sort_keys=True)

    rng = np.random.default_rng(2024)
    mort = {}
    for d in (2, 3):
        pts = rng.uniform(-3, 7, (500, d)).astype(np.float32)
        lo_b = np.array([-2.0, 0.0, 1.0][:d], np.float32)
        hi_b = np.array([3.0, 10.0, 4.0][:d], np.float32)
        mort[f"pts{d}"] = pts
        mort[f"lo{d}"] = lo_b
        mort[f"hi{d}"] = hi_b
        mort[f"codes{d}"] = ref.morton_codes(pts, lo_b, hi_b)
    np.savez_compressed(os.path.join(HERE, "morton.npz"), **mort)

    bv = {}
    sets = {
        "two": np.array([[0, 0], [3, 1]], np.float32),
        "dups": np.array([[1, 1], [1, 1], [1, 1], [2, 2]], np.float32),
        "rand2": rng.uniform(0, 10, (777, 2)).astype(np.float32),
        "rand3": rng.uniform(0, 10, (1000, 3)).astype(np.float32),
        "clump3": np.concatenate([rng.normal(0, 1e-4, (300, 3)), rng.normal(5, 1, (200, 3)),
                                  np.zeros((20, 3))]).astype(np.float32),
    }
    for name, pts in sets.items():
        t = ref.point_bvh(pts)
        bv[f"{name}_pts"] = pts
        for k, v in t.items():
            bv[f"{name}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "bvh.npz"), **bv)

    gr = {}
    for s in (3, 8):
        c, eps, mp = ref.random_instance(s, MIN_N, MAX_N)
        g = ref.build_grid(c, eps, mp)
        for k, v in g.items():
            gr[f"s{s}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "grid.npz"), **gr)

    db = {}
    for s in SEEDS:
        c, eps, mp = ref.random_instance(s, MIN_N, MAX_N)
        for algo in (0, 1, 2):
            r = ref.dbscan(c, eps, mp, algo, threads=1)
            db[f"s{s}_a{algo}_labels"] = r["labels"]
            db[f"s{s}_a{algo}_core"] = r["core"]
            st = r["stats"]
            db[f"s{s}_a{algo}_counters"] = np.array(
                [st["preprocess_skipped"], st["pair_resolutions"], st["distance_evaluations"],
                 st["cluster_count"], st["core_count"], st["noise_count"]], np.int64)
            db[f"s{s}_a{algo}_dense_fraction"] = np.float64(st["dense_point_fraction"])
    np.savez_compressed(os.path.join(HERE, "dbscan.npz"), **db)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
