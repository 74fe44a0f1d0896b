"""TEST INFRASTRUCTURE ONLY — ctypes access to the C restatement (tc_oracle.c).

The checker of the parity tests, ``__graft_entry__.smoke()`` and bench.py's
cpu_baseline leg; never the thing measured or shipped. Pinned against the
reference's golden vectors and against the compiled reference itself in
tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise FileNotFoundError(f"{LIB} not built (make -C oracle liboracle.so)")
        L = C.CDLL(LIB)
        f32p = C.POINTER(C.c_float)
        i32p = C.POINTER(C.c_int32)
        u8p = C.POINTER(C.c_uint8)
        u64p = C.POINTER(C.c_uint64)
        i64p = C.POINTER(C.c_int64)
        L.oracle_morton_codes.argtypes = [f32p, C.c_int64, C.c_int, f32p, f32p, u64p]
        L.oracle_morton_codes.restype = None
        L.oracle_point_bvh.argtypes = [f32p, C.c_int64, C.c_int, i32p, i32p, i32p, i32p, f32p]
        L.oracle_build_grid.restype = C.c_int64
        L.oracle_build_grid.argtypes = [f32p, C.c_int64, C.c_int, C.c_float, C.c_int, i32p, i32p,
                                        u64p, i32p, i32p, u8p, C.c_int64]
        L.oracle_dbscan.argtypes = [f32p, C.c_int64, C.c_int, C.c_float, C.c_int, C.c_int, i32p,
                                    u8p, i64p]
        L.oracle_check_equivalence.argtypes = [f32p, C.c_int64, C.c_int, C.c_float, i32p, u8p,
                                               i32p, u8p, C.c_char_p, C.c_int64]
        L.oracle_gen_hacc_like.argtypes = [C.c_int64, C.c_double, C.c_double, C.c_uint64, f32p]
        L.oracle_gen_taxi_like.argtypes = [C.c_int64, C.c_uint64, f32p]
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def morton_codes(coords, lo, hi) -> np.ndarray:
    a = np.ascontiguousarray(coords, np.float32)
    lo = np.ascontiguousarray(lo, np.float32).reshape(-1)
    hi = np.ascontiguousarray(hi, np.float32).reshape(-1)
    out = np.empty(a.shape[0], np.uint64)
    lib().oracle_morton_codes(_p(a, C.c_float), a.shape[0], a.shape[1], _p(lo, C.c_float),
                              _p(hi, C.c_float), _p(out, C.c_uint64))
    return out


def point_bvh(coords) -> dict:
    a = np.ascontiguousarray(coords, np.float32)
    n, d = a.shape
    m = max(n - 1, 1)
    leaf = np.empty(n, np.int32)
    left, right, mr = (np.zeros(m, np.int32) for _ in range(3))
    boxes = np.zeros((m, 6), np.float32)
    assert lib().oracle_point_bvh(_p(a, C.c_float), n, d, _p(leaf, C.c_int32),
                                  _p(left, C.c_int32), _p(right, C.c_int32), _p(mr, C.c_int32),
                                  _p(boxes, C.c_float)) == 0
    k = n - 1
    return {"leaf_ids": leaf, "left": left[:k], "right": right[:k], "max_rank": mr[:k],
            "boxes": boxes[:k]}


def build_grid(coords, eps, minpts) -> dict:
    a = np.ascontiguousarray(coords, np.float32)
    n, d = a.shape
    perm, cop, cb, ce = (np.empty(n, np.int32) for _ in range(4))
    cid = np.empty(n, np.uint64)
    cd = np.empty(n, np.uint8)
    m = lib().oracle_build_grid(_p(a, C.c_float), n, d, C.c_float(eps), int(minpts),
                                _p(perm, C.c_int32), _p(cop, C.c_int32), _p(cid, C.c_uint64),
                                _p(cb, C.c_int32), _p(ce, C.c_int32), _p(cd, C.c_uint8), n)
    if m < 0:
        raise ValueError("build_grid: cell id overflow")
    return {"perm": perm, "cell_of_point": cop, "cell_id": cid[:m], "begin": cb[:m],
            "end": ce[:m], "dense": cd[:m].astype(bool)}


COUNTERS = ("preprocess_skipped", "pair_resolutions", "distance_evaluations", "cluster_count",
            "core_count", "noise_count", "dense_point_count")


def dbscan(coords, eps, minpts, algo: int) -> dict:
    """algo 0 FDBSCAN, 1 DenseBox, 2 brute force; single-threaded, deterministic."""
    a = np.ascontiguousarray(coords, np.float32)
    n, d = a.shape
    labels = np.empty(n, np.int32)
    core = np.empty(n, np.uint8)
    ctr = np.zeros(7, np.int64)
    rc = lib().oracle_dbscan(_p(a, C.c_float), n, d, C.c_float(eps), int(minpts), int(algo),
                             _p(labels, C.c_int32), _p(core, C.c_uint8), _p(ctr, C.c_int64))
    if rc != 0:
        raise ValueError("invalid argument")
    stats = dict(zip(COUNTERS, (int(v) for v in ctr)))
    stats["dense_point_fraction"] = stats["dense_point_count"] / n if algo == 1 else 0.0
    return {"labels": labels, "core": core, "stats": stats}


def check_equivalence(coords, eps, la, ca, lb, cb):
    a = np.ascontiguousarray(coords, np.float32)
    n, d = a.shape
    la, lb = (np.ascontiguousarray(v, np.int32) for v in (la, lb))
    ca, cb = (np.ascontiguousarray(v, np.uint8) for v in (ca, cb))
    msg = C.create_string_buffer(256)
    ok = lib().oracle_check_equivalence(_p(a, C.c_float), n, d, C.c_float(eps),
                                        _p(la, C.c_int32), _p(ca, C.c_uint8), _p(lb, C.c_int32),
                                        _p(cb, C.c_uint8), msg, len(msg))
    return bool(ok), msg.value.decode()


def hacc_like(n: int, box_len=None, halo_frac=0.23, seed=11) -> np.ndarray:
    """SURVEY §8d HACC-like halos (C2/C3/C5 inputs); box_len defaults to the
    C2 density, 36.8 * (n / 37e6)^(1/3)."""
    if box_len is None:
        box_len = 36.8 * (n / 37e6) ** (1.0 / 3.0)
    out = np.empty((n, 3), np.float32)
    if lib().oracle_gen_hacc_like(n, float(box_len), float(halo_frac), seed,
                                  _p(out, C.c_float)) != 0:
        raise ValueError("invalid argument")
    return out


def taxi_like(n: int, seed=5) -> np.ndarray:
    """SURVEY §8d taxi-like 2D road points (C4 input)."""
    out = np.empty((n, 2), np.float32)
    if lib().oracle_gen_taxi_like(n, seed, _p(out, C.c_float)) != 0:
        raise ValueError("invalid argument")
    return out


def write_bin(path: str, coords) -> None:
    """The reference's binary point format (REF io.cpp:124-134): u32 n, u32 dim,
    n*dim little-endian f32."""
    a = np.ascontiguousarray(coords, np.float32)
    with open(path, "wb") as f:
        f.write(np.array(a.shape, dtype="<u4").tobytes())
        f.write(a.astype("<f4", copy=False).tobytes())
