"""TEST INFRASTRUCTURE ONLY — ctypes access to the UNMODIFIED reference.

``oracle/_ref/libtreeclust_ref.so`` is the reference treeclust compiled from
its own sources under /root/reference/proj (recipe: ``oracle/Makefile``) plus
``oracle/ref_shim.cpp``, which exposes the reference's internal C++ building
blocks (Morton codes, BVH accessors, build_grid, dbscan_run + RunStats,
check_equivalence, random_instance). It also exports the reference's own
``tc_*`` ABI. Only tests/, ``__graft_entry__.smoke()`` and bench.py's
reference / cpu_baseline legs may load it, and only as the checker or the
CPU baseline — never as the thing measured or shipped.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libtreeclust_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{REF_LIB} not built (make -C oracle ref)")
        L = C.CDLL(REF_LIB)
        f32p = C.POINTER(C.c_float)
        i32p = C.POINTER(C.c_int32)
        u8p = C.POINTER(C.c_uint8)
        u64p = C.POINTER(C.c_uint64)
        L.ref_morton_codes.argtypes = [f32p, C.c_int64, C.c_int, f32p, f32p, u64p]
        L.ref_point_bvh.argtypes = [f32p, C.c_int64, C.c_int, i32p, i32p, i32p, i32p, f32p]
        L.ref_build_grid.restype = C.c_int64
        L.ref_build_grid.argtypes = [f32p, C.c_int64, C.c_int, C.c_float, C.c_int, i32p, i32p,
                                     u64p, i32p, i32p, u8p, C.c_int64]
        L.ref_mixed_bvh.restype = C.c_int64
        L.ref_mixed_bvh.argtypes = [f32p, C.c_int64, C.c_int, C.c_float, C.c_int, u8p, i32p,
                                    i32p, i32p, i32p, f32p, C.c_int64]
        L.ref_dbscan.argtypes = [f32p, C.c_int64, C.c_int, C.c_float, C.c_int, C.c_int, C.c_int,
                                 i32p, u8p, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
        L.ref_check_equivalence.argtypes = [f32p, C.c_int64, C.c_int, C.c_float, C.c_int, i32p,
                                            u8p, i32p, u8p, C.c_char_p, C.c_int64]
        L.ref_random_instance.restype = C.c_int64
        L.ref_random_instance.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_int),
                                          C.POINTER(C.c_float), C.POINTER(C.c_int), f32p]
        _lib = L
    return _lib


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(C.POINTER(C.c_float))


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def morton_codes(coords, lo, hi) -> np.ndarray:
    a, p = _f32(coords)
    n, d = a.shape
    lo_a, plo = _f32(np.asarray(lo, dtype=np.float32).reshape(-1))
    hi_a, phi = _f32(np.asarray(hi, dtype=np.float32).reshape(-1))
    out = np.empty(n, dtype=np.uint64)
    lib().ref_morton_codes(p, n, d, plo, phi, _ptr(out, C.c_uint64))
    return out


def point_bvh(coords) -> dict:
    a, p = _f32(coords)
    n, d = a.shape
    m = max(n - 1, 1)
    leaf = np.empty(n, np.int32)
    left = np.zeros(m, np.int32)
    right = np.zeros(m, np.int32)
    mr = np.zeros(m, np.int32)
    boxes = np.zeros((m, 6), np.float32)
    rc = lib().ref_point_bvh(p, n, d, _ptr(leaf, C.c_int32), _ptr(left, C.c_int32),
                             _ptr(right, C.c_int32), _ptr(mr, C.c_int32), _ptr(boxes, C.c_float))
    assert rc == 0
    k = n - 1
    return {"leaf_ids": leaf, "left": left[:k], "right": right[:k], "max_rank": mr[:k],
            "boxes": boxes[:k]}


def build_grid(coords, eps, minpts) -> dict:
    a, p = _f32(coords)
    n, d = a.shape
    perm = np.empty(n, np.int32)
    cop = np.empty(n, np.int32)
    cid = np.empty(n, np.uint64)
    cb = np.empty(n, np.int32)
    ce = np.empty(n, np.int32)
    cd = np.empty(n, np.uint8)
    m = lib().ref_build_grid(p, n, d, C.c_float(eps), int(minpts), _ptr(perm, C.c_int32),
                             _ptr(cop, C.c_int32), _ptr(cid, C.c_uint64), _ptr(cb, C.c_int32),
                             _ptr(ce, C.c_int32), _ptr(cd, C.c_uint8), n)
    if m < 0:
        raise ValueError("build_grid rejected the input (code %d)" % m)
    return {"perm": perm, "cell_of_point": cop, "cell_id": cid[:m], "begin": cb[:m],
            "end": ce[:m], "dense": cd[:m].astype(bool)}


def mixed_bvh(coords, eps, minpts) -> dict:
    """The DenseBox tree over make_mixed_primitives (dense_grid.cpp:79-98): leaf
    kinds (1 = DenseBox) / ids per rank and the Bvh node accessors."""
    a, p = _f32(coords)
    n, d = a.shape
    kind = np.empty(n, np.uint8)
    lid = np.empty(n, np.int32)
    m1 = max(n - 1, 1)
    left, right, mr = (np.zeros(m1, np.int32) for _ in range(3))
    boxes = np.zeros((m1, 6), np.float32)
    m = lib().ref_mixed_bvh(p, n, d, C.c_float(eps), int(minpts), _ptr(kind, C.c_uint8),
                            _ptr(lid, C.c_int32), _ptr(left, C.c_int32), _ptr(right, C.c_int32),
                            _ptr(mr, C.c_int32), _ptr(boxes, C.c_float), n)
    if m < 0:
        raise ValueError("reference mixed BVH build failed")
    return {"leaf_kind": kind[:m], "leaf_id": lid[:m], "left": left[:m - 1],
            "right": right[:m - 1], "max_rank": mr[:m - 1], "boxes": boxes[:m - 1]}


def dbscan(coords, eps, minpts, algo: int, threads: int = 1) -> dict:
    """dbscan_run (algo 0 FDBSCAN, 1 DenseBox) or dbscan_bruteforce (algo 2)."""
    a, p = _f32(coords)
    n, d = a.shape
    labels = np.empty(n, np.int32)
    core = np.empty(n, np.uint8)
    st = np.zeros(5, np.float64)
    ct = np.zeros(6, np.int64)
    rc = lib().ref_dbscan(p, n, d, C.c_float(eps), int(minpts), int(algo), int(threads),
                          _ptr(labels, C.c_int32), _ptr(core, C.c_uint8),
                          _ptr(st, C.c_double), _ptr(ct, C.c_int64))
    if rc != 0:
        raise ValueError("reference dbscan_run failed with status %d" % rc)
    return {"labels": labels, "core": core,
            "stats": {"build_seconds": st[0], "preprocess_seconds": st[1], "main_seconds": st[2],
                      "finalize_seconds": st[3], "dense_point_fraction": st[4],
                      "preprocess_skipped": int(ct[0]), "pair_resolutions": int(ct[1]),
                      "distance_evaluations": int(ct[2]), "cluster_count": int(ct[3]),
                      "core_count": int(ct[4]), "noise_count": int(ct[5])}}


def check_equivalence(coords, eps, minpts, la, ca, lb, cb):
    a, p = _f32(coords)
    n, d = a.shape
    la = np.ascontiguousarray(la, np.int32)
    lb = np.ascontiguousarray(lb, np.int32)
    ca = np.ascontiguousarray(ca, np.uint8)
    cb = np.ascontiguousarray(cb, np.uint8)
    msg = C.create_string_buffer(512)
    ok = lib().ref_check_equivalence(p, n, d, C.c_float(eps), int(minpts), _ptr(la, C.c_int32),
                                     _ptr(ca, C.c_uint8), _ptr(lb, C.c_int32), _ptr(cb, C.c_uint8),
                                     msg, len(msg))
    return bool(ok), msg.value.decode("utf-8", "replace")


def random_instance(seed, min_n=50, max_n=2000):
    dim = C.c_int()
    eps = C.c_float()
    minpts = C.c_int()
    n = lib().ref_random_instance(seed, min_n, max_n, C.byref(dim), C.byref(eps),
                                  C.byref(minpts), None)
    coords = np.empty((n, dim.value), np.float32)
    lib().ref_random_instance(seed, min_n, max_n, C.byref(dim), C.byref(eps), C.byref(minpts),
                              _ptr(coords, C.c_float))
    return coords, eps.value, minpts.value


# ---------------------------------------------------------------------------
# The reference's own public C ABI (REF include/treeclust.h:52-103), for the
# CPU baseline: bench.py's reference arm loads its input through
# tc_dataset_load and times tc_cluster exactly as a reference caller would.
# ---------------------------------------------------------------------------
class RefStats(C.Structure):
    """tc_cluster_stats (REF include/treeclust.h:38-50)."""

    _fields_ = [("build_seconds", C.c_double), ("preprocess_seconds", C.c_double),
                ("main_seconds", C.c_double), ("finalize_seconds", C.c_double),
                ("preprocess_skipped", C.c_int), ("dense_point_fraction", C.c_double),
                ("pair_resolutions", C.c_uint64), ("distance_evaluations", C.c_uint64),
                ("cluster_count", C.c_int64), ("core_count", C.c_int64),
                ("noise_count", C.c_int64)]

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


def _capi():
    L = lib()
    if not getattr(L, "_capi_ready", False):
        V, PP = C.c_void_p, C.POINTER(C.c_void_p)
        L.tc_dataset_load.argtypes = [C.c_char_p, C.c_int, PP]
        L.tc_dataset_create.argtypes = [C.POINTER(C.c_float), C.c_int64, C.c_int, PP]
        L.tc_dataset_size.restype = C.c_int64
        L.tc_dataset_size.argtypes = [V]
        L.tc_dataset_free.argtypes = [V]
        L.tc_cluster.argtypes = [V, C.c_float, C.c_int, C.c_int, C.c_int, C.c_int64, PP]
        L.tc_result_stats.argtypes = [V, C.POINTER(RefStats)]
        L.tc_result_labels.restype = C.POINTER(C.c_int32)
        L.tc_result_labels.argtypes = [V]
        L.tc_result_core_flags.restype = C.POINTER(C.c_uint8)
        L.tc_result_core_flags.argtypes = [V]
        L.tc_result_free.argtypes = [V]
        L._capi_ready = True
    return L


class RefDataset:
    """A reference tc_dataset handle (tc_dataset_load / tc_dataset_create)."""

    def __init__(self, handle):
        self.h = handle

    @classmethod
    def load(cls, path: str) -> "RefDataset":
        h = C.c_void_p()
        st = _capi().tc_dataset_load(path.encode(), 0, C.byref(h))
        if st != 0:
            raise RuntimeError(f"reference tc_dataset_load({path}) -> status {st}")
        return cls(h)

    @classmethod
    def from_array(cls, coords) -> "RefDataset":
        a, p = _f32(coords)
        h = C.c_void_p()
        st = _capi().tc_dataset_create(p, a.shape[0], a.shape[1], C.byref(h))
        if st != 0:
            raise RuntimeError(f"reference tc_dataset_create -> status {st}")
        return cls(h)

    @property
    def size(self) -> int:
        return int(_capi().tc_dataset_size(self.h))

    def cluster(self, eps, minpts, algo, threads=0, want_labels=False):
        """Reference tc_cluster (REF capi.cpp:150-184). Returns (wall seconds of
        the call, stats dict, labels or None, core flags or None)."""
        import time

        L = _capi()
        res = C.c_void_p()
        t0 = time.perf_counter()
        st = L.tc_cluster(self.h, C.c_float(eps), int(minpts), int(algo), int(threads), 0,
                          C.byref(res))
        dt = time.perf_counter() - t0
        if st != 0:
            raise RuntimeError(f"reference tc_cluster -> status {st}")
        try:
            s = RefStats()
            L.tc_result_stats(res, C.byref(s))
            labels = core = None
            if want_labels:
                n = self.size
                labels = np.ctypeslib.as_array(L.tc_result_labels(res), shape=(n,)).copy()
                core = np.ctypeslib.as_array(L.tc_result_core_flags(res), shape=(n,)).copy()
            return dt, s.to_dict(), labels, core
        finally:
            L.tc_result_free(res)

    def close(self):
        if self.h:
            _capi().tc_dataset_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_cpu_model() -> str:
    """`lscpu` model name of this host (for the cpu_baseline record)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
