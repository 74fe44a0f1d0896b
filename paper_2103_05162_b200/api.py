"""Python mirror of the reference C ABI (``/root/reference/proj/include/treeclust.h``).

Same names, argument meaning and error behaviour as the ``tc_*`` functions:
a non-``TC_OK`` status raises :class:`TreeclustError` carrying the status code.
Everything runs through ``libtreeclust_b200.so`` (C ABI, sm_100a kernels);
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from ._lib import TcClusterStats, lib


class Status(enum.IntEnum):
    OK = 0
    INVALID_ARGUMENT = 1
    IO = 2
    VERIFY_FAIL = 3
    CAP_EXCEEDED = 4
    INTERNAL = 5


class Algorithm(enum.IntEnum):
    FDBSCAN = 0
    DENSEBOX = 1
    BRUTEFORCE = 2


class FileFormat(enum.IntEnum):
    AUTO = 0
    CSV = 1
    BINARY = 2


class TreeclustError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = Status(status)
        msg = lib.tc_status_string(int(status)).decode()
        super().__init__(f"{where}: {msg} ({self.status.name})")


def _check(status: int, where: str) -> None:
    if status != 0:
        raise TreeclustError(status, where)


STAGES = ("bounds_morton", "sort", "topology_refit", "grid", "core", "main", "finalize", "total")


class Dataset:
    """Owns a ``tc_dataset*`` (host points, row-major n x dim float32)."""

    def __init__(self, handle: int):
        if not handle:
            raise ValueError("null tc_dataset")
        self._h = C.c_void_p(handle)

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.tc_dataset_free(h)
            self._h = C.c_void_p()

    # ---- constructors (tc_dataset_create / _load / tc_generate_*) ----
    @classmethod
    def from_array(cls, coords) -> "Dataset":
        a = np.ascontiguousarray(coords, dtype=np.float32)
        if a.ndim != 2:
            raise TreeclustError(Status.INVALID_ARGUMENT, "tc_dataset_create")
        out = C.c_void_p()
        _check(lib.tc_dataset_create(a.ctypes.data_as(C.POINTER(C.c_float)), a.shape[0],
                                     a.shape[1], C.byref(out)), "tc_dataset_create")
        return cls(out.value)

    @classmethod
    def load(cls, path: str, fmt: FileFormat = FileFormat.AUTO) -> "Dataset":
        out = C.c_void_p()
        _check(lib.tc_dataset_load(path.encode(), int(fmt), C.byref(out)), "tc_dataset_load")
        return cls(out.value)

    @classmethod
    def blobs(cls, k, per_blob, dim, separation, sigma, seed) -> "Dataset":
        out = C.c_void_p()
        _check(lib.tc_generate_blobs(k, per_blob, dim, separation, sigma, seed, C.byref(out)),
               "tc_generate_blobs")
        return cls(out.value)

    @classmethod
    def uniform(cls, n, dim, lo, hi, seed) -> "Dataset":
        lo_a = (C.c_float * 3)(*([float(v) for v in lo] + [0.0] * (3 - len(lo))))
        hi_a = (C.c_float * 3)(*([float(v) for v in hi] + [0.0] * (3 - len(hi))))
        out = C.c_void_p()
        _check(lib.tc_generate_uniform(n, dim, lo_a, hi_a, seed, C.byref(out)),
               "tc_generate_uniform")
        return cls(out.value)

    @classmethod
    def lattice(cls, side, dim, spacing) -> "Dataset":
        out = C.c_void_p()
        _check(lib.tc_generate_lattice(side, dim, spacing, C.byref(out)), "tc_generate_lattice")
        return cls(out.value)

    @classmethod
    def hacc_like(cls, n, box_len=None, halo_frac=0.23, seed=11) -> "Dataset":
        """L = 36.8 * (n / 37e6)^(1/3) keeps the C2 density."""
        if box_len is None:
            box_len = 36.8 * (n / 37e6) ** (1.0 / 3.0)
        out = C.c_void_p()
        _check(lib.tcg_generate_hacc_like(n, box_len, halo_frac, seed, C.byref(out)),
               "tcg_generate_hacc_like")
        return cls(out.value)

    @classmethod
    def taxi_like(cls, n, seed=5) -> "Dataset":
        out = C.c_void_p()
        _check(lib.tcg_generate_taxi_like(n, seed, C.byref(out)), "tcg_generate_taxi_like")
        return cls(out.value)

    @classmethod
    def random_instance(cls, seed, min_n=50, max_n=2000):
        """testutil::random_instance -> (Dataset, eps, minpts)."""
        eps = C.c_float()
        minpts = C.c_int()
        out = C.c_void_p()
        _check(lib.tcg_random_instance(seed, min_n, max_n, C.byref(eps), C.byref(minpts),
                                       C.byref(out)), "tcg_random_instance")
        return cls(out.value), eps.value, minpts.value

    # ---- accessors ----
    def save(self, path: str, fmt: FileFormat = FileFormat.AUTO) -> None:
        _check(lib.tc_dataset_save(self._h, path.encode(), int(fmt)), "tc_dataset_save")

    @property
    def size(self) -> int:
        return int(lib.tc_dataset_size(self._h))

    @property
    def dim(self) -> int:
        return int(lib.tc_dataset_dim(self._h))

    def coords(self) -> np.ndarray:
        n, d = self.size, self.dim
        ptr = lib.tc_dataset_coords(self._h)
        return np.ctypeslib.as_array(ptr, shape=(n, d)).copy()

    def __len__(self) -> int:
        return self.size


@dataclass
class Result:
    labels: np.ndarray
    core_flags: np.ndarray
    stats: dict


def cluster(ds: Dataset, eps: float, minpts: int, algorithm: Algorithm = Algorithm.FDBSCAN,
            threads: int = 0, oracle_cap: int = 0) -> Result:
    """``tc_cluster`` + ``tc_result_*``: host dataset in, host labels/flags out."""
    res = C.c_void_p()
    _check(lib.tc_cluster(ds.handle, C.c_float(eps), int(minpts), int(algorithm), int(threads),
                          int(oracle_cap), C.byref(res)), "tc_cluster")
    try:
        n = int(lib.tc_result_size(res))
        labels = np.ctypeslib.as_array(lib.tc_result_labels(res), shape=(n,)).copy()
        core = np.ctypeslib.as_array(lib.tc_result_core_flags(res), shape=(n,)).copy()
        st = TcClusterStats()
        _check(lib.tc_result_stats(res, C.byref(st)), "tc_result_stats")
        return Result(labels, core, st.to_dict())
    finally:
        lib.tc_result_free(res)


def cluster_multi(ds: Dataset, eps: float, minpts: int, devices,
                  algorithm: Algorithm = Algorithm.FDBSCAN) -> Result:
    """``tcg_cluster_multi``: the Morton-range sharded path over the listed CUDA
    devices (one shard per entry; entries may repeat), host in / host out."""
    devs = (C.c_int * len(devices))(*[int(d) for d in devices])
    res = C.c_void_p()
    _check(lib.tcg_cluster_multi(ds.handle, C.c_float(eps), int(minpts), int(algorithm), devs,
                                 len(devices), C.byref(res)), "tcg_cluster_multi")
    try:
        n = int(lib.tc_result_size(res))
        labels = np.ctypeslib.as_array(lib.tc_result_labels(res), shape=(n,)).copy()
        core = np.ctypeslib.as_array(lib.tc_result_core_flags(res), shape=(n,)).copy()
        st = TcClusterStats()
        _check(lib.tc_result_stats(res, C.byref(st)), "tc_result_stats")
        return Result(labels, core, st.to_dict())
    finally:
        lib.tc_result_free(res)


def cluster_raw(ds: Dataset, eps: float, minpts: int, algorithm: Algorithm = Algorithm.FDBSCAN,
                threads: int = 0, oracle_cap: int = 0) -> int:
    """``tc_cluster`` then ``tc_result_free``; returns the status (for timing the ABI)."""
    res = C.c_void_p()
    st = lib.tc_cluster(ds.handle, C.c_float(eps), int(minpts), int(algorithm), int(threads),
                        int(oracle_cap), C.byref(res))
    if st == 0:
        lib.tc_result_free(res)
    return st


def cluster_device(coords, eps: float, minpts: int, algorithm: Algorithm = Algorithm.FDBSCAN,
                   labels=None, core=None, stream=None, stats: bool = False, oracle_cap: int = 0):
    """``tcg_cluster_device`` on torch CUDA tensors (coords: float32 [n, dim], contiguous).

    Launches on ``stream`` (a torch.cuda.Stream; default: the current stream) and
    returns ``(labels, core, stats_or_None)``; with ``stats=False`` the call does
    not synchronize at the end.
    """
    import torch

    if not (coords.is_cuda and coords.dtype == torch.float32 and coords.dim() == 2
            and coords.is_contiguous()):
        raise TreeclustError(Status.INVALID_ARGUMENT, "tcg_cluster_device")
    n, d = coords.shape
    if labels is None:
        labels = torch.empty(n, dtype=torch.int32, device=coords.device)
    if core is None:
        core = torch.empty(n, dtype=torch.uint8, device=coords.device)
    s = stream if stream is not None else torch.cuda.current_stream(coords.device)
    st = TcClusterStats() if stats else None
    _check(lib.tcg_cluster_device(C.c_void_p(coords.data_ptr()), n, d, C.c_float(eps),
                                  int(minpts), int(algorithm), int(oracle_cap),
                                  C.c_void_p(labels.data_ptr()), C.c_void_p(core.data_ptr()),
                                  C.c_void_p(s.cuda_stream),
                                  C.byref(st) if st is not None else None),
           "tcg_cluster_device")
    return labels, core, (st.to_dict() if st is not None else None)


def cluster_device_async(coords, eps: float, minpts: int,
                         algorithm: Algorithm = Algorithm.FDBSCAN, labels=None, core=None,
                         status=None, stream=None, oracle_cap: int = 0):
    """``tcg_cluster_device_async``: ``cluster_device`` without stats, the run's
    status written to ``status`` (an int32 CUDA tensor of one element; the
    non-finite-coordinate error of FDBSCAN is found on the device). For FDBSCAN
    the call never synchronizes the host, so it can be captured in a CUDA graph.
    Returns ``(labels, core, status)``."""
    import torch

    if not (coords.is_cuda and coords.dtype == torch.float32 and coords.dim() == 2
            and coords.is_contiguous()):
        raise TreeclustError(Status.INVALID_ARGUMENT, "tcg_cluster_device_async")
    n, d = coords.shape
    if labels is None:
        labels = torch.empty(n, dtype=torch.int32, device=coords.device)
    if core is None:
        core = torch.empty(n, dtype=torch.uint8, device=coords.device)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=coords.device)
    s = stream if stream is not None else torch.cuda.current_stream(coords.device)
    _check(lib.tcg_cluster_device_async(C.c_void_p(coords.data_ptr()), n, d, C.c_float(eps),
                                        int(minpts), int(algorithm), int(oracle_cap),
                                        C.c_void_p(labels.data_ptr()),
                                        C.c_void_p(core.data_ptr()), C.c_void_p(s.cuda_stream),
                                        C.c_void_p(status.data_ptr())),
           "tcg_cluster_device_async")
    return labels, core, status


def load_device(path: str, device=None):
    """``tcg_binary_info`` + ``tcg_load_binary_device``: a .bin point file to a
    (n, dim) float32 CUDA tensor, file reads overlapped with the copies."""
    import torch

    n, d = C.c_int64(), C.c_int()
    _check(lib.tcg_binary_info(path.encode(), C.byref(n), C.byref(d)), "tcg_binary_info")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    out = torch.empty((n.value, d.value), dtype=torch.float32, device=dev)
    s = torch.cuda.current_stream(dev)
    _check(lib.tcg_load_binary_device(path.encode(), C.c_void_p(out.data_ptr()), n.value, d.value,
                                      C.c_void_p(s.cuda_stream)), "tcg_load_binary_device")
    return out


def verify(ds: Dataset, eps: float, minpts: int, threads: int = 0, oracle_cap: int = 0):
    """``tc_verify`` -> (Status, report text)."""
    buf = C.create_string_buffer(8192)
    st = lib.tc_verify(ds.handle, C.c_float(eps), int(minpts), int(threads), int(oracle_cap),
                       buf, len(buf))
    return Status(st), buf.value.decode("utf-8", "replace")


EQUIVALENCE_CHECKS = ("PASS", "core flags differ", "noise sets differ", "core partitions differ",
                      "first clustering has an invalid border label",
                      "second clustering has an invalid border label")


def _dev_ptrs(coords, *arrays):
    import torch

    if not (coords.is_cuda and coords.dtype == torch.float32 and coords.dim() == 2
            and coords.is_contiguous()):
        raise TreeclustError(Status.INVALID_ARGUMENT, "device coords")
    for a in arrays:
        if not (a.is_cuda and a.is_contiguous() and a.shape[0] == coords.shape[0]):
            raise TreeclustError(Status.INVALID_ARGUMENT, "device arrays")
    return [C.c_void_p(a.data_ptr()) for a in (coords,) + arrays]


def check_equivalence_device(coords, eps, labels_a, core_a, labels_b, core_b, stream=None):
    """``tcg_check_equivalence_device`` (REF oracle.cpp:120-163 on the GPU):
    returns (check code, point index, message) with check 0 = PASS."""
    import torch

    ptrs = _dev_ptrs(coords, labels_a, core_a, labels_b, core_b)
    s = stream if stream is not None else torch.cuda.current_stream(coords.device)
    chk, at = C.c_int(), C.c_int64()
    _check(lib.tcg_check_equivalence_device(ptrs[0], coords.shape[0], coords.shape[1],
                                            C.c_float(eps), *ptrs[1:], C.c_void_p(s.cuda_stream),
                                            C.byref(chk), C.byref(at)),
           "tcg_check_equivalence_device")
    msg = EQUIVALENCE_CHECKS[chk.value]
    if chk.value:
        msg += f" (first divergence at point {at.value})"
    return chk.value, at.value, msg


def first_bad_border(coords, eps, labels, core, stream=None) -> int:
    """``tcg_first_bad_border_device`` (REF oracle.cpp:72-116): smallest border
    index with no same-label core within eps, or -1."""
    import torch

    ptrs = _dev_ptrs(coords, labels, core)
    s = stream if stream is not None else torch.cuda.current_stream(coords.device)
    at = C.c_int64()
    _check(lib.tcg_first_bad_border_device(ptrs[0], coords.shape[0], coords.shape[1],
                                           C.c_float(eps), ptrs[1], ptrs[2],
                                           C.c_void_p(s.cuda_stream), C.byref(at)),
           "tcg_first_bad_border_device")
    return at.value


def last_stage_ms() -> dict:
    arr = (C.c_double * len(STAGES))()
    k = lib.tcg_last_stage_ms(arr, len(STAGES))
    return {STAGES[i]: arr[i] for i in range(k)}


def set_pool_release_threshold(nbytes: int) -> None:
    """Scratch bytes the library's device memory pool keeps across calls
    (tcg_set_pool_release_threshold; default 24 GiB). Raise it for repeated
    runs larger than that (the 497M-point case needs ~80 GB of scratch)."""
    _check(lib.tcg_set_pool_release_threshold(int(nbytes)), "tcg_set_pool_release_threshold")


def release_cached_memory() -> None:
    """Frees the library's cached device scratch and pinned host staging now."""
    lib.tcg_release_cached_memory()


def last_launch_count() -> int:
    return int(lib.tcg_last_launch_count())


def device_count() -> int:
    return int(lib.tcg_device_count())


def status_string(status: int) -> str:
    return lib.tc_status_string(int(status)).decode()


# ---- stage probes (tcg_debug_*): one device stage, host in / host out ----
def debug_point_bvh(coords) -> dict:
    a = np.ascontiguousarray(coords, np.float32)
    n, d = a.shape
    m = max(n - 1, 1)
    leaf = np.empty(n, np.int32)
    left, right, mr = (np.zeros(m, np.int32) for _ in range(3))
    boxes = np.zeros((m, 6), np.float32)
    p = lambda v, t: v.ctypes.data_as(C.POINTER(t))  # noqa: E731
    _check(lib.tcg_debug_point_bvh(p(a, C.c_float), n, d, p(leaf, C.c_int32), p(left, C.c_int32),
                                   p(right, C.c_int32), p(mr, C.c_int32), p(boxes, C.c_float)),
           "tcg_debug_point_bvh")
    k = n - 1
    return {"leaf_ids": leaf, "left": left[:k], "right": right[:k], "max_rank": mr[:k],
            "boxes": boxes[:k]}


def debug_sort_pairs(keys):
    k = np.ascontiguousarray(keys, np.uint64)
    ko = np.empty_like(k)
    vo = np.empty(k.shape[0], np.int32)
    _check(lib.tcg_debug_sort_pairs(k.ctypes.data_as(C.POINTER(C.c_uint64)), k.shape[0],
                                    ko.ctypes.data_as(C.POINTER(C.c_uint64)),
                                    vo.ctypes.data_as(C.POINTER(C.c_int32))), "tcg_debug_sort_pairs")
    return ko, vo


def debug_union_find(edges, n: int) -> np.ndarray:
    e = np.ascontiguousarray(edges, np.int32).reshape(-1, 2)
    out = np.empty(n, np.int32)
    _check(lib.tcg_debug_union_find(e.ctypes.data_as(C.POINTER(C.c_int32)), e.shape[0], n,
                                    out.ctypes.data_as(C.POINTER(C.c_int32))),
           "tcg_debug_union_find")
    return out


def debug_grid(coords, eps: float, minpts: int) -> dict:
    """tcg_debug_grid: the device build_grid in the reference's DenseGrid view."""
    a = np.ascontiguousarray(coords, np.float32)
    n, d = a.shape
    perm = np.empty(n, np.int32)
    cop = np.empty(n, np.int32)
    cid = np.empty(n, np.uint64)
    cb, ce = np.empty(n, np.int32), np.empty(n, np.int32)
    cd = np.empty(n, np.uint8)
    m = C.c_int64(0)
    p = lambda v, t: v.ctypes.data_as(C.POINTER(t))  # noqa: E731
    _check(lib.tcg_debug_grid(p(a, C.c_float), n, d, C.c_float(eps), int(minpts),
                              p(perm, C.c_int32), p(cop, C.c_int32), p(cid, C.c_uint64),
                              p(cb, C.c_int32), p(ce, C.c_int32), p(cd, C.c_uint8), n,
                              C.byref(m)), "tcg_debug_grid")
    k = m.value
    return {"perm": perm, "cell_of_point": cop, "cell_id": cid[:k], "begin": cb[:k],
            "end": ce[:k], "dense": cd[:k].astype(bool)}


def debug_mixed_bvh(coords, eps: float, minpts: int) -> dict:
    """tcg_debug_mixed_bvh: the DenseBox tree in the reference's node view."""
    a = np.ascontiguousarray(coords, np.float32)
    n, d = a.shape
    cap = n
    kind = np.empty(cap, np.uint8)
    lid = np.empty(cap, np.int32)
    m1 = max(cap - 1, 1)
    left, right, mr = (np.zeros(m1, np.int32) for _ in range(3))
    boxes = np.zeros((m1, 6), np.float32)
    m = C.c_int64(0)
    p = lambda v, t: v.ctypes.data_as(C.POINTER(t))  # noqa: E731
    _check(lib.tcg_debug_mixed_bvh(p(a, C.c_float), n, d, C.c_float(eps), int(minpts),
                                   p(kind, C.c_uint8), p(lid, C.c_int32), p(left, C.c_int32),
                                   p(right, C.c_int32), p(mr, C.c_int32), p(boxes, C.c_float),
                                   cap, C.byref(m)), "tcg_debug_mixed_bvh")
    k = m.value
    return {"leaf_kind": kind[:k], "leaf_id": lid[:k], "left": left[:k - 1],
            "right": right[:k - 1], "max_rank": mr[:k - 1], "boxes": boxes[:k - 1]}


def generate_device(kind: str, *args, device=None, stream=None):
    """Device-side generators (tcg_generate_*_device): a
    float32 [n, dim] CUDA tensor equal to the host generator's output.

      generate_device("blobs", k, per_blob, dim, separation, sigma, seed)
      generate_device("uniform", n, dim, lo, hi, seed)
      generate_device("lattice", side, dim, spacing)
      generate_device("hacc_like", n, box_len=None, halo_frac=0.23, seed=11)
      generate_device("taxi_like", n, seed=5)
    """
    import torch

    dev = torch.device(device) if device is not None else torch.device("cuda")
    if kind == "blobs":
        k, per_blob, dim, sep, sigma, seed = args
        shape = (k * per_blob, dim)
        call = lambda o, s: lib.tcg_generate_blobs_device(k, per_blob, dim, sep, sigma, seed, o, s)  # noqa: E731
    elif kind == "uniform":
        n, dim, lo, hi, seed = args
        lo_a = (C.c_float * 3)(*([float(v) for v in lo] + [0.0] * (3 - len(lo))))
        hi_a = (C.c_float * 3)(*([float(v) for v in hi] + [0.0] * (3 - len(hi))))
        shape = (n, dim)
        call = lambda o, s: lib.tcg_generate_uniform_device(n, dim, lo_a, hi_a, seed, o, s)  # noqa: E731
    elif kind == "lattice":
        side, dim, spacing = args
        shape = (side ** dim, dim)
        call = lambda o, s: lib.tcg_generate_lattice_device(side, dim, spacing, o, s)  # noqa: E731
    elif kind == "hacc_like":
        n = args[0]
        box_len = args[1] if len(args) > 1 and args[1] is not None else 36.8 * (n / 37e6) ** (1 / 3)
        halo_frac = args[2] if len(args) > 2 else 0.23
        seed = args[3] if len(args) > 3 else 11
        shape = (n, 3)
        call = lambda o, s: lib.tcg_generate_hacc_like_device(n, box_len, halo_frac, seed, o, s)  # noqa: E731
    elif kind == "taxi_like":
        n = args[0]
        seed = args[1] if len(args) > 1 else 5
        shape = (n, 2)
        call = lambda o, s: lib.tcg_generate_taxi_like_device(n, seed, o, s)  # noqa: E731
    else:
        raise ValueError(kind)
    out = torch.empty(shape, dtype=torch.float32, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    _check(call(C.c_void_p(out.data_ptr()), C.c_void_p(st.cuda_stream)), f"tcg_generate_{kind}_device")
    return out
