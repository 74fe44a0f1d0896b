"""ctypes binding of the C ABI in ``include/treeclust.h`` + ``include/treeclust_gpu.h``.

The shared library ``libtreeclust_b200.so`` is built in-tree by
``__graft_entry__.build()`` (``make -C paper_2103_05162_b200/csrc``). There is
no fallback: importing this module without the library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TCB_LIB_PATH") or os.path.join(_HERE, "libtreeclust_b200.so")


class TcClusterStats(C.Structure):
    """``tc_cluster_stats`` (treeclust.h; reference treeclust.h:38-50)."""

    _fields_ = [
        ("build_seconds", C.c_double),
        ("preprocess_seconds", C.c_double),
        ("main_seconds", C.c_double),
        ("finalize_seconds", C.c_double),
        ("preprocess_skipped", C.c_int),
        ("dense_point_fraction", C.c_double),
        ("pair_resolutions", C.c_uint64),
        ("distance_evaluations", C.c_uint64),
        ("cluster_count", C.c_int64),
        ("core_count", C.c_int64),
        ("noise_count", C.c_int64),
    ]

    def to_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes). Every symbol declared in include/*.h.
SIGNATURES = {
    # treeclust.h (reference ABI)
    "tc_status_string": (C.c_char_p, [C.c_int]),
    "tc_dataset_create": (C.c_int, [C.POINTER(C.c_float), C.c_int64, C.c_int, _PP]),
    "tc_dataset_load": (C.c_int, [C.c_char_p, C.c_int, _PP]),
    "tc_dataset_save": (C.c_int, [_P, C.c_char_p, C.c_int]),
    "tc_dataset_size": (C.c_int64, [_P]),
    "tc_dataset_dim": (C.c_int, [_P]),
    "tc_dataset_coords": (C.POINTER(C.c_float), [_P]),
    "tc_dataset_free": (None, [_P]),
    "tc_generate_blobs": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_float, C.c_float,
                                    C.c_uint64, _PP]),
    "tc_generate_uniform": (C.c_int, [C.c_int64, C.c_int, C.POINTER(C.c_float),
                                      C.POINTER(C.c_float), C.c_uint64, _PP]),
    "tc_generate_lattice": (C.c_int, [C.c_int64, C.c_int, C.c_float, _PP]),
    "tc_cluster": (C.c_int, [_P, C.c_float, C.c_int, C.c_int, C.c_int, C.c_int64, _PP]),
    "tc_result_size": (C.c_int64, [_P]),
    "tc_result_labels": (C.POINTER(C.c_int32), [_P]),
    "tc_result_core_flags": (C.POINTER(C.c_uint8), [_P]),
    "tc_result_stats": (C.c_int, [_P, C.POINTER(TcClusterStats)]),
    "tc_result_free": (None, [_P]),
    "tc_verify": (C.c_int, [_P, C.c_float, C.c_int, C.c_int, C.c_int64, C.c_char_p, C.c_size_t]),
    # treeclust_gpu.h (additive)
    "tcg_device_count": (C.c_int, []),
    "tcg_version": (C.c_char_p, []),
    "tcg_cluster_device": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, C.c_int, C.c_int,
                                     C.c_int64, _P, _P, _P, C.POINTER(TcClusterStats)]),
    "tcg_last_stage_ms": (C.c_int, [C.POINTER(C.c_double), C.c_int]),
    "tcg_last_launch_count": (C.c_int64, []),
    "tcg_generate_hacc_like": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_uint64, _PP]),
    "tcg_generate_taxi_like": (C.c_int, [C.c_int64, C.c_uint64, _PP]),
    "tcg_generate_blobs_device": (C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_float, C.c_float,
                                            C.c_uint64, _P, _P]),
    "tcg_generate_uniform_device": (C.c_int, [C.c_int64, C.c_int, C.POINTER(C.c_float),
                                              C.POINTER(C.c_float), C.c_uint64, _P, _P]),
    "tcg_generate_lattice_device": (C.c_int, [C.c_int64, C.c_int, C.c_float, _P, _P]),
    "tcg_generate_hacc_like_device": (C.c_int, [C.c_int64, C.c_double, C.c_double, C.c_uint64,
                                                _P, _P]),
    "tcg_generate_taxi_like_device": (C.c_int, [C.c_int64, C.c_uint64, _P, _P]),
    "tcg_random_instance": (C.c_int, [C.c_uint64, C.c_int64, C.c_int64, C.POINTER(C.c_float),
                                      C.POINTER(C.c_int), _PP]),
    "tcg_morton_codes_device": (C.c_int, [_P, C.c_int64, C.c_int, C.POINTER(C.c_float),
                                          C.POINTER(C.c_float), _P, _P]),
    "tcg_near_boxes_device": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, _P, _P, C.c_int64,
                                        _P, _P]),
    "tcg_shard_route_device": (C.c_int, [_P, _P, _P, C.c_int64, C.c_int, _P, C.c_int, _P, _P,
                                         _P]),
    "tcg_shard_unpack_rows_device": (C.c_int, [_P, C.c_int64, C.c_int, _P, _P, _P, _P]),
    "tcg_shard_region_boxes_device": (C.c_int, [_P, _P, C.c_int64, C.c_int, _P, _P, _P, _P]),
    "tcg_near_peers_device": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, _P, _P, _P, C.c_int64,
                                        _P, _P]),
    "tcg_core_flags_device": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, C.c_int, _P, _P]),
    "tcg_binary_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int)]),
    "tcg_load_binary_device": (C.c_int, [C.c_char_p, _P, C.c_int64, C.c_int, _P]),
    "tcg_local_create": (C.c_int, [_P, _P, C.c_int64, C.c_int, C.c_float, _P, _PP]),
    "tcg_local_core_flags": (C.c_int, [_P, C.c_int, _P]),
    "tcg_local_cluster": (C.c_int, [_P, _P, _P, _P]),
    "tcg_local_free": (None, [_P]),
    "tcg_cluster_multi": (C.c_int, [_P, C.c_float, C.c_int, C.c_int, C.POINTER(C.c_int), C.c_int,
                                    _PP]),
    "tcg_cluster_device_async": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, C.c_int, C.c_int,
                                         C.c_int64, _P, _P, _P, _P]),
    "tcg_cluster_keyed_device": (C.c_int, [_P, _P, C.c_int64, C.c_int, C.c_float, C.c_int, _P, _P,
                                         _P, C.POINTER(TcClusterStats)]),
    "tcg_cluster_given_core_device": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, _P, _P, _P,
                                                _P, C.POINTER(TcClusterStats)]),
    "tcg_union_edges_device": (C.c_int, [_P, C.c_int64, C.c_int32, _P, _P]),
    "tcg_debug_point_bvh": (C.c_int, [C.POINTER(C.c_float), C.c_int64, C.c_int,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_float)]),
    "tcg_debug_sort_pairs": (C.c_int, [C.POINTER(C.c_uint64), C.c_int64, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_int32)]),
    "tcg_debug_union_find": (C.c_int, [C.POINTER(C.c_int32), C.c_int64, C.c_int32,
                                       C.POINTER(C.c_int32)]),
    "tcg_debug_grid": (C.c_int, [C.POINTER(C.c_float), C.c_int64, C.c_int, C.c_float, C.c_int,
                                 C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                 C.POINTER(C.c_uint64), C.POINTER(C.c_int32),
                                 C.POINTER(C.c_int32), C.POINTER(C.c_uint8), C.c_int64,
                                 C.POINTER(C.c_int64)]),
    "tcg_debug_mixed_bvh": (C.c_int, [C.POINTER(C.c_float), C.c_int64, C.c_int, C.c_float,
                                      C.c_int, C.POINTER(C.c_uint8), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32), C.POINTER(C.c_float), C.c_int64,
                                      C.POINTER(C.c_int64)]),
    "tcg_check_equivalence_device": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, _P, _P, _P, _P,
                                               _P, C.POINTER(C.c_int), C.POINTER(C.c_int64)]),
    "tcg_first_bad_border_device": (C.c_int, [_P, C.c_int64, C.c_int, C.c_float, _P, _P, _P,
                                              C.POINTER(C.c_int64)]),
    "tcg_set_pool_release_threshold": (C.c_int, [C.c_uint64]),
    "tcg_release_cached_memory": (None, []),
    "tcg_dataset_create_pinned": (C.c_int, [C.POINTER(C.c_float), C.c_int64, C.c_int, _PP]),
}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("TCB_LIB_PATH") and not hasattr(lib, name):
            continue  # A/B of an older build (tools/ab_libs.sh): newer entry points absent
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()
