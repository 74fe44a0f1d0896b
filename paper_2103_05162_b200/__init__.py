"""B200-native DBSCAN engine (FDBSCAN / FDBSCAN-DenseBox, arXiv 2103.05162).

The product is the C-ABI shared library ``libtreeclust_b200.so`` (include/
treeclust.h is the reference's ABI, include/treeclust_gpu.h the additive
device-resident / generator entry points). This package is a thin ctypes
mirror of that ABI for tests and benchmarks.
"""
from ._lib import LIB_PATH, lib  # noqa: F401  (raises ImportError if the .so is missing)
from .api import (  # noqa: F401
    STAGES,
    Algorithm,
    Dataset,
    FileFormat,
    Result,
    Status,
    TreeclustError,
    cluster,
    cluster_device,
    cluster_device_async,
    cluster_multi,
    cluster_raw,
    device_count,
    generate_device,
    last_launch_count,
    last_stage_ms,
    load_device,
    release_cached_memory,
    set_pool_release_threshold,
    status_string,
    verify,
)
