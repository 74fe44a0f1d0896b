"""Device-side generators (REF datagen.cpp:10-88 and the
§8d HACC-like / taxi-like recipes): the tcg_generate_*_device output is the
host generator's output, byte for byte, including the C2 benchmark input
(sha256 pinned in tests/golden/bench_inputs.json)."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2103_05162_b200 as tb
from paper_2103_05162_b200 import Dataset, Status, TreeclustError

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _same(dev, host, tag):
    got = dev.cpu().numpy()
    assert got.shape == host.shape, tag
    diff = np.flatnonzero(got.view(np.uint32) != host.view(np.uint32))
    assert diff.size == 0, f"{tag}: {diff.size} of {got.size} values differ, first {diff[:5]}"


@pytest.mark.parametrize("dim", [2, 3])
def test_blobs_uniform_lattice_device_equal_host(dim):
    _same(tb.api.generate_device("blobs", 7, 30011, dim, 0.8333333, 0.08333333, 7),
          Dataset.blobs(7, 30011, dim, 0.8333333, 0.08333333, 7).coords(), "blobs")
    _same(tb.api.generate_device("blobs", 100, 10000, dim, 20.0, 1.0, 1003),
          Dataset.blobs(100, 10000, dim, 20.0, 1.0, 1003).coords(), "blobs-acceptance")
    lo, hi = [-1.5, 0.0, 2.0][:dim], [3.0, 220.0, 2.5][:dim]
    _same(tb.api.generate_device("uniform", 123457, dim, lo, hi, 99),
          Dataset.uniform(123457, dim, lo, hi, 99).coords(), "uniform")
    _same(tb.api.generate_device("lattice", 57, dim, 0.1), Dataset.lattice(57, dim, 0.1).coords(),
          "lattice")


@pytest.mark.parametrize("n,seed", [(1, 11), (5, 3), (250_000, 11), (2_000_000, 4)])
def test_hacc_like_device_equal_host(n, seed):
    _same(tb.api.generate_device("hacc_like", n, None, 0.23, seed),
          Dataset.hacc_like(n, seed=seed).coords(), f"hacc {n}")


@pytest.mark.parametrize("n,seed", [(1, 5), (40, 2), (3_000_001, 5)])
def test_taxi_like_device_equal_host(n, seed):
    _same(tb.api.generate_device("taxi_like", n, seed), Dataset.taxi_like(n, seed=seed).coords(),
          f"taxi {n}")


def test_bench_inputs_on_device_match_pinned_sha():
    """The full-size benchmark inputs generated on the device hash to the
    sha256 the reference-side oracle generator is pinned to (C2 = 37M
    HACC-like, C4 = 80M taxi-like)."""
    with open(os.path.join(GOLDEN, "bench_inputs.json")) as f:
        pins = json.load(f)
    for key, (kind, n) in {"hacc_like(37000000,L=36.8,0.23,seed=11)": ("hacc_like", 37_000_000),
                           "taxi_like(80000000,seed=5)": ("taxi_like", 80_000_000)}.items():
        x = tb.api.generate_device(kind, n)
        h = hashlib.sha256(x.cpu().numpy().tobytes()).hexdigest()
        assert h == pins[key], key


def test_device_generator_argument_errors():
    with pytest.raises(TreeclustError) as e:
        tb.api.generate_device("uniform", 10, 4, [0, 0, 0], [1, 1, 1], 1)
    assert e.value.status == Status.INVALID_ARGUMENT
    with pytest.raises(TreeclustError) as e:
        tb.api.generate_device("lattice", 1, 2, 0.1)
    assert e.value.status == Status.INVALID_ARGUMENT
