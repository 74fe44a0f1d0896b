"""The reference's acceptance suite (REF tests/acceptance.cpp, criteria 1-9)
replayed against the GPU path at the reference's own sizes and seeds.

Each test names the criterion and follows its instance generation, oracle
and pass condition; "threads" become repeated GPU runs (the device has no
thread-count knob, so determinism is checked run to run and against the
single-threaded oracle)."""
import time

import numpy as np
import pytest

import paper_2103_05162_b200 as tb
from oracle import oracle
from paper_2103_05162_b200 import Algorithm, Dataset

from ._util import assert_parity, brute_pair_count

pytestmark = pytest.mark.gpu

FD, DB, BF = Algorithm.FDBSCAN, Algorithm.DENSEBOX, Algorithm.BRUTEFORCE


def _equiv(coords, eps, a, b):
    ok, msg = oracle.check_equivalence(coords, eps, a.labels, a.core_flags, b.labels, b.core_flags)
    return ok, msg


def test_criterion_1_oracle_equivalence_200_instances():
    """acceptance.cpp:70-98: random_instance(seed, 50, 2000) for seeds 1..200,
    both algorithms against dbscan_bruteforce, under 2 minutes."""
    t0 = time.time()
    failed = []
    for seed in range(1, 201):
        ds, eps, mp = Dataset.random_instance(seed, 50, 2000)
        c = ds.coords()
        want = oracle.dbscan(c, eps, mp, 2)
        for algo in (FD, DB):
            got = tb.cluster(ds, eps, mp, algo)
            ok, msg = oracle.check_equivalence(c, eps, got.labels, got.core_flags,
                                               want["labels"], want["core"])
            if not ok:
                failed.append((seed, algo.name, msg))
    assert not failed, failed[:3]
    assert time.time() - t0 < 120.0


def _blob_mixture(n, dim, seed):
    """acceptance.cpp:54-68: 90% Gaussian blobs (k = 10, separation 20,
    sigma 1), 10% uniform background over [0, 20 (k + 1)]^dim."""
    k = 10
    per_blob = (n * 9) // (10 * k)
    blobs = Dataset.blobs(k, per_blob, dim, 20.0, 1.0, seed).coords()
    hi = 20.0 * (k + 1)
    noise = Dataset.uniform(n - blobs.shape[0], dim, [0.0] * dim, [hi] * dim, seed + 1).coords()
    return np.ascontiguousarray(np.concatenate([blobs, noise]), np.float32)


def test_criterion_2_cross_algorithm_20_instances_100k():
    """acceptance.cpp:100-123: FDBSCAN vs DenseBox on 20 blob mixtures of
    n = 100000 (eps 0.1 in 2D / 0.3 in 3D, minpts 2 + 3 (seed mod 3)),
    check_equivalence (device checker), under 2 minutes."""
    import torch

    t0 = time.time()
    for seed in range(20):
        dim = 3 if seed % 2 else 2
        c = _blob_mixture(100_000, dim, 1000 + seed)
        eps = 0.1 if dim == 2 else 0.3
        mp = 2 + 3 * (seed % 3)
        ds = Dataset.from_array(c)
        fd = tb.cluster(ds, eps, mp, FD)
        db = tb.cluster(ds, eps, mp, DB)
        x = torch.from_numpy(c).cuda()
        v = tb.api.check_equivalence_device(
            x, eps, *(torch.from_numpy(np.ascontiguousarray(a)).cuda()
                      for a in (fd.labels, fd.core_flags, db.labels, db.core_flags)))
        assert v[0] == 0, (seed, v)
        # same partition, and the core labels are equal, not just isomorphic
        assert_parity(db.labels, db.core_flags, fd.labels, fd.core_flags, f"seed {seed}")
    assert time.time() - t0 < 120.0


def test_criterion_3_pair_resolutions_exact_50_instances():
    """acceptance.cpp:125-139: main-phase pair resolutions equal the
    brute-force within-eps pair count (seeds 300..349)."""
    for seed in range(300, 350):
        ds, eps, mp = Dataset.random_instance(seed, 50, 2000)
        got = tb.cluster(ds, eps, mp, FD)
        assert got.stats["pair_resolutions"] == brute_pair_count(ds.coords(), eps), seed


def test_criterion_4_border_never_bridges_100_runs():
    """acceptance.cpp:141-172: two blobs 1.5 eps apart, the midpoint border
    joins exactly one cluster; 100 runs alternating the algorithms."""
    xs = [-0.75] + [-1.05 - 0.1 * i for i in range(4)] + [0.75] + \
         [1.05 + 0.1 * i for i in range(4)] + [0.0]
    c = np.array([[np.float32(x), 0.0] for x in xs], np.float32)
    ds = Dataset.from_array(c)
    for rep in range(100):
        algo = DB if rep % 2 else FD
        got = tb.cluster(ds, 1.0, 5, algo)
        in_left = got.labels[10] == got.labels[0]
        in_right = got.labels[10] == got.labels[5]
        assert got.stats["cluster_count"] == 2 and not got.core_flags[10], rep
        assert in_left != in_right, rep


def test_criterion_5_union_find_flatten_and_50_replays():
    """acceptance.cpp:174-233: (a) after flatten every parent is a root,
    20 random graphs; (b) 50 trials of 100000 random edges over 10000
    elements, concurrent device unite() vs sequential replay."""
    rng = np.random.default_rng(99)
    for trial in range(20):
        n = 1000 + int(rng.integers(0, 9000))
        edges = rng.integers(0, n, (2 * n, 2)).astype(np.int32)
        got = tb.api.debug_union_find(edges, n)
        assert np.array_equal(got, got[got]), trial
    n, m = 10000, 100_000
    for trial in range(50):
        edges = rng.integers(0, n, (m, 2)).astype(np.int32)
        got = tb.api.debug_union_find(edges, n)
        # sequential replay with min-index hooks, vectorised per round via
        # label propagation to the component minimum
        lab = np.arange(n)
        a, b = edges[:, 0], edges[:, 1]
        while True:
            mn = np.minimum(lab[a], lab[b])
            new = lab.copy()
            np.minimum.at(new, a, mn)
            np.minimum.at(new, b, mn)
            new = new[new]
            if np.array_equal(new, lab):
                break
            lab = new
        assert np.array_equal(got, lab), trial


def test_criterion_6_early_exit_core_flags_50_instances():
    """acceptance.cpp:235-255: early-exit core marking equals exhaustive
    counting (seeds 600..649, random_instance(seed, 50, 1500), minpts 2 -> 5)."""
    for seed in range(600, 650):
        ds, eps, mp = Dataset.random_instance(seed, 50, 1500)
        if mp == 2:
            mp = 5
        got = tb.cluster(ds, eps, mp, FD)
        want = oracle.dbscan(ds.coords(), eps, mp, 2)
        assert np.array_equal(got.core_flags, want["core"]), seed


def test_criterion_7_dense_cells_exact_and_fewer_evaluations():
    """acceptance.cpp:257-292: in the DEVICE grid every pair of a dense cell
    is within eps, and DenseBox never computes more distances than FDBSCAN;
    lattices (40^2 / 12^3 at spacing 0.1) + random_instance seeds 700..711."""
    cases = [(Dataset.lattice(40, 2, 0.1), 0.5, 4), (Dataset.lattice(12, 3, 0.1), 0.6, 5)]
    for seed in range(700, 712):
        cases.append(Dataset.random_instance(seed, 500, 2000))
    with_dense = 0
    for ds, eps, mp in cases:
        c = ds.coords()
        g = tb.api.debug_grid(c, eps, mp)
        eps2 = np.float64(np.float32(eps)) ** 2
        for b, e in zip(g["begin"][g["dense"]], g["end"][g["dense"]]):
            m = c[g["perm"][b:e]].astype(np.float64)
            d = m[:, None, :] - m[None, :, :]
            assert ((d * d).sum(-1) <= eps2).all()
        if not g["dense"].any():
            continue
        with_dense += 1
        fd = tb.cluster(ds, eps, mp, FD)
        db = tb.cluster(ds, eps, mp, DB)
        assert db.stats["distance_evaluations"] <= fd.stats["distance_evaluations"]
    assert with_dense >= 3


def test_criterion_8_deterministic_20_instances():
    """acceptance.cpp:294-318: cores, noise and core labels identical run to
    run (seeds 800..819, random_instance(seed, 200, 2000)) and equal to the
    single-threaded reference semantics (the oracle)."""
    for seed in range(800, 820):
        ds, eps, mp = Dataset.random_instance(seed, 200, 2000)
        c = ds.coords()
        for algo in (FD, DB):
            a = tb.cluster(ds, eps, mp, algo)
            b = tb.cluster(ds, eps, mp, algo)
            assert_parity(b.labels, b.core_flags, a.labels, a.core_flags, f"{seed} rerun")
            want = oracle.dbscan(c, eps, mp, int(algo))
            assert_parity(a.labels, a.core_flags, want["labels"], want["core"], f"{seed} oracle")


def test_criterion_9_performance_smoke():
    """acceptance.cpp:320-349: 10^6 points (100 blobs of 10^4, separation 10,
    sigma 1, eps 0.12, minpts 5) end to end under 60 s with 85-99% clustered,
    and 4x the points costing < 8x the time."""
    def timed(n, clustered=None):
        ds = Dataset.blobs(n // 10000, 10000, 2, 10.0, 1.0, 7)
        tb.cluster(ds, 0.12, 5, FD)  # warm
        t0 = time.perf_counter()
        r = tb.cluster(ds, 0.12, 5, FD)
        dt = time.perf_counter() - t0
        return dt, 1.0 - r.stats["noise_count"] / n

    small, _ = timed(250_000)
    large, clustered = timed(1_000_000)
    assert large < 60.0 and 0.85 < clustered < 0.99
    assert large / small < 8.0
