"""Parity of the sm_100a path against the oracle / the reference (the gates of
SURVEY.md §8): core flags bit-exact, noise set exact, core labels EQUAL (the
minimum core index of the cluster), every border valid, pair_resolutions and
distance_evaluations exact. Everything goes through the C ABI."""
import numpy as np
import pytest

import paper_2103_05162_b200 as tb
from oracle import oracle, ref
from paper_2103_05162_b200 import Algorithm, Dataset, Status, TreeclustError

from ._util import SEEDS, assert_parity, brute_pair_count, golden_run, instance, npz

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _device():
    assert tb.device_count() > 0, "GPU tests need a CUDA device (no CPU fallback exists)"


def run(coords, eps, minpts, algo, cap=0):
    return tb.cluster(Dataset.from_array(coords), eps, minpts, Algorithm(algo), oracle_cap=cap)


def check_against_oracle(coords, eps, minpts, algo, tag=""):
    got = run(coords, eps, minpts, algo)
    want = oracle.dbscan(coords, eps, minpts, algo)
    assert_parity(got.labels, got.core_flags, want["labels"], want["core"], tag)
    ok, msg = oracle.check_equivalence(coords, eps, got.labels, got.core_flags, want["labels"],
                                       want["core"])
    assert ok, f"{tag}: {msg}"
    if algo < 2:
        for k in ("pair_resolutions", "distance_evaluations", "cluster_count", "core_count",
                  "noise_count", "preprocess_skipped"):
            assert got.stats[k] == want["stats"][k], (tag, k, got.stats[k], want["stats"][k])
    if algo == 1:
        assert got.stats["dense_point_fraction"] == want["stats"]["dense_point_fraction"]
    return got, want


# ---------------- golden instances (reference outputs, committed) ----------------
@pytest.mark.parametrize("seed", SEEDS)
def test_golden_instances(seed):
    _, coords, eps, mp = instance(seed)
    db = npz("dbscan.npz")
    for algo in (0, 1, 2):
        want = golden_run(db, seed, algo)
        got = run(coords, eps, mp, algo)
        assert_parity(got.labels, got.core_flags, want["labels"], want["core"], f"{seed}/{algo}")
        ok, msg = oracle.check_equivalence(coords, eps, got.labels, got.core_flags,
                                           want["labels"], want["core"])
        assert ok, msg
        if algo == 2:  # brute force is deterministic end to end
            assert np.array_equal(got.labels, want["labels"])
        else:
            for k, v in want["counters"].items():
                assert got.stats[k] == v, (seed, algo, k)
        if algo == 1:
            assert got.stats["dense_point_fraction"] == want["dense_fraction"]


@pytest.mark.parametrize("seed", range(100, 140))
def test_more_random_instances_against_oracle(seed):
    import paper_2103_05162_b200 as t

    ds, eps, mp = t.Dataset.random_instance(seed, 50, 2500)
    for algo in (0, 1, 2):
        check_against_oracle(ds.coords(), eps, mp, algo, f"seed {seed} algo {algo}")


# ---------------- stage probes vs the reference's own accessors ----------------
def test_device_bvh_is_the_reference_tree():
    g = npz("bvh.npz")
    for name in ("two", "dups", "rand2", "rand3", "clump3"):
        t = tb.api.debug_point_bvh(g[f"{name}_pts"])
        for k in ("leaf_ids", "left", "right", "max_rank", "boxes"):
            assert np.array_equal(t[k], g[f"{name}_{k}"]), (name, k)
    rng = np.random.default_rng(5)
    for d in (2, 3):
        pts = np.concatenate([rng.normal(0, 1, (30000, d)), rng.uniform(-5, 5, (20000, d)),
                              np.repeat(rng.normal(0, 1, (10, d)), 50, axis=0)]).astype(np.float32)
        t = tb.api.debug_point_bvh(pts)
        w = oracle.point_bvh(pts)
        for k in ("leaf_ids", "left", "right", "max_rank", "boxes"):
            assert np.array_equal(t[k], w[k]), (d, k)


def test_device_grid_golden():
    """Device build_grid (REF dense_grid.cpp:23-77) == the reference's grid.npz:
    perm, cell of every point, cell ids, ranges and dense flags."""
    g = npz("grid.npz")
    for s in (3, 8):
        _, coords, eps, mp = instance(s)
        got = tb.api.debug_grid(coords, eps, mp)
        for k in ("perm", "cell_of_point", "cell_id", "begin", "end", "dense"):
            assert np.array_equal(got[k], g[f"s{s}_{k}"]), (s, k)


def _stage_inputs():
    rng = np.random.default_rng(12)
    lattice = np.stack(np.meshgrid(np.arange(150), np.arange(150)), -1).reshape(-1, 2)
    yield "taxi2d", Dataset.taxi_like(200_000, seed=3).coords(), 0.001, 40
    yield "blobs3d", Dataset.blobs(20, 8000, 3, 1.0, 0.15, 9).coords(), 0.2, 30
    yield "lattice2d", (lattice * 0.01 + rng.uniform(-0.004, 0.004, lattice.shape)).astype(
        np.float32), 0.1, 20
    yield "sparse3d", Dataset.hacc_like(150_000, seed=4).coords(), 0.042, 5


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_device_grid_and_mixed_tree_are_the_reference():
    """Stage by stage against the compiled reference (not only end to end):
    the device grid equals build_grid and the DenseBox tree over the mixed
    primitives equals the reference's Bvh (leaf kinds / ids per rank, node
    links, max ranks and boxes), node for node."""
    for name, c, eps, mp in _stage_inputs():
        got = tb.api.debug_grid(c, eps, mp)
        want = ref.build_grid(c, eps, mp)
        for k in ("perm", "cell_of_point", "cell_id", "begin", "end", "dense"):
            assert np.array_equal(got[k], want[k]), (name, k)
        t = tb.api.debug_mixed_bvh(c, eps, mp)
        w = ref.mixed_bvh(c, eps, mp)
        assert want["dense"].any() or name == "sparse3d", name
        for k in ("leaf_kind", "leaf_id", "left", "right", "max_rank", "boxes"):
            assert np.array_equal(t[k], w[k]), (name, k)


@pytest.mark.parametrize("d", [2, 3])
def test_morton_prefix_sort_fixup_and_fallback(d):
    """The build sorts Morton codes on their top bits and fixes equal-prefix
    groups afterwards (radix_sort_pairs_prefix); groups longer than kFixMax
    fall back to the full sort. Both must give the reference's tree."""
    rng = np.random.default_rng(17 + d)
    wide = rng.uniform(-5, 5, (40000, d))
    cases = {
        # many small groups at the cut (tight pairs / triples)
        "pairs": np.concatenate([wide, wide[:5000] + rng.normal(0, 1e-6, (5000, d))]),
        # one group of 600 coincident points: fallback
        "dups600": np.concatenate([wide, np.repeat(wide[:1], 600, axis=0)]),
        # 3000 distinct points inside one top-bits cell: fallback
        "clump": np.concatenate([wide, rng.normal(1.0, 1e-7, (3000, d))]),
        # groups just under the cap
        "dups200": np.concatenate([wide, np.repeat(wide[:20], 200, axis=0)]),
    }
    for name, pts in cases.items():
        pts = pts.astype(np.float32)
        t = tb.api.debug_point_bvh(pts)
        w = oracle.point_bvh(pts)
        for k in ("leaf_ids", "left", "right", "max_rank", "boxes"):
            assert np.array_equal(t[k], w[k]), (name, d, k)


def test_radix_sort_is_stable_and_exact():
    rng = np.random.default_rng(7)
    cases = [
        rng.integers(0, 2 ** 63, 1_000_003, dtype=np.uint64),
        rng.integers(0, 50, 300_000).astype(np.uint64) << np.uint64(40),  # heavy duplicates
        np.full(5000, 12345, np.uint64),  # all digits constant
        np.array([7], np.uint64),
        rng.integers(0, 2 ** 64 - 1, 100_000, dtype=np.uint64, endpoint=True),
    ]
    for keys in cases:
        ko, vo = tb.api.debug_sort_pairs(keys)
        order = np.argsort(keys, kind="stable")
        assert np.array_equal(vo, order)
        assert np.array_equal(ko, keys[order])


def test_device_union_find_matches_sequential_replay():  # REF acceptance criterion 5
    rng = np.random.default_rng(99)
    for trial in range(10):
        n = 10000
        edges = rng.integers(0, n, (100_000, 2)).astype(np.int32)
        got = tb.api.debug_union_find(edges, n)
        parent = np.arange(n)

        def find(i):
            while parent[i] != i:
                parent[i] = parent[parent[i]]
                i = parent[i]
            return i

        for a, b in edges:
            ra, rb = find(a), find(b)
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
        want = np.array([find(i) for i in range(n)])
        assert np.array_equal(got, want), trial
        assert np.array_equal(got, got[got])  # flattened


# ---------------- edge cases the reference tests ----------------
@pytest.mark.parametrize("algo", [0, 1, 2])
def test_single_and_pair(algo):
    one = run(np.array([[1, 1]], np.float32), 1.0, 2, algo)
    assert one.labels[0] == -1 and one.core_flags[0] == 0
    pair = run(np.array([[0, 0], [0.5, 0]], np.float32), 1.0, 2, algo)
    assert list(pair.labels) == [0, 0] and list(pair.core_flags) == [1, 1]


@pytest.mark.parametrize("algo", [0, 1, 2])
def test_degenerate_inputs(algo):
    cases = [
        (np.ones((3, 2), np.float32), 0.5, 3),                      # coincident points
        (np.ones((500, 3), np.float32), 0.5, 10),                   # one dense cell / 1-leaf tree
        (np.array([[5.0, y] for y in np.linspace(0, 1, 200)], np.float32), 0.01, 2),  # zero-width x
        (np.array([[0.9 * i, 0] for i in range(50)], np.float32), 1.0, 2),  # chain
        (np.array([[0, 0], [.1, 0], [0, .1], [5, 5], [5.1, 5], [5, 5.1]], np.float32), 0.2, 3),
        (np.random.default_rng(3).normal(0, 1e30, (400, 2)).astype(np.float32), 3e29, 3),
        (np.random.default_rng(4).uniform(-1e-30, 1e-30, (300, 3)).astype(np.float32), 1e-31, 4),
    ]
    for i, (c, eps, mp) in enumerate(cases):
        check_against_oracle(c, eps, mp, algo, f"case {i} algo {algo}")


@pytest.mark.parametrize("algo", [0, 1, 2])
def test_eps_boundary_is_the_exact_fp64_predicate(algo):
    """Pairs at, one ulp inside and one ulp outside eps: fp32 arithmetic would
    get some of these wrong; the fp64 chain of geometry.hpp:72-79 decides."""
    eps = np.float32(0.1)
    pts = [[0.0, 0.0]]
    x = np.float32(0.1)
    for dx in (x, np.nextafter(x, np.float32(0)), np.nextafter(x, np.float32(1))):
        base = np.float32(len(pts) * 10.0)
        pts += [[base, 0.0], [base + dx, 0.0]]
    # diagonal pairs whose squared distance is within 1e-7 relative of eps^2
    rng = np.random.default_rng(11)
    for _ in range(300):
        a = rng.uniform(100, 200, 2).astype(np.float32)
        ang = rng.uniform(0, 2 * np.pi)
        b = (a + np.array([np.cos(ang), np.sin(ang)]) * float(eps) * (1 + rng.normal(0, 1e-7))).astype(np.float32)
        pts += [a.tolist(), b.tolist()]
    c = np.array(pts, np.float32)
    got, want = check_against_oracle(c, float(eps), 2, algo, f"boundary algo {algo}")
    if algo == 0:
        assert got.stats["pair_resolutions"] == brute_pair_count(c, float(eps))


def test_invalid_inputs_return_status_codes():
    c = np.random.default_rng(0).uniform(0, 1000, (1000, 3)).astype(np.float32)
    with pytest.raises(TreeclustError) as e:  # grid would exceed 2^62 cells
        tb.cluster(Dataset.from_array(c), 1e-12, 5, Algorithm.DENSEBOX)
    assert e.value.status == Status.INVALID_ARGUMENT
    import torch

    x = torch.tensor([[0.0, 0.0], [float("nan"), 1.0]], device="cuda")
    for algo in (0, 1, 2):
        with pytest.raises(TreeclustError) as e:
            tb.cluster_device(x, 1.0, 2, Algorithm(algo), stats=True)
        assert e.value.status == Status.INVALID_ARGUMENT
    with pytest.raises(TreeclustError) as e:
        tb.cluster(Dataset.from_array(c), 1.0, 5, Algorithm.BRUTEFORCE, oracle_cap=500)
    assert e.value.status == Status.CAP_EXCEEDED
    # a library error leaves the device usable
    ok = tb.cluster(Dataset.from_array(c[:100]), 50.0, 3)
    assert ok.labels.shape == (100,)


def test_verify_passes():  # REF test_capi.cpp:142-150
    ds = Dataset.blobs(3, 100, 2, 10.0, 0.6, 31)
    st, report = tb.verify(ds, 1.2, 5)
    assert st == Status.OK, report
    assert "PASS" in report and "FAIL" not in report
    big = Dataset.blobs(5, 4000, 3, 10.0, 0.6, 3)
    st, report = tb.verify(big, 0.3, 5)
    assert st == Status.OK and "skipped" in report, report


def test_device_api_matches_host_api():
    import torch

    ds = Dataset.blobs(10, 5000, 3, 3.0, 0.5, 9)
    c = ds.coords()
    for algo, mp in ((0, 5), (1, 5), (0, 2), (1, 2)):
        host = tb.cluster(ds, 0.2, mp, Algorithm(algo))
        lab, core, st = tb.cluster_device(torch.from_numpy(c).cuda(), 0.2, mp, Algorithm(algo),
                                          stats=True)
        assert_parity(lab.cpu().numpy(), core.cpu().numpy(), host.labels, host.core_flags)
        assert st["pair_resolutions"] == host.stats["pair_resolutions"]


# ---------------- medium / full size against the compiled reference ----------------
@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("algo", [0, 1])
def test_c1_blobs_1m_against_reference(algo):
    """C1: 2D Gaussian blobs, 1M points, eps 0.01, minpts 5 (BASELINE configs[0])."""
    ds = Dataset.blobs(100, 10000, 2, 0.8333333, 0.08333333, 7)
    c = ds.coords()
    got = tb.cluster(ds, 0.01, 5, Algorithm(algo))
    want = ref.dbscan(c, 0.01, 5, algo, threads=0)
    assert_parity(got.labels, got.core_flags, want["labels"], want["core"], "C1")
    ok, msg = ref.check_equivalence(c, 0.01, 5, got.labels, got.core_flags, want["labels"],
                                    want["core"])
    assert ok, msg
    for k in ("pair_resolutions", "distance_evaluations", "cluster_count", "core_count",
              "noise_count"):
        assert got.stats[k] == want["stats"][k], k


_FULL = {}


def _full_input(name):
    """The §8d inputs at full size, from the oracle's generator (sha256 pinned in
    tests/golden/bench_inputs.json; byte-identical to tcg_generate_*)."""
    if name not in _FULL:
        _FULL.clear()  # hold one full-size input at a time
        _FULL[name] = oracle.hacc_like(37_000_000) if name == "hacc" else \
            oracle.taxi_like(80_000_000)
    return _FULL[name]


def _assert_reference_parity(got, want, coords, eps, minpts, tag, counters=True):
    """SURVEY §8 gates at full size against the compiled reference: core flags
    bit-exact, noise set exact, core labels EQUAL, every border label valid
    (reference check_equivalence semantics, device border check), and the
    reference's own counters."""
    import torch

    assert_parity(got.labels, got.core_flags, want["labels"], want["core"], tag)
    x = torch.from_numpy(coords).cuda()
    bad = tb.api.first_bad_border(x, eps, torch.from_numpy(got.labels).cuda(),
                                  torch.from_numpy(got.core_flags).cuda())
    assert bad < 0, f"{tag}: invalid border label at point {bad}"
    for k in ("cluster_count", "core_count", "noise_count", "preprocess_skipped"):
        assert got.stats[k] == want["stats"][k], (tag, k, got.stats[k], want["stats"][k])
    if counters:
        for k in ("pair_resolutions", "distance_evaluations"):
            assert got.stats[k] == want["stats"][k], (tag, k, got.stats[k], want["stats"][k])
        assert got.stats["dense_point_fraction"] == want["stats"]["dense_point_fraction"], tag


@pytest.mark.slow
@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_c2_hacc_37m_against_reference():
    """C2 at full size (BASELINE configs[1], the bench workload): 37M HACC-like
    points, eps 0.042, minpts 2 — FDBSCAN AND DenseBox (north star: "minpts=2
    and minpts=100 ... core partition bit-exact vs the CPU reference") against
    the reference's FDBSCAN and DenseBox runs on the host cores."""
    c = _full_input("hacc")
    ds = Dataset.from_array(c)
    want = ref.dbscan(c, 0.042, 2, 0, threads=0)
    got = tb.cluster(ds, 0.042, 2, Algorithm.FDBSCAN)
    _assert_reference_parity(got, want, c, 0.042, 2, "C2 FDBSCAN")
    assert got.stats["pair_resolutions"] == 898_475_393
    # minpts == 2: no borders, so labels are fully determined
    assert np.array_equal(got.labels, want["labels"])
    want_db = ref.dbscan(c, 0.042, 2, 1, threads=0)
    assert np.array_equal(want_db["labels"], want["labels"])  # the reference agrees with itself
    got_db = tb.cluster(ds, 0.042, 2, Algorithm.DENSEBOX)
    _assert_reference_parity(got_db, want_db, c, 0.042, 2, "C2 DenseBox")
    assert np.array_equal(got_db.labels, want_db["labels"])


@pytest.mark.slow
@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_c3_hacc_37m_densebox_against_reference():
    """C3 at full size: 37M HACC-like points, eps 0.042, minpts 100, DenseBox
    (REF dbscan.cpp:110-200) against the reference's DenseBox run; our FDBSCAN
    on the same input must give the same core partition and noise set."""
    c = _full_input("hacc")
    ds = Dataset.from_array(c)
    want = ref.dbscan(c, 0.042, 100, 1, threads=0)
    got = tb.cluster(ds, 0.042, 100, Algorithm.DENSEBOX)
    _assert_reference_parity(got, want, c, 0.042, 100, "C3 DenseBox")
    assert want["stats"]["core_count"] == 4_243_007 and want["stats"]["cluster_count"] == 5000
    got_fd = tb.cluster(ds, 0.042, 100, Algorithm.FDBSCAN)
    _assert_reference_parity(got_fd, want, c, 0.042, 100, "C3 FDBSCAN", counters=False)
    again = tb.cluster(ds, 0.042, 100, Algorithm.DENSEBOX)  # determinism (acceptance crit. 8)
    assert np.array_equal(again.labels, got.labels)
    assert np.array_equal(again.core_flags, got.core_flags)
    for k, v in got.stats.items():
        assert k.endswith("_seconds") or again.stats[k] == v, k


@pytest.mark.slow
@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_c4_taxi_80m_densebox_against_reference():
    """C4 at full size: 80M 2D taxi-like points, eps 0.001, minpts 1000,
    DenseBox, against the reference's DenseBox run (counters included: the
    member-tree scans and primitive runs must reproduce the reference's
    member-by-member scans exactly)."""
    c = _full_input("taxi")
    want = ref.dbscan(c, 0.001, 1000, 1, threads=0)
    got = tb.cluster(Dataset.from_array(c), 0.001, 1000, Algorithm.DENSEBOX)
    _assert_reference_parity(got, want, c, 0.001, 1000, "C4 DenseBox")


@pytest.mark.slow
def test_c3_full_size_properties():
    """C3 on the device only: FDBSCAN and DenseBox agree exactly on cores /
    noise / core labels, and the result is identical run to run."""
    import torch

    x = torch.from_numpy(_full_input("hacc")).cuda()
    l0, c0, s0 = tb.cluster_device(x, 0.042, 100, Algorithm.FDBSCAN, stats=True)
    l1, c1, s1 = tb.cluster_device(x, 0.042, 100, Algorithm.DENSEBOX, stats=True)
    l2, c2, _ = tb.cluster_device(x, 0.042, 100, Algorithm.FDBSCAN, stats=True)
    assert torch.equal(c0, c1) and torch.equal(c0, c2)
    assert torch.equal(l0 == -1, l1 == -1)
    m = c0.bool()
    assert torch.equal(l0[m], l1[m]) and torch.equal(l0[m], l2[m])
    assert s0["core_count"] == s1["core_count"]


# ---------------- contained subtrees / member tree vs the reference ----------------
@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("case", ["taxi2d", "blobs3d", "lattice2d"])
def test_densebox_large_cells_exact_counters(case):
    """DenseBox with large dense cells (hundreds to thousands of members): the
    member-tree scans (first hit / minpts-th hit in member order) and the
    contained-subtree runs must reproduce the reference's counters exactly,
    together with the clustering itself."""
    if case == "taxi2d":
        c, eps, mp = Dataset.taxi_like(400_000, seed=3).coords(), 0.001, 300
    elif case == "blobs3d":
        c = Dataset.blobs(20, 15000, 3, 1.0, 0.15, 9).coords()
        eps, mp = 0.2, 150
    else:
        rng = np.random.default_rng(4)
        g = np.stack(np.meshgrid(np.arange(300), np.arange(300)), -1).reshape(-1, 2)
        c = (g * 0.01 + rng.uniform(-0.004, 0.004, g.shape)).astype(np.float32)
        eps, mp = 0.1, 20
    got = tb.cluster(Dataset.from_array(c), eps, mp, Algorithm.DENSEBOX)
    want = ref.dbscan(c, eps, mp, 1, threads=0)
    assert_parity(got.labels, got.core_flags, want["labels"], want["core"], case)
    for k in ("pair_resolutions", "distance_evaluations", "cluster_count", "core_count",
              "noise_count"):
        assert got.stats[k] == want["stats"][k], (case, k, got.stats[k], want["stats"][k])
    assert got.stats["dense_point_fraction"] > 0.2, case


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("minpts", [2, 7, 60])
def test_fdbscan_contained_runs_exact_counters(minpts):
    """FDBSCAN on dense clumps, where most pairs come from contained subtrees
    (rank runs): pair and distance counters and the clustering equal the
    reference's for the minpts == 2 path and the minpts > 2 path."""
    c = Dataset.blobs(30, 8000, 3, 1.0, 0.05, 13).coords()
    got = tb.cluster(Dataset.from_array(c), 0.03, minpts, Algorithm.FDBSCAN)
    want = ref.dbscan(c, 0.03, minpts, 0, threads=0)
    assert_parity(got.labels, got.core_flags, want["labels"], want["core"], f"fd{minpts}")
    for k in ("pair_resolutions", "distance_evaluations", "cluster_count", "core_count",
              "noise_count"):
        assert got.stats[k] == want["stats"][k], (minpts, k, got.stats[k], want["stats"][k])


def test_load_binary_device_matches_host_load(tmp_path):
    """§8f row f1: a .bin file streamed to the device equals tc_dataset_load's
    points; bad files fail like tc_dataset_load (TC_ERR_IO)."""
    import torch

    ds = Dataset.hacc_like(3_000_000, seed=5)  # > 2 staging chunks of 32 MiB
    path = str(tmp_path / "pts.bin")
    ds.save(path)
    x = tb.load_device(path)
    assert x.shape == (3_000_000, 3)
    assert torch.equal(x.cpu(), torch.from_numpy(Dataset.load(path).coords()))
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\x05\x00\x00\x00\x07\x00\x00\x00")  # dim 7
    with pytest.raises(TreeclustError) as e:
        tb.load_device(str(bad))
    assert e.value.status == Status.IO
    trunc = tmp_path / "trunc.bin"
    trunc.write_bytes(open(path, "rb").read()[:1000])
    with pytest.raises(TreeclustError) as e:
        tb.load_device(str(trunc))
    assert e.value.status == Status.IO


@pytest.mark.parametrize("minpts,top", [(2, False), (6, False), (2, True), (6, True)])
def test_keyed_and_local_context_label_in_keys(minpts, top):
    """tcg_cluster_keyed_device and the tcg_local_* context (the sharded
    path's local runs): with arbitrary unique keys, a cluster is labelled by
    the key of its minimum-key core, and the partition equals tc_cluster's.
    top: the keys run up to INT32_MAX (labels travel through the finalize
    entries untouched)."""
    import torch
    from paper_2103_05162_b200.shard import DeviceEngine

    c = Dataset.blobs(12, 3000, 3, 1.0, 0.12, 17).coords()
    eps = 0.09
    want = tb.cluster(Dataset.from_array(c), eps, minpts, Algorithm.FDBSCAN)
    rng = np.random.default_rng(3)
    base = 2**31 - 1 - 7 * (len(c) - 1) if top else 10**6
    keys = rng.permutation(np.arange(base, base + 7 * len(c), 7, dtype=np.int64)).astype(np.int32)
    assert not top or keys.max() == 2**31 - 1
    eng = DeviceEngine("cuda:0")
    x = torch.from_numpy(c).cuda()
    kd = torch.from_numpy(keys).cuda()
    core = want.core_flags.astype(bool)
    lab_w = want.labels
    # expected: key of the minimum-key core of each reference cluster
    best = {}
    for i in np.nonzero(core)[0]:
        best[lab_w[i]] = min(best.get(lab_w[i], 2**31), int(keys[i]))
    if minpts == 2:
        lab, cf = eng.cluster_keyed(x, kd, eps, minpts)
    else:
        ctx = eng.local(x, kd, eps)
        cf = ctx.core_flags(minpts)
        lab = ctx.cluster(cf)
        ctx.close()
    lab = lab.cpu().numpy()
    assert np.array_equal(cf.cpu().numpy(), want.core_flags)
    assert np.array_equal(lab == -1, lab_w == -1)
    for i in np.nonzero(core)[0]:
        assert lab[i] == best[lab_w[i]], i
    # borders: a core's cluster within eps (any valid claim)
    border = (~core) & (lab_w != -1)
    inv = {v: k for k, v in best.items()}
    for i in np.nonzero(border)[0]:
        assert lab[i] in inv, i


@pytest.mark.parametrize("minpts", [2, 5, 3000])
def test_massive_duplicates_and_flat_axis(minpts):
    """Stress of the contained-run paths: 1.5M copies of one point plus a flat
    (z = 0) uniform background. All copies form one cluster whose pair count is
    n(n-1)/2 (every pair of copies), counted exactly through rank runs."""
    rng = np.random.default_rng(8)
    dup = np.tile(np.array([[-5.0, -5.0, 0.0]], np.float32), (1_500_000, 1))
    bg = np.concatenate([rng.uniform(0, 100, (200_000, 2)), np.zeros((200_000, 1))], 1)
    c = np.concatenate([dup, bg.astype(np.float32)])
    eps = 0.05
    got = tb.cluster(Dataset.from_array(c), eps, minpts, Algorithm.FDBSCAN)
    nd = len(dup)
    assert (got.labels[:nd] == 0).all() and (got.core_flags[:nd] == 1).all()
    # background pairs: brute force on the sparse part only (no background
    # point is within eps of the duplicate point here)
    b = bg.astype(np.float32).astype(np.float64)
    assert np.sqrt(((b[:, :2] + 5.0) ** 2).sum(1)).min() > eps
    want_bg = tb.cluster(Dataset.from_array(bg.astype(np.float32)), eps, minpts, Algorithm.FDBSCAN)
    assert got.stats["pair_resolutions"] == nd * (nd - 1) // 2 + want_bg.stats["pair_resolutions"]
    assert np.array_equal(got.core_flags[nd:], want_bg.core_flags)
    lab = got.labels[nd:]
    wl = want_bg.labels
    assert np.array_equal(lab == -1, wl == -1)
    cm = want_bg.core_flags == 1
    assert np.array_equal(lab[cm], wl[cm] + nd)
    db = tb.cluster(Dataset.from_array(c), eps, minpts, Algorithm.DENSEBOX)
    assert np.array_equal(db.core_flags, got.core_flags)
    assert np.array_equal(db.labels[got.core_flags == 1], got.labels[got.core_flags == 1])


# ---------------- device check_equivalence (§8f row f2) ----------------
def test_device_check_equivalence_matches_reference_checker():
    """tcg_check_equivalence_device reports the same verdict and the same
    first-divergence index as the reference's check_equivalence
    (REF oracle.cpp:120-163) on a passing pair and on one corrupted pair per
    check (core flag, noise, core partition, border in a / in b)."""
    import torch

    ds, eps, mp = Dataset.random_instance(11, 3000, 3000)
    c = ds.coords()
    a = tb.cluster(ds, eps, 5, Algorithm.FDBSCAN)
    b = tb.cluster(ds, eps, 5, Algorithm.DENSEBOX)
    x = torch.from_numpy(c).cuda()

    def both(la, ca, lb, cb):
        dev = tb.api.check_equivalence_device(
            x, eps, *(torch.from_numpy(np.ascontiguousarray(v)).cuda() for v in (la, ca, lb, cb)))
        ok, msg = oracle.check_equivalence(c, eps, la, ca, lb, cb)
        if ref.available():
            rok, rmsg = ref.check_equivalence(c, eps, 5, la, ca, lb, cb)
            assert (rok, rmsg) == (ok, msg)
        assert (dev[0] == 0) == ok and dev[2] == msg, (dev, msg)
        return dev[0]

    assert both(a.labels, a.core_flags, b.labels, b.core_flags) == 0
    core = np.nonzero(a.core_flags)[0]
    border = np.nonzero((a.core_flags == 0) & (a.labels != -1))[0]
    noise = np.nonzero(a.labels == -1)[0]
    assert len(core) > 10 and len(border) > 0 and len(noise) > 0
    cb = b.core_flags.copy(); cb[core[7]] = 0
    assert both(a.labels, a.core_flags, b.labels, cb) == 1
    lb = b.labels.copy(); lb[noise[3]] = b.labels[core[0]]
    assert both(a.labels, a.core_flags, lb, b.core_flags) == 2
    # merge two clusters of b: a core partition difference at the first core
    # of the second cluster
    lab_ids = np.unique(b.labels[core])
    assert len(lab_ids) >= 2
    lb = b.labels.copy(); lb[lb == lab_ids[1]] = lab_ids[0]
    assert both(a.labels, a.core_flags, lb, b.core_flags) == 3
    # relabel a border into a cluster none of its cores reach
    la = a.labels.copy()
    far = [l for l in np.unique(a.labels[core]) if l != la[border[0]]][0]
    la[border[0]] = far
    assert both(la, a.core_flags, b.labels, b.core_flags) == 4
    assert both(a.labels, a.core_flags, la, a.core_flags) == 5
    # bijective relabeling of a core partition (arbitrary label values) passes
    perm = {l: 10_000_000 + 3 * k for k, l in enumerate(np.unique(b.labels))}
    perm[-1] = -1
    lb = np.array([perm[v] for v in b.labels], np.int32)
    assert both(a.labels, a.core_flags, lb, b.core_flags) == 0


def test_device_morton_codes_golden():
    """Device Morton codes (the tree build's quantization, REF
    geometry.hpp:132-156) equal the reference's codes in morton.npz."""
    import ctypes as C
    import torch
    from paper_2103_05162_b200._lib import lib

    g = npz("morton.npz")
    for d in (2, 3):
        pts = torch.from_numpy(g[f"pts{d}"]).cuda()
        lo = np.ascontiguousarray(g[f"lo{d}"], np.float32)
        hi = np.ascontiguousarray(g[f"hi{d}"], np.float32)
        out = torch.empty(pts.shape[0], dtype=torch.int64, device="cuda")
        st = lib.tcg_morton_codes_device(C.c_void_p(pts.data_ptr()), pts.shape[0], d,
                                         lo.ctypes.data_as(C.POINTER(C.c_float)),
                                         hi.ctypes.data_as(C.POINTER(C.c_float)),
                                         C.c_void_p(out.data_ptr()),
                                         C.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert st == 0
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64), g[f"codes{d}"]), d


def test_fof_action_queue_never_overflows():
    """Regression: with eps near the cloud's extent nearly every child is a
    contained run, lanes queue two union actions per step, and the per-warp
    action queue must be drained below 32 after every step (it overflowed
    into the next warp's queue before; intermittent illegal address). Many
    repetitions, each against the oracle's labels."""
    c = oracle.hacc_like(20_000)
    ds = Dataset.from_array(c)
    want = oracle.dbscan(c, 0.3, 2, 0)
    for _ in range(40):
        got = tb.cluster(ds, 0.3, 2, Algorithm.FDBSCAN)
        assert np.array_equal(got.labels, want["labels"])
        assert np.array_equal(got.core_flags, want["core"])
        assert got.stats["pair_resolutions"] == want["stats"]["pair_resolutions"]


def test_randomized_stress_against_oracle():
    """300 random clouds (blobs, uniform, heavy duplicates, near-lattices;
    2D/3D) with eps from 1e-4 of the extent to beyond it and minpts 2..64,
    all three algorithms through tc_cluster and the device entry, against
    the oracle (tools/stress.py; a 10-minute run of it: 45 697 cases, 0
    differences)."""
    import os
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "tools"))
    import stress

    runs, bad = stress.run(600.0, max_runs=300, seed=2024, verbose=False)
    assert runs == 300 and not bad, bad[:5]


# ---------------- stream-ordered FDBSCAN: CUDA-graph capture ----------------
@pytest.mark.parametrize("minpts,dup,dim", [(2, 0, 3), (5, 0, 3), (2, 3000, 3), (5, 3000, 3),
                                            (2, 0, 2), (5, 3000, 2)])
def test_fdbscan_captured_in_cuda_graph(minpts, dup, dim):
    """tcg_cluster_device_async (FDBSCAN) never synchronizes the host, so one
    call captures into a CUDA graph; replays on new coordinates (copied into
    the captured input buffer) equal eager runs. dup > 256 coincident points
    make the Morton prefix sort take its device-guarded fallback."""
    import torch

    rng = np.random.default_rng(minpts + dup)

    def cloud(seed):
        ds = Dataset.blobs(12, 4000, dim, 4.0, 0.4, seed)
        c = ds.coords()
        if dup:
            c[:dup] = c[dup]  # one point repeated dup + 1 times
        return torch.from_numpy(c).cuda()

    x = cloud(1)
    n = x.shape[0]
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    core = torch.empty(n, dtype=torch.uint8, device="cuda")
    status = torch.full((1,), 77, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):  # warm-up (lazy pool / attribute setup) off the capture
        tb.cluster_device_async(x, 0.15, minpts, Algorithm.FDBSCAN, labels, core, status, s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
        tb.cluster_device_async(x, 0.15, minpts, Algorithm.FDBSCAN, labels, core, status, s)
    for seed in (2, 3, 4):
        new = cloud(seed + int(rng.integers(1000)))
        x.copy_(new)
        status.fill_(77)
        g.replay()
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        want_l, want_c, _ = tb.cluster_device(new, 0.15, minpts, Algorithm.FDBSCAN, stats=True)
        torch.cuda.synchronize()
        assert torch.equal(core, want_c)
        cm = core == 1  # core labels are deterministic (min core index); borders valid
        assert torch.equal(labels[cm], want_l[cm]), seed
        assert torch.equal(labels == -1, want_l == -1), seed
        ref_run = oracle.dbscan(new.cpu().numpy(), 0.15, minpts, 0) if n <= 50000 else None
        if ref_run is not None:
            assert_parity(labels.cpu().numpy(), core.cpu().numpy(), ref_run["labels"],
                          ref_run["core"], f"graph {seed}")


def test_async_status_reports_nonfinite_on_device():
    import torch

    c = np.random.default_rng(3).uniform(0, 10, (5000, 3)).astype(np.float32)
    for bad in (0, 4321, 4999):
        x = torch.from_numpy(c.copy()).cuda()
        x[bad, 1] = float("nan") if bad % 2 == 0 else float("inf")
        lab, core, st = tb.cluster_device_async(x, 0.5, 3)
        torch.cuda.synchronize()
        assert int(st.item()) == int(Status.INVALID_ARGUMENT)
        assert (lab == -1).all() and (core == 0).all()
        with pytest.raises(TreeclustError) as e:
            tb.cluster_device(x, 0.5, 3, stats=True)
        assert e.value.status == Status.INVALID_ARGUMENT
    # all points non-finite: still no traversal work, status set
    x = torch.full((100000, 3), float("nan"), device="cuda")
    lab, core, st = tb.cluster_device_async(x, 0.5, 2)
    torch.cuda.synchronize()
    assert int(st.item()) == int(Status.INVALID_ARGUMENT) and (lab == -1).all()
    # a clean run afterwards reports OK and matches the host API
    x = torch.from_numpy(c).cuda()
    lab, core, st = tb.cluster_device_async(x, 0.5, 3)
    torch.cuda.synchronize()
    assert int(st.item()) == int(Status.OK)
    host = tb.cluster(Dataset.from_array(c), 0.5, 3)
    assert_parity(lab.cpu().numpy(), core.cpu().numpy(), host.labels, host.core_flags)
    for algo in (1, 2):  # the other algorithms write the status too
        lab, core, st = tb.cluster_device_async(x, 0.5, 3, Algorithm(algo))
        torch.cuda.synchronize()
        assert int(st.item()) == int(Status.OK)


def test_capture_of_a_synchronizing_call_is_refused_cleanly():
    """DenseBox / brute force (and stats read-backs) synchronize the host, so on
    a capturing stream they return INVALID_ARGUMENT before enqueuing anything:
    the capture stays valid and the FDBSCAN call captured next replays."""
    import torch

    c = Dataset.blobs(4, 3000, 3, 4.0, 0.4, 21).coords()
    x = torch.from_numpy(c).cuda()
    s = torch.cuda.Stream()
    lab = torch.empty(len(c), dtype=torch.int32, device="cuda")
    core = torch.empty(len(c), dtype=torch.uint8, device="cuda")
    st = torch.empty(1, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        tb.cluster_device_async(x, 0.2, 5, Algorithm.FDBSCAN, lab, core, st, s)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s, capture_error_mode="relaxed"):
        for algo in (Algorithm.DENSEBOX, Algorithm.BRUTEFORCE):
            with pytest.raises(TreeclustError) as e:
                tb.cluster_device_async(x, 0.2, 5, algo, lab, core, st, s)
            assert e.value.status == Status.INVALID_ARGUMENT
        with pytest.raises(TreeclustError) as e:
            tb.cluster_device(x, 0.2, 5, Algorithm.FDBSCAN, lab, core, s, stats=True)
        assert e.value.status == Status.INVALID_ARGUMENT
        tb.cluster_device_async(x, 0.2, 5, Algorithm.FDBSCAN, lab, core, st, s)
    lab.fill_(-7)
    g.replay()
    torch.cuda.synchronize()
    host = tb.cluster(Dataset.from_array(c), 0.2, 5)
    assert int(st.item()) == 0
    assert_parity(lab.cpu().numpy(), core.cpu().numpy(), host.labels, host.core_flags)
