"""Pins the checker: the C restatement (oracle/tc_oracle.c) against the
reference's own known-answer tests (REF tests/test_*.cpp), against golden
vectors produced by running the reference (tests/golden/), and — when the
compiled reference oracle/_ref is present — against the reference itself."""
import numpy as np
import pytest

from oracle import oracle, ref

from ._util import SEEDS, assert_parity, brute_pair_count, golden_run, instance, npz


# ---------------- Morton (REF tests/test_geometry.cpp:80-132) ----------------
def morton_bitwise(p, lo, hi):
    """testutil::morton_reference (REF tests/test_util.hpp:89-100)."""
    dim = len(p)
    bits = 31 if dim == 2 else 21
    code = 0
    for a in range(dim):
        w = float(hi[a]) - float(lo[a])
        if w <= 0:
            q = 0
        else:
            t = max((float(p[a]) - float(lo[a])) / w, 0.0)
            q = min(int(t * float(1 << bits)), (1 << bits) - 1)
        for b in range(bits):
            code |= ((q >> b) & 1) << (b * dim + a)
    return code


def test_morton_known_answers():
    lo, hi = np.zeros(3, np.float32), np.ones(3, np.float32)
    assert oracle.morton_codes(np.zeros((1, 2), np.float32), lo[:2], hi[:2])[0] == 0
    assert int(oracle.morton_codes(np.ones((1, 2), np.float32), lo[:2], hi[:2])[0]) == (1 << 62) - 1
    assert int(oracle.morton_codes(np.ones((1, 3), np.float32), lo, hi)[0]) == (1 << 63) - 1
    # zero-width axis normalizes to 0 (REF test_geometry.cpp:96-102)
    assert oracle.morton_codes(np.array([[0, 5]], np.float32), [0, 5], [1, 5])[0] == 0


def test_morton_golden_and_bitwise():
    g = npz("morton.npz")
    for d in (2, 3):
        codes = oracle.morton_codes(g[f"pts{d}"], g[f"lo{d}"], g[f"hi{d}"])
        assert np.array_equal(codes, g[f"codes{d}"])
        for p, c in zip(g[f"pts{d}"][:100], codes[:100]):
            assert int(c) == morton_bitwise(p, g[f"lo{d}"], g[f"hi{d}"])


# ---------------- BVH (REF tests/test_bvh.cpp:82-202) ----------------
def test_bvh_golden_trees():
    g = npz("bvh.npz")
    for name in ("two", "dups", "rand2", "rand3", "clump3"):
        t = oracle.point_bvh(g[f"{name}_pts"])
        for k in ("leaf_ids", "left", "right", "max_rank", "boxes"):
            assert np.array_equal(t[k], g[f"{name}_{k}"]), (name, k)


def test_bvh_two_primitives_known_answer():
    t = oracle.point_bvh(np.array([[0, 0], [3, 1]], np.float32))
    assert np.array_equal(t["boxes"][0], [0, 0, 0, 3, 1, 0]) and t["max_rank"][0] == 1


def test_bvh_recursive_containment():
    rng = np.random.default_rng(101)
    for d in (2, 3):
        pts = rng.uniform(0, 10, (5000, d)).astype(np.float32)
        t = oracle.point_bvh(pts)
        seen = np.zeros(len(pts), int)

        def walk(node):
            mr = -1
            for child in (t["left"][node], t["right"][node]):
                if child < 0:
                    r = ~child
                    seen[r] += 1
                    p = pts[t["leaf_ids"][r]]
                    assert np.all(t["boxes"][node][:d] <= p) and np.all(p <= t["boxes"][node][3:3 + d])
                    mr = max(mr, r)
                else:
                    sub = walk(child)
                    assert t["max_rank"][child] == sub
                    assert np.all(t["boxes"][node][:d] <= t["boxes"][child][:d])
                    mr = max(mr, sub)
            return mr

        import sys
        sys.setrecursionlimit(10000)
        assert walk(0) == len(pts) - 1
        assert np.all(seen == 1)


# ---------------- driver known answers (REF tests/test_dbscan.cpp) ----------------
@pytest.mark.parametrize("algo", [0, 1])
def test_single_point_is_noise(algo):
    r = oracle.dbscan(np.array([[1, 1]], np.float32), 1.0, 2, algo)
    assert r["labels"][0] == -1 and r["core"][0] == 0


@pytest.mark.parametrize("algo", [0, 1])
def test_pair_minpts2(algo):
    r = oracle.dbscan(np.array([[0, 0], [0.5, 0]], np.float32), 1.0, 2, algo)
    assert r["stats"]["preprocess_skipped"] == 1
    assert list(r["core"]) == [1, 1] and list(r["labels"]) == [0, 0]
    assert r["stats"]["cluster_count"] == 1


def test_two_triangles_roots():
    pts = np.array([[0, 0], [.1, 0], [0, .1], [5, 5], [5.1, 5], [5, 5.1]], np.float32)
    r = oracle.dbscan(pts, 0.2, 3, 0)
    assert set(r["labels"].tolist()) == {0, 3}


def test_chain_is_one_cluster():
    pts = np.array([[0.9 * i, 0] for i in range(50)], np.float32)
    assert np.all(oracle.dbscan(pts, 1.0, 2, 0)["labels"] == 0)


def test_duplicates_core_at_minpts3():
    r = oracle.dbscan(np.ones((3, 2), np.float32), 0.5, 3, 0)
    assert np.all(r["core"] == 1)


@pytest.mark.parametrize("algo", [0, 1])
def test_bridging_border_joins_exactly_one(algo):  # REF test_dbscan.cpp:138-165
    xs = [-0.75] + [-1.05 - 0.1 * i for i in range(4)] + [0.75] + [1.05 + 0.1 * i for i in range(4)] + [0.0]
    pts = np.array([[x, 0] for x in xs], np.float32)
    r = oracle.dbscan(pts, 1.0, 5, algo)
    assert r["stats"]["cluster_count"] == 2 and r["core"][10] == 0
    assert (r["labels"][10] == r["labels"][0]) != (r["labels"][10] == r["labels"][5])


def test_densebox_adjacent_cells_and_border_claim():  # REF test_densebox.cpp:179-210
    pts = np.array([[0.1 + 0.01 * i, 0.1] for i in range(4)] + [[0.9 + 0.01 * i, 0.1] for i in range(4)],
                   np.float32)
    r = oracle.dbscan(pts, 1.0, 4, 1)
    assert r["stats"]["dense_point_fraction"] == 1.0
    assert np.all(r["core"] == 1) and np.all(r["labels"] == r["labels"][0])
    pts = np.array([[0.15 * i, 0] for i in range(5)] + [[1.55, 0]], np.float32)
    r = oracle.dbscan(pts, 1.0, 5, 1)
    assert r["core"][5] == 0 and r["labels"][5] == r["labels"][0]


def test_densebox_fewer_distance_evaluations_on_lattice():  # REF test_densebox.cpp:223-231
    xs, ys = np.meshgrid(np.arange(40) * 0.1, np.arange(40) * 0.1, indexing="xy")
    pts = np.stack([xs.ravel(), ys.ravel()], 1).astype(np.float32)
    fd = oracle.dbscan(pts, 0.5, 4, 0)
    db = oracle.dbscan(pts, 0.5, 4, 1)
    assert db["stats"]["dense_point_fraction"] > 0
    assert db["stats"]["distance_evaluations"] < fd["stats"]["distance_evaluations"]


def test_capi_three_algorithms_identical_labels():  # REF test_capi.cpp:103-129
    import paper_2103_05162_b200 as tb

    pts = tb.Dataset.blobs(3, 80, 2, 20.0, 0.5, 21).coords()
    runs = [oracle.dbscan(pts, 1.5, 5, a) for a in (0, 1, 2)]
    assert all(r["stats"]["cluster_count"] == 3 for r in runs)
    assert np.array_equal(runs[0]["labels"], runs[1]["labels"])
    assert np.array_equal(runs[0]["labels"], runs[2]["labels"])


def test_invalid_arguments_rejected():
    with pytest.raises(ValueError):
        oracle.dbscan(np.zeros((2, 2), np.float32), -1.0, 2, 0)
    with pytest.raises(ValueError):
        oracle.dbscan(np.zeros((2, 2), np.float32), 1.0, 1, 0)


# ---------------- golden dbscan runs (reference, threads = 1) ----------------
@pytest.mark.parametrize("seed", SEEDS)
def test_oracle_matches_reference_golden(seed):
    _, coords, eps, mp = instance(seed)
    db = npz("dbscan.npz")
    for algo in (0, 1, 2):
        want = golden_run(db, seed, algo)
        got = oracle.dbscan(coords, eps, mp, algo)
        # single-threaded: every label, border ones included, is deterministic
        assert np.array_equal(got["labels"], want["labels"]), (seed, algo)
        assert np.array_equal(got["core"], want["core"]), (seed, algo)
        if algo < 2:
            for k, v in want["counters"].items():
                assert got["stats"][k] == v, (seed, algo, k)
        if algo == 1:
            assert got["stats"]["dense_point_fraction"] == want["dense_fraction"]


def test_pair_resolutions_equal_brute_pair_count():  # REF acceptance criterion 3
    for seed in (2, 5, 11):
        _, coords, eps, mp = instance(seed)
        assert oracle.dbscan(coords, eps, mp, 0)["stats"]["pair_resolutions"] == \
            brute_pair_count(coords, eps)


def test_grid_golden():
    g = npz("grid.npz")
    for s in (3, 8):
        _, coords, eps, mp = instance(s)
        got = oracle.build_grid(coords, eps, mp)
        for k in ("perm", "cell_of_point", "cell_id", "begin", "end", "dense"):
            assert np.array_equal(got[k], g[f"s{s}_{k}"]), (s, k)


def test_check_equivalence_detects_divergence():
    _, coords, eps, mp = instance(4)
    r = oracle.dbscan(coords, eps, mp, 0)
    ok, msg = oracle.check_equivalence(coords, eps, r["labels"], r["core"], r["labels"], r["core"])
    assert ok and msg == "PASS"
    core2 = r["core"].copy()
    core2[np.flatnonzero(core2)[0]] ^= 1
    ok, msg = oracle.check_equivalence(coords, eps, r["labels"], r["core"], r["labels"], core2)
    assert not ok and msg.startswith("core flags differ")
    lab2 = r["labels"].copy()
    cores = np.flatnonzero(r["core"])
    lab2[cores[-1]] = 10 ** 6  # split one core off its cluster
    ok, msg = oracle.check_equivalence(coords, eps, r["labels"], r["core"], lab2, r["core"])
    assert not ok


# ---------------- against the compiled reference itself ----------------
@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_oracle_matches_compiled_reference_more_seeds():
    for seed in range(25, 61):
        coords, eps, mp = ref.random_instance(seed, 50, 2000)
        for algo in (0, 1, 2):
            got = oracle.dbscan(coords, eps, mp, algo)
            want = ref.dbscan(coords, eps, mp, algo, threads=1)
            assert np.array_equal(got["labels"], want["labels"]), (seed, algo)
            assert np.array_equal(got["core"], want["core"]), (seed, algo)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_reference_threaded_core_labels_equal_oracle():
    """The reference with 8 threads: border labels may differ, core labels may
    not — the parity bar the GPU is held to."""
    for seed in (30, 31, 32):
        coords, eps, mp = ref.random_instance(seed, 500, 2000)
        for algo in (0, 1):
            want = oracle.dbscan(coords, eps, mp, algo)
            got = ref.dbscan(coords, eps, mp, algo, threads=8)
            assert_parity(got["labels"], got["core"], want["labels"], want["core"], f"{seed}/{algo}")


# ---------------- benchmark inputs ----------------
def test_oracle_bench_generators_match_product():
    """The oracle's HACC-like / taxi-like generators (used by bench.py's
    reference arm and the full-size parity tests, so that those never load the
    product library) are byte-identical to the product's."""
    import paper_2103_05162_b200 as tb

    for n, seed in ((150_000, 11), (777, 3)):
        assert np.array_equal(oracle.hacc_like(n, seed=seed),
                              tb.Dataset.hacc_like(n, seed=seed).coords())
        assert np.array_equal(oracle.taxi_like(n, seed=seed),
                              tb.Dataset.taxi_like(n, seed=seed).coords())
    with pytest.raises(ValueError):
        oracle.hacc_like(0)


def test_bench_inputs_full_size_sha():
    """C2/C3 (37M HACC-like) and C4 (80M taxi-like) inputs pinned by sha256."""
    import hashlib
    import json
    import os

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "bench_inputs.json")))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(oracle.hacc_like(37_000_000)) == g["hacc_like(37000000,L=36.8,0.23,seed=11)"]
    assert sha(oracle.taxi_like(80_000_000)) == g["taxi_like(80000000,seed=5)"]


def test_write_bin_loads_in_reference(tmp_path):
    """oracle.write_bin produces the reference's binary format (REF io.cpp:106-134)."""
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    import ctypes as C

    a = oracle.hacc_like(1000, seed=4)
    path = str(tmp_path / "p.bin")
    oracle.write_bin(path, a)
    L = ref.lib()
    L.tc_dataset_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
    L.tc_dataset_size.restype = C.c_int64
    L.tc_dataset_size.argtypes = [C.c_void_p]
    L.tc_dataset_coords.restype = C.POINTER(C.c_float)
    L.tc_dataset_coords.argtypes = [C.c_void_p]
    L.tc_dataset_free.argtypes = [C.c_void_p]
    ds = C.c_void_p()
    assert L.tc_dataset_load(path.encode(), 0, C.byref(ds)) == 0
    assert L.tc_dataset_size(ds) == 1000
    got = np.ctypeslib.as_array(L.tc_dataset_coords(ds), shape=(3000,)).reshape(1000, 3).copy()
    L.tc_dataset_free(ds)
    assert np.array_equal(got, a)


def test_check_equivalence_arbitrary_label_values():
    """Labels are arbitrary int32 values in check_equivalence (REF
    oracle.cpp:144-152 maps them through hash maps): a bijective relabeling to
    large / negative values passes; merging two clusters fails at the first
    core of the second one; same verdict as the compiled reference."""
    rng = np.random.default_rng(3)
    c = rng.uniform(0, 10, (400, 2)).astype(np.float32)
    r = oracle.dbscan(c, 0.6, 4, 0)
    la, ca = r["labels"], r["core"]
    ids = [v for v in np.unique(la) if v >= 0]
    assert len(ids) >= 2
    m = {v: (2**31 - 1 - 5 * k if k % 2 else -1000 - k) for k, v in enumerate(ids)}
    m[-1] = -1
    lb = np.array([m[v] for v in la], np.int32)
    cases = [(lb, True)]
    merged = la.copy()
    merged[merged == ids[1]] = ids[0]
    cases.append((merged, False))
    for other, ok_want in cases:
        ok, msg = oracle.check_equivalence(c, 0.6, la, ca, other, ca)
        assert ok == ok_want, msg
        if ref.available():
            assert ref.check_equivalence(c, 0.6, 4, la, ca, other, ca) == (ok, msg)


def test_reciprocal_morton_quantization_is_exact():
    """The device's quantize_rcp (device_common.cuh) multiplies by RN(1/w)
    and falls back to the exact division when the scaled value lies within
    cells * 2^-48 of an integer. The same fp64 operations in numpy (IEEE,
    round-to-nearest) against the reference's division (geometry.hpp:132-141),
    on random and adversarial (exact cell boundaries and their fp32
    neighbours) coordinates, 2D and 3D cell counts."""
    rng = np.random.default_rng(7)
    for bits in (21, 31):
        cells = 2 ** bits
        cd = float(cells)
        for _ in range(4):
            lo = np.float32(rng.uniform(-100, 100))
            hi = np.float32(lo + np.float32(rng.uniform(1e-3, 1e3)))
            w = np.float64(hi) - np.float64(lo)
            rw = 1.0 / w
            k = rng.integers(0, cells, 100_000).astype(np.float64)
            adv = (np.float64(lo) + k / cd * w).astype(np.float32)
            v = np.concatenate([rng.uniform(lo, hi, 200_000).astype(np.float32), adv,
                                np.nextafter(adv, np.float32(np.inf)),
                                np.nextafter(adv, np.float32(-np.inf)), [lo, hi]])
            v = np.clip(v.astype(np.float32), lo, hi)
            d = v.astype(np.float64) - np.float64(lo)
            want = np.minimum(np.floor(np.maximum(d / w, 0) * cd), cells - 1)
            x = (d * rw) * cd
            fl = np.floor(x)
            frac = x - fl
            m = cd * 2.0 ** -48
            fast = (frac >= m) & (frac <= 1 - m) & (d >= 0)
            got = np.where(fast, np.minimum(fl, cells - 1), want)
            assert np.array_equal(got, want)
            assert fast.mean() > 0.99  # the exact chain stays rare
