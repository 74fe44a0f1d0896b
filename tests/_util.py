"""Shared helpers for the parity tests (loading golden fixtures, comparing
clusterings the way SURVEY.md §8 defines parity)."""
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SEEDS = list(range(1, 25))
MIN_N, MAX_N = 50, 1500
COUNTER_NAMES = ("preprocess_skipped", "pair_resolutions", "distance_evaluations",
                 "cluster_count", "core_count", "noise_count")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, np.float32).tobytes()).hexdigest()


def generators():
    with open(os.path.join(GOLDEN, "generators.json")) as f:
        return json.load(f)


def npz(name):
    return np.load(os.path.join(GOLDEN, name))


def instance(seed):
    """random_instance(seed) from the product generator, pinned to the
    reference generator by the committed sha256."""
    import paper_2103_05162_b200 as tb

    ds, eps, mp = tb.Dataset.random_instance(seed, MIN_N, MAX_N)
    coords = ds.coords()
    g = generators()[f"random_instance({seed},{MIN_N},{MAX_N})"]
    assert sha(coords) == g["sha256"] and eps == g["eps"] and mp == g["minpts"]
    return ds, coords, eps, mp


def golden_run(db, seed, algo):
    c = db[f"s{seed}_a{algo}_counters"]
    return {"labels": db[f"s{seed}_a{algo}_labels"], "core": db[f"s{seed}_a{algo}_core"],
            "counters": dict(zip(COUNTER_NAMES, (int(v) for v in c))),
            "dense_fraction": float(db[f"s{seed}_a{algo}_dense_fraction"])}


def assert_parity(labels, core, want_labels, want_core, tag=""):
    """Core flags bit-exact, noise set exact, core labels EQUAL (the
    representative is the minimum core index), not merely isomorphic."""
    labels = np.asarray(labels)
    core = np.asarray(core)
    assert np.array_equal(core, want_core), f"{tag}: core flags differ at {np.flatnonzero(core != want_core)[:5]}"
    assert np.array_equal(labels == -1, want_labels == -1), f"{tag}: noise sets differ"
    cm = want_core == 1
    bad = np.flatnonzero(labels[cm] != want_labels[cm])
    assert bad.size == 0, f"{tag}: {bad.size} core labels differ"


def brute_pair_count(coords, eps):
    """testutil::brute_pair_count (tests/test_util.hpp:64-72), vectorised."""
    c = coords.astype(np.float64)
    eps2 = np.float64(np.float32(eps)) * np.float64(np.float32(eps))
    total = 0
    for i in range(len(c) - 1):
        d = c[i + 1:] - c[i]
        s = d[:, 0] * d[:, 0]
        for k in range(1, c.shape[1]):
            s = s + d[:, k] * d[:, k]
        total += int(np.count_nonzero(s <= eps2))
    return total
