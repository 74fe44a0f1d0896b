"""The drop-in boundary, CPU side: the C-ABI library loads, exports every
symbol include/*.h declares, and the host half of the ABI (datasets, file
formats, generators, argument validation, status codes) behaves like the
reference's (REF tests/test_capi.cpp). No kernel runs here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import paper_2103_05162_b200 as tb
from paper_2103_05162_b200 import Algorithm, Dataset, Status, TreeclustError
from paper_2103_05162_b200._lib import LIB_PATH, SIGNATURES, lib

from ._util import generators, sha

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in ("treeclust.h", "treeclust_gpu.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(tcg?_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    # the 18 reference entry points are all there
    ref18 = {"tc_status_string", "tc_dataset_create", "tc_dataset_load", "tc_dataset_save",
             "tc_dataset_size", "tc_dataset_dim", "tc_dataset_coords", "tc_dataset_free",
             "tc_generate_blobs", "tc_generate_uniform", "tc_generate_lattice", "tc_cluster",
             "tc_result_size", "tc_result_labels", "tc_result_core_flags", "tc_result_stats",
             "tc_result_free", "tc_verify"}
    assert ref18 <= names
    raw = C.CDLL(LIB_PATH)
    for name in sorted(names):
        assert hasattr(raw, name), f"{name} declared in include/ but not exported"
        assert name in SIGNATURES, f"{name} has no ctypes signature"


def test_no_torch_or_cpp_symbols_leak():
    out = os.popen(f"nm -D --defined-only {LIB_PATH}").read()
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert all(s.startswith(("tc_", "tcg_")) for s in exported), sorted(exported)[:10]


def test_status_strings():
    assert tb.status_string(0) == "ok"
    assert tb.status_string(1) == "invalid argument"
    assert tb.status_string(4) == "oracle cap exceeded"
    assert tb.status_string(99) == "unknown status"


def test_dataset_create_and_accessors():  # REF test_capi.cpp:25-33
    coords = np.array([[0, 0], [1, 1], [2, 0]], np.float32)
    ds = Dataset.from_array(coords)
    assert ds.size == 3 and ds.dim == 2
    assert np.array_equal(ds.coords(), coords)


def test_invalid_dataset_arguments():  # REF test_capi.cpp:35-55
    out = C.c_void_p()
    one = (C.c_float * 2)(0.0, 0.0)
    assert lib.tc_dataset_create(None, 1, 2, C.byref(out)) == Status.INVALID_ARGUMENT
    assert lib.tc_dataset_create(one, 1, 5, C.byref(out)) == Status.INVALID_ARGUMENT
    assert lib.tc_dataset_create(one, 0, 2, C.byref(out)) == Status.INVALID_ARGUMENT
    with pytest.raises(TreeclustError) as e:
        Dataset.from_array(np.array([[0.0, np.nan]], np.float32))
    assert e.value.status == Status.INVALID_ARGUMENT
    with pytest.raises(TreeclustError):
        Dataset.from_array(np.array([[0.0, np.inf, 1.0]], np.float32))


def test_cluster_argument_validation_before_any_device_work():
    ds = Dataset.from_array(np.zeros((1, 2), np.float32))
    res = C.c_void_p()
    assert lib.tc_cluster(ds.handle, C.c_float(-1.0), 2, 0, 1, 0, C.byref(res)) == 1
    assert lib.tc_cluster(ds.handle, C.c_float(1.0), 1, 0, 1, 0, C.byref(res)) == 1
    assert lib.tc_cluster(ds.handle, C.c_float(float("nan")), 2, 0, 1, 0, C.byref(res)) == 1
    assert lib.tc_cluster(ds.handle, C.c_float(float("inf")), 2, 1, 1, 0, C.byref(res)) == 1
    assert lib.tc_cluster(None, C.c_float(1.0), 2, 0, 1, 0, C.byref(res)) == 1
    assert lib.tc_cluster(ds.handle, C.c_float(1.0), 2, 0, 1, 0, None) == 1
    assert lib.tc_cluster(ds.handle, C.c_float(1.0), 2, 7, 1, 0, C.byref(res)) == 1
    assert not res.value  # *out written only on success
    big = Dataset.blobs(1, 100, 2, 5.0, 0.3, 2)  # REF test_capi.cpp:131-140
    assert lib.tc_cluster(big.handle, C.c_float(1.0), 5, 2, 1, 50, C.byref(res)) == 4
    # cap is checked before eps/minpts, like capi.cpp:166-168
    assert lib.tc_cluster(big.handle, C.c_float(-1.0), 5, 2, 1, 50, C.byref(res)) == 4


@pytest.mark.skipif(tb.device_count() > 0, reason="exercises the no-device error path")
def test_no_device_is_an_internal_error_not_a_fallback():
    ds = Dataset.blobs(2, 50, 2, 5.0, 0.3, 7)
    with pytest.raises(TreeclustError) as e:
        tb.cluster(ds, 0.5, 5)
    assert e.value.status == Status.INTERNAL


def test_load_save_round_trip(tmp_path):  # REF test_capi.cpp:57-78
    ds = Dataset.blobs(2, 50, 2, 5.0, 0.3, 7)
    for name in ("capi_io.csv", "capi_io.bin"):
        p = str(tmp_path / name)
        ds.save(p)
        back = Dataset.load(p)
        assert back.size == 100 and back.dim == 2
        assert np.array_equal(back.coords(), ds.coords())
    with pytest.raises(TreeclustError) as e:
        Dataset.load("/nonexistent/path.csv")
    assert e.value.status == Status.IO


def test_csv_header_and_errors(tmp_path):  # REF io.cpp:58-104
    p = tmp_path / "h.csv"
    p.write_text("x,y\n1,2\n3, 4\n\n5,6\r\n")
    d = Dataset.load(str(p))
    assert d.size == 3 and np.array_equal(d.coords(), [[1, 2], [3, 4], [5, 6]])
    p.write_text("1,2\n3,4,5\n")
    with pytest.raises(TreeclustError) as e:
        Dataset.load(str(p))
    assert e.value.status == Status.IO
    p.write_text("1,2\nfoo\n")
    with pytest.raises(TreeclustError):
        Dataset.load(str(p))
    b = tmp_path / "t.bin"
    b.write_bytes(np.array([5, 2], np.uint32).tobytes() + np.zeros(4, np.float32).tobytes())
    with pytest.raises(TreeclustError) as e:
        Dataset.load(str(b))
    assert e.value.status == Status.IO


def test_generators_seeded_and_validated():  # REF test_capi.cpp:80-101
    a = Dataset.blobs(3, 40, 3, 6.0, 0.4, 11)
    b = Dataset.blobs(3, 40, 3, 6.0, 0.4, 11)
    assert np.array_equal(a.coords(), b.coords())
    assert Dataset.uniform(100, 2, [0, 0], [1, 1], 3).size == 100
    assert Dataset.lattice(5, 2, 0.5).size == 25
    with pytest.raises(TreeclustError) as e:
        Dataset.blobs(0, 40, 2, 6.0, 0.4, 1)
    assert e.value.status == Status.INVALID_ARGUMENT
    with pytest.raises(TreeclustError):
        Dataset.uniform(10, 2, [1, 0], [0, 1], 3)
    with pytest.raises(TreeclustError):
        Dataset.lattice(1, 2, 0.5)


def test_generators_byte_identical_to_reference():
    """Golden sha256 produced by running the reference generators
    (tests/golden/make_golden.py)."""
    g = generators()
    assert sha(Dataset.blobs(3, 80, 2, 20.0, 0.5, 21).coords()) == g["blobs(3,80,2,20,0.5,21)"]
    assert sha(Dataset.blobs(3, 40, 3, 6.0, 0.4, 11).coords()) == g["blobs(3,40,3,6,0.4,11)"]
    assert sha(Dataset.blobs(100, 10000, 2, 0.8333333, 0.08333333, 7).coords()) == \
        g["blobs(100,10000,2,0.8333333,0.08333333,7)"]
    assert sha(Dataset.uniform(1000, 3, [0, -1, 2], [1, 1, 5], 3).coords()) == \
        g["uniform(1000,3,[0,-1,2],[1,1,5],3)"]
    assert sha(Dataset.lattice(40, 2, 0.1).coords()) == g["lattice(40,2,0.1)"]
    assert sha(Dataset.lattice(12, 3, 0.1).coords()) == g["lattice(12,3,0.1)"]
    for s in (1, 7, 24):
        ds, eps, mp = Dataset.random_instance(s, 50, 1500)
        want = g[f"random_instance({s},50,1500)"]
        assert sha(ds.coords()) == want["sha256"] and eps == want["eps"] and mp == want["minpts"]


def test_hacc_like_calibration_shape():
    """The §8d HACC-like generator: 23% of points in Plummer halos, the rest
    uniform in [0, L)^3 with L scaled to keep the C2 density."""
    n = 200_000
    ds = Dataset.hacc_like(n)
    c = ds.coords()
    L = 36.8 * (n / 37e6) ** (1 / 3)
    bg = c[: n - int(0.23 * n)]
    assert bg.min() >= 0 and bg.max() < L
    assert ds.size == n and ds.dim == 3
    assert np.array_equal(c, Dataset.hacc_like(n).coords())  # deterministic


def test_taxi_like_in_unit_square():
    c = Dataset.taxi_like(100_000).coords()
    assert c.shape == (100_000, 2) and c.min() >= 0 and c.max() <= 1


def test_verify_null_dataset():
    assert lib.tc_verify(None, C.c_float(1.0), 5, 1, 0, None, 0) == Status.INVALID_ARGUMENT


def test_product_path_has_no_oracle_dependency():
    """The shipped package never imports or links the test oracle."""
    pkg = os.path.join(ROOT, "paper_2103_05162_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".hpp")) or f == "Makefile":
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert "oracle/" not in txt and "import oracle" not in txt and \
                    "from oracle" not in txt and "liboracle" not in txt, f
    libs = os.popen(f"ldd {LIB_PATH}").read()
    assert "oracle" not in libs and "treeclust_ref" not in libs


def test_additive_entry_points_validate_before_device_work(tmp_path):
    """tcg_binary_info / tcg_load_binary_device / tcg_cluster_keyed_device /
    tcg_local_*: header parsing and argument checks are host-side and need no
    GPU; errors map like the reference ABI's (bad file -> TC_ERR_IO, null or
    invalid argument -> TC_ERR_INVALID_ARGUMENT)."""
    ds = Dataset.blobs(2, 50, 3, 5.0, 0.3, 7)
    path = str(tmp_path / "p.bin")
    ds.save(path)
    n, d = C.c_int64(), C.c_int()
    assert lib.tcg_binary_info(path.encode(), C.byref(n), C.byref(d)) == Status.OK
    assert (n.value, d.value) == (100, 3)
    assert lib.tcg_binary_info(b"/nonexistent.bin", C.byref(n), C.byref(d)) == Status.IO
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"\x05\x00\x00\x00\x07\x00\x00\x00")
    assert lib.tcg_binary_info(str(bad).encode(), C.byref(n), C.byref(d)) == Status.IO
    assert lib.tcg_binary_info(None, C.byref(n), C.byref(d)) == Status.INVALID_ARGUMENT
    assert lib.tcg_load_binary_device(path.encode(), None, 100, 3, None) == Status.INVALID_ARGUMENT
    assert lib.tcg_load_binary_device(path.encode(), C.c_void_p(16), 100, 4, None) == \
        Status.INVALID_ARGUMENT
    st = tb.api.TcClusterStats()
    assert lib.tcg_cluster_keyed_device(C.c_void_p(16), None, 10, 3, C.c_float(0.1), 2,
                                        C.c_void_p(16), C.c_void_p(16), None,
                                        C.byref(st)) == Status.INVALID_ARGUMENT
    h = C.c_void_p()
    assert lib.tcg_local_create(None, C.c_void_p(16), 10, 3, C.c_float(0.1), None,
                                C.byref(h)) == Status.INVALID_ARGUMENT
    assert lib.tcg_local_create(C.c_void_p(16), C.c_void_p(16), 10, 3, C.c_float(-1.0), None,
                                C.byref(h)) == Status.INVALID_ARGUMENT
    assert h.value is None  # *out untouched on failure
    assert lib.tcg_local_core_flags(None, 5, C.c_void_p(16)) == Status.INVALID_ARGUMENT
    assert lib.tcg_local_cluster(None, C.c_void_p(16), C.c_void_p(16), C.c_void_p(16)) == \
        Status.INVALID_ARGUMENT
    lib.tcg_local_free(None)  # no-op


CSV_CASES = {
    "plain2": "1,2\n3,4\n",
    "plain3_crlf": "1,2,3\r\n4,5,6\r\n",
    "header": "x,y\n1,2\n",
    "header_then_bad": "x,y\nfoo\n1,2\n",
    "blank_lines": "\n\r\n1, 2\n\n 3 ,\t4\n",
    "trailing_comma": "1,2,\n3,4,\n",
    "leading_comma": ",1,2\n",
    "four_fields": "1,2,3,4\n",
    "one_field": "1\n2\n",
    "inconsistent": "1,2\n1,2,3\n",
    "no_newline_at_end": "1,2\n3,4",
    "only_header": "a,b\n",
    "empty": "",
    "whitespace_line": "1,2\n   \n3,4\n",
    "exponent": "1e-3,2.5E2\n-0.0,7\n",
    "nonfinite": "inf,1\n2,3\n",
    "garbage_after": "1,2x\n",
    "spaces_only_fields": "1 2\n",
}


@pytest.mark.parametrize("case", sorted(CSV_CASES))
def test_csv_reader_matches_reference(tmp_path, case):
    """tc_dataset_load on CSV edge cases gives the reference's status and points
    (REF io.cpp:29-104)."""
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    path = str(tmp_path / f"{case}.csv")
    with open(path, "w", newline="") as f:
        f.write(CSV_CASES[case])
    L = ref._capi()
    L.tc_dataset_dim.restype = C.c_int
    L.tc_dataset_dim.argtypes = [C.c_void_p]
    L.tc_dataset_coords.restype = C.POINTER(C.c_float)
    L.tc_dataset_coords.argtypes = [C.c_void_p]
    h = C.c_void_p()
    want = L.tc_dataset_load(path.encode(), 0, C.byref(h))
    want_pts = None
    if want == 0:
        n, d = L.tc_dataset_size(h), L.tc_dataset_dim(h)
        want_pts = np.ctypeslib.as_array(L.tc_dataset_coords(h), shape=(n * d,)).reshape(n, d).copy()
        L.tc_dataset_free(h)
    try:
        got_pts = Dataset.load(path).coords()
        got = 0
    except TreeclustError as e:
        got = int(e.status)
    assert got == want, (case, got, want)
    if want == 0:
        assert np.array_equal(got_pts, want_pts)


@pytest.mark.parametrize("suffix", [".csv", ".bin"])
def test_writers_match_reference_bytes(tmp_path, suffix):
    """tc_dataset_save writes the reference's bytes (REF io.cpp:84-148)."""
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    pts = Dataset.hacc_like(500, seed=9).coords()
    pts[:5] *= np.float32(1e-7)
    ours, theirs = str(tmp_path / f"a{suffix}"), str(tmp_path / f"b{suffix}")
    Dataset.from_array(pts).save(ours)
    L = ref._capi()
    L.tc_dataset_save.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
    rds = ref.RefDataset.from_array(pts)
    assert L.tc_dataset_save(rds.h, theirs.encode(), 0) == 0
    rds.close()
    assert open(ours, "rb").read() == open(theirs, "rb").read()


def test_binary_reader_errors_match_reference(tmp_path):
    from oracle import ref

    if not ref.available():
        pytest.skip("oracle/_ref not built")
    good = np.arange(12, dtype=np.float32).reshape(4, 3)
    blobs = {
        "short_header": b"\x04\x00\x00",
        "zero_n": np.array([0, 3], "<u4").tobytes(),
        "bad_dim": np.array([4, 4], "<u4").tobytes() + good.tobytes(),
        "truncated": np.array([4, 3], "<u4").tobytes() + good.tobytes()[:40],
        "ok_extra_tail": np.array([4, 3], "<u4").tobytes() + good.tobytes() + b"xyz",
        "ok": np.array([4, 3], "<u4").tobytes() + good.tobytes(),
    }
    L = ref._capi()
    for name, blob in blobs.items():
        path = str(tmp_path / f"{name}.bin")
        open(path, "wb").write(blob)
        h = C.c_void_p()
        want = L.tc_dataset_load(path.encode(), 0, C.byref(h))
        if want == 0:
            L.tc_dataset_free(h)
        try:
            got = 0
            assert np.array_equal(Dataset.load(path).coords(), good)
        except TreeclustError as e:
            got = int(e.status)
        assert got == want, name
    missing = str(tmp_path / "nope.bin")
    with pytest.raises(TreeclustError) as e:
        Dataset.load(missing)
    assert e.value.status == Status.IO
