"""A C program compiled against include/treeclust.h and linked to
libtreeclust_b200.so (tests/c/capi_client.c): the drop-in as a reference
caller sees it, struct layout included."""
import ctypes as C
import os
import subprocess

import pytest

from paper_2103_05162_b200._lib import LIB_PATH, TcClusterStats

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def client(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("c") / "capi_client")
    libdir = os.path.dirname(LIB_PATH)
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-Wextra", "-Werror",
                    "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c",
                                                                     "capi_client.c"),
                    "-o", exe, "-L", libdir, "-l:" + os.path.basename(LIB_PATH),
                    "-Wl,-rpath," + libdir], check=True)
    return exe


def test_struct_layout_and_enums_match_the_mirror(client):
    out = subprocess.run([client, "layout"], capture_output=True, text=True, check=True).stdout
    lines = dict(line.split(" ", 1) for line in out.splitlines())
    assert int(lines["sizeof"]) == C.sizeof(TcClusterStats)
    for name, _ in TcClusterStats._fields_:
        assert int(lines[name]) == getattr(TcClusterStats, name).offset, name
    assert lines["enums"] == "0 1 2 3 4 5 | 0 1 2 | 0 1 2"


def test_c_client_host_checks(client, tmp_path):
    r = subprocess.run([client, "host", str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_c_client_three_algorithms_identical_labels(client):
    """REF tests/test_capi.cpp:103-150 through a C caller on the GPU build."""
    r = subprocess.run([client, "device"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.fixture(scope="module")
def graph_client(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cg") / "graph_client")
    libdir = os.path.dirname(LIB_PATH)
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["gcc", "-std=c11", "-O1", "-Wall", "-Wextra", "-Werror",
                    "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
                    os.path.join(ROOT, "tests", "c", "graph_client.c"), "-o", exe,
                    "-L", libdir, "-l:" + os.path.basename(LIB_PATH), "-L",
                    os.path.join(cuda, "lib64"), "-lcudart", "-Wl,-rpath," + libdir,
                    "-Wl,-rpath," + os.path.join(cuda, "lib64")], check=True)
    return exe


def test_graph_client_compiles(graph_client):
    assert os.path.exists(graph_client)


@pytest.mark.gpu
def test_c_client_captures_fdbscan_in_a_cuda_graph(graph_client):
    """tcg_cluster_device_async captured with cudaStreamBeginCapture from C and
    replayed on new points: equal to eager tcg_cluster_device runs; a
    non-finite coordinate is reported through the device status word."""
    r = subprocess.run([graph_client], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == "ok"
