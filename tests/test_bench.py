"""bench.py contract checks that run without a GPU: the reference arm measures
the reference's own CPU path on our arm's workload and never loads the
product library."""
import json
import os
import subprocess
import sys

import pytest

from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, sys
sys.argv = ["bench.py", "--impl", "reference", "--points", "120000", "--steps", "2",
            "--warmup", "1"]
import bench
rc = bench.main()
maps = open("/proc/self/maps").read()
print(json.dumps({"rc": rc, "product_imported": "paper_2103_05162_b200" in sys.modules,
                  "product_so_mapped": "libtreeclust_b200" in maps,
                  "ref_so_mapped": "libtreeclust_ref" in maps}))
"""


def test_reference_arm_is_self_contained():
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True,
                         timeout=600, env={**os.environ, "WORLD_SIZE": "1", "RANK": "0"})
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert probe == {"rc": 0, "product_imported": False, "product_so_mapped": False,
                     "ref_so_mapped": True}
    assert line["impl"] == "reference" and line["steps"] == 2 and line["warmup"] == 1
    assert line["config"]["points_per_rank"] == 120000 and line["config"]["minpts"] == 2
    assert line["cpu_baseline"]["kind"] == "reference" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"],
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert line["stats"]["pair_resolutions"] > 0


def test_reference_arm_other_ranks_exit_quietly():
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--points", "1000",
                          "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=120, env={**os.environ, "RANK": "1", "WORLD_SIZE": "2"})
    assert out.returncode == 0 and out.stdout.strip() == ""


@pytest.mark.gpu
def test_sweep_rows_match_the_reference(tmp_path):
    """bench.py --sweep (REF treeclust_cli.cpp:146-198):
    the reference's CSV columns plus device / tc_cluster times, and per row the
    reference CPU path on the same points with a parity verdict — every row
    of the small sweep must be parity-exact."""
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    import csv

    out = tmp_path / "tiny.csv"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--sweep", "tiny",
                        "--sweep-out", str(out)], capture_output=True, text=True, cwd=ROOT,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 2 * 2 * 2 * 2
    assert rows[0].keys() >= {"algorithm", "n", "eps", "minpts", "build_s", "total_s",
                              "clusters", "cores", "noise", "dense_fraction", "device_ms",
                              "ref_s", "parity"}
    assert all(row["parity"] == "True" for row in rows)
    assert all(float(row["ref_s"]) > 0 and float(row["device_ms"]) > 0 for row in rows)
