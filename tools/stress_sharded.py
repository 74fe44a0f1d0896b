"""Randomized stress of the multi-process sharded path (shard.py with the
product DeviceEngine, world 2-3 over gloo, every rank on cuda:0) against the
oracle (developer tool). python tools/stress_sharded.py [cases]"""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tools")
sys.path.insert(0, "tests")
from stress import cloud  # noqa: E402
from test_shard import check_against_oracle, run_sharded  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    rng = np.random.default_rng(4242)
    bad = 0
    for c in range(cases):
        kind, pts = cloud(rng)
        pts = pts[:2500]
        n = len(pts)
        ext = float(np.max(pts.max(0) - pts.min(0))) if n > 1 else 1.0
        eps = float(np.float32(max(ext, 1e-3) * 10 ** rng.uniform(-3, 0.2)))
        minpts = int(rng.choice([2, 3, 5]))
        world = int(rng.choice([2, 3]))
        try:
            labels, core = run_sharded(pts, eps, minpts, world=world, use_gpu=True)
            check_against_oracle(pts, eps, minpts, labels, core)
        except Exception as e:  # noqa: BLE001
            bad += 1
            print("BAD", kind, n, pts.shape[1], eps, minpts, world, repr(e)[:200], flush=True)
    print(f"cases {cases} bad {bad}", flush=True)


if __name__ == "__main__":  # (spawned ranks re-import this module)
    main()
