"""Repeats one configuration (developer tool):
python tools/repro_one.py n eps minpts algo reps [device|abi]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2103_05162_b200 as tb  # noqa: E402
from oracle import oracle  # noqa: E402

n, eps, minpts, algo, reps = int(sys.argv[1]), float(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
mode = sys.argv[6] if len(sys.argv) > 6 else "both"
c = oracle.hacc_like(n)
ds = tb.Dataset.from_array(c)
x = torch.from_numpy(c).cuda()
for r in range(reps):
    if mode in ("both", "abi"):
        tb.cluster(ds, eps, minpts, tb.Algorithm(algo))
    if mode in ("both", "device"):
        tb.cluster_device(x, eps, minpts, tb.Algorithm(algo))
        torch.cuda.synchronize()
print("ok", reps, flush=True)
