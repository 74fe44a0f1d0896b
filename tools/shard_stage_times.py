import sys, torch
sys.path.insert(0, ".")
import paper_2103_05162_b200 as tb
from paper_2103_05162_b200.shard import DeviceEngine
x = tb.generate_device("hacc_like", 37_000_000)
eng = DeviceEngine("cuda:0")
codes = eng.morton(x, x.min(0).values, x.max(0).values)
gid = torch.arange(x.shape[0], dtype=torch.int64, device="cuda")
perm = torch.randperm(x.shape[0], device="cuda")
xs, cs = x[perm].contiguous(), codes[perm].contiguous()   # the route's source-ordered arrival
for name, fn in (("region_boxes", lambda: eng.region_boxes(xs, cs)),
                 ("route", lambda: eng.route(x, gid, codes, torch.empty(0, dtype=torch.int64, device="cuda"))),
                 ("unpack", lambda: eng.unpack(eng.route(x, gid, codes, torch.empty(0, dtype=torch.int64, device="cuda"))[0], 3, True))):
    for it in range(4):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    print(name, round(e0.elapsed_time(e1), 3), "ms")
