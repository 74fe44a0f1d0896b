import time, torch, sys
sys.path.insert(0, ".")
import paper_2103_05162_b200 as tb
ds = tb.Dataset.hacc_like(37_000_000)
for _ in range(3): tb.cluster_raw(ds, 0.042, 2, tb.Algorithm.FDBSCAN)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); tb.cluster_raw(ds, 0.042, 2, tb.Algorithm.FDBSCAN); ts.append(time.perf_counter() - t0)
print("tc_cluster wall ms", [round(t * 1e3, 2) for t in ts], "stages", tb.last_stage_ms())
h = torch.empty(37_000_000 * 3, dtype=torch.float32).pin_memory()
d = torch.empty_like(h, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True); torch.cuda.synchronize()
t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); print("H2D 444MB ms", (time.perf_counter() - t0) * 1e3)
h2 = torch.empty(185_000_000, dtype=torch.uint8).pin_memory(); d2 = torch.empty_like(h2, device="cuda")
for _ in range(3): h2.copy_(d2, non_blocking=True); torch.cuda.synchronize()
t0 = time.perf_counter(); h2.copy_(d2, non_blocking=True); torch.cuda.synchronize(); print("D2H 185MB ms", (time.perf_counter() - t0) * 1e3)
