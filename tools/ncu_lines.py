"""Per-source-line totals (instructions executed, warp stall samples) of one
kernel from `ncu -i REP --page source --csv --print-source cuda,sass`.

  python tools/ncu_lines.py gpurun_out/x.ncu-rep [top] [kernel-regex]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 3:
    cmd += ["--kernel-name", "regex:" + sys.argv[3]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
path = None
hdr = None
src_lines = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr) or r[0] == "":
        continue
    key = (path, int(r[0]))
    ii = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    ti = hdr.index("Thread Instructions Executed")
    try:
        a = agg.setdefault(key, [0.0, 0.0, 0.0])
        a[0] += float(r[ii] or 0)
        a[1] += float(r[ws] or 0)
        a[2] += float(r[ti] or 0)
    except ValueError:
        continue
    src_lines[key] = r[1]
ti = sum(v[0] for v in agg.values()) or 1
tw = sum(v[1] for v in agg.values()) or 1
print(f"total warp inst {ti:.3e}, stall samples {tw:.0f}")
for key, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    eff = v[2] / v[0] if v[0] else 0
    print(f"{key[0]}:{key[1]:<5} inst {100 * v[0] / ti:5.1f}%  stall {100 * v[1] / tw:5.1f}%  thr/inst {eff:4.1f}  {src_lines[key].strip()[:70]}")
