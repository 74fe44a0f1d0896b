"""Summarize ncu outputs into profiles/ (tracked): per-kernel launch shares from a
`--metrics gpu__time_duration.sum` launch list, and the key counters of a
`--set full` capture. Also writes profiles/traffic.json, which bench.py reads
for roofline.traffic (DRAM bytes per launch of the dominant kernel).

  python tools/summarize_ncu.py <tag> <launches.csv> <full_raw.csv[,more.csv]> [kernel-substring]
                                [--no-traffic]
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[h], rows[h + 1:]
    ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in data:
        name = r[ik].split("(")[0].replace("void ", "")
        if "::k_" in name:
            name = "k_" + name.split("::k_", 1)[1]
        v = float(r[iv].replace(",", ""))
        agg.setdefault(name, [0, 0.0])
        agg[name][0] += 1
        agg[name][1] += v
    return agg


METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers / thread"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
     "L1 LSU data-pipe wavefronts % of peak"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue slots busy %"),
]


def full(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        rec = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                rec[label] = (r[i], units[i])
        out.append(rec)
    return out


def to_bytes(val, unit):
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return v * scale.get(unit, 1)


def main():
    argv = [a for a in sys.argv[1:] if a != "--no-traffic"]
    write_traffic = "--no-traffic" not in sys.argv
    tag, lpath, fpaths = argv[0:3]
    kfilter = argv[3] if len(argv) > 3 else "k_fd_main"
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary {tag}", ""]
    agg = launches(lpath)
    tot = sum(v[1] for v in agg.values())
    lines += ["## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
              "Cold-cache, serialised per-launch times: compare SHARES, not absolutes.", "",
              "| kernel | launches | avg us | share |", "|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {v / c / 1e3:.1f} | {v / tot * 100:.1f}% |")
    lines += ["", "## `--set full` captures", ""]
    traffic = None
    bound = {}
    recs = [r for fp in fpaths.split(",") for r in full(fp)]
    for rec in recs:
        lines.append(f"### `{rec['kernel']}`")
        for m, label in METRICS:
            if label in rec:
                lines.append(f"- {label}: {rec[label][0]} {rec[label][1]}")
        lines.append("")
        if kfilter in rec["kernel"] and traffic is None and "DRAM read" in rec:
            traffic = to_bytes(*rec["DRAM read"]) + to_bytes(*rec["DRAM write"])
            for key, label in (("l1_lsu_wavefront_pct", "L1 LSU data-pipe wavefronts % of peak"),
                               ("issue_active_pct", "issue slots busy %"),
                               ("dram_pct", "DRAM % of peak")):
                if label in rec:
                    bound[key] = round(float(rec[label][0].replace(",", "")), 1)
    with open(os.path.join(ROOT, "profiles", f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic is not None and write_traffic:
        with open(os.path.join(ROOT, "profiles", "traffic.json"), "w") as f:
            json.dump({"k_fd_main_dram_bytes_per_launch": traffic, "source": f"{tag} ncu --set full",
                       "kernel": kfilter, "limiter": bound}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
