"""Per-kernel table from one or more `ncu --set full` raw CSV exports
(`ncu -i X.ncu-rep --page raw --csv`): duration, DRAM bytes and GB/s against
the measured HBM peak (MEASURED_PEAKS.json), L1/L2 hit rates, warp execution
efficiency (active threads per warp instruction / 32), occupancy, SM
throughput. Markdown on stdout.

  python tools/ncu_table.py a_raw.csv [b_raw.csv ...]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
         "nsecond": 1e-9, "second": 1.0}


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def val(row, hdr, units, name):
    if name not in hdr:
        return None
    i = hdr.index(name)
    try:
        v = float(row[i].replace(",", ""))
    except ValueError:
        return None
    return v * SCALE.get(units[i], 1.0)


def main():
    pk = peak()
    print(f"| kernel | ms | DRAM GB | DRAM GB/s | % of {pk:.0f} GB/s | L1 hit % | L2 hit % | "
          "warp eff. % | occupancy % | SM % | regs |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    seen = set()
    for path in sys.argv[1:]:
        rows = list(csv.reader(open(path)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
            if "::k_" in name:
                name = "k_" + name.split("::k_", 1)[1]
            if name in seen:
                continue
            seen.add(name)
            t = val(r, hdr, units, "gpu__time_duration.sum")
            rd = val(r, hdr, units, "dram__bytes_read.sum") or 0.0
            wr = val(r, hdr, units, "dram__bytes_write.sum") or 0.0
            gbs = (rd + wr) / t / 1e9 if t else 0.0
            th = val(r, hdr, units, "smsp__thread_inst_executed_per_inst_executed.ratio") or 0.0
            l1 = val(r, hdr, units, "l1tex__t_sector_hit_rate.pct")
            l2 = val(r, hdr, units, "lts__t_sector_hit_rate.pct")
            occ = val(r, hdr, units, "sm__warps_active.avg.pct_of_peak_sustained_active")
            sm = val(r, hdr, units, "sm__throughput.avg.pct_of_peak_sustained_elapsed")
            regs = val(r, hdr, units, "launch__registers_per_thread")
            f = lambda v, d=1: "-" if v is None else f"{v:.{d}f}"
            print(f"| `{name[:48]}` | {t * 1e3:.3f} | {(rd + wr) / 1e9:.3f} | {gbs:.0f} | "
                  f"{gbs / pk * 100:.1f} | {f(l1)} | {f(l2)} | {th / 32 * 100:.0f} | {f(occ)} | "
                  f"{f(sm)} | {f(regs, 0)} |")


if __name__ == "__main__":
    main()
