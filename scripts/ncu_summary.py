"""Summarise ncu outputs for profiles/: a launch list (--metrics gpu__time_duration.sum --csv)
and/or a --set full report (.ncu-rep).

    python scripts/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/prof.ncu-rep > profiles/x.md
"""
import argparse
import csv
import io
import re
import subprocess
from collections import OrderedDict


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("pmfem::", "").replace("<unnamed>::", "").replace("(anonymous namespace)::", "")
    return name.strip()[:48]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[vi]:
            out.append((short(r[ki]), float(r[vi].replace(",", "")) / 1e3))   # ns -> us
    return out


def rep(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h = rows[0]
    want = OrderedDict([("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"),
                        ("dram__bytes_read.sum", "dram_rd_MB"), ("dram__bytes_write.sum", "dram_wr_MB"),
                        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
                        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
                        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
                        ("launch__registers_per_thread", "regs"),
                        ("lts__t_sector_hit_rate.pct", "L2_hit_%"),
                        ("l1tex__t_sector_hit_rate.pct", "L1_hit_%")])
    units = rows[1]
    idx = [(h.index(k), v) for k, v in want.items() if k in h]
    out = []
    for r in rows[2:]:
        d = {}
        for i, v in idx:
            val = r[i]
            if v == "kernel":
                val = short(val)
            elif v.startswith("dram_") and v.endswith("MB"):
                u = units[i]
                f = float(val.replace(",", ""))
                f *= {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                val = "%.2f" % f
            elif v == "us":
                u = units[i]
                f = float(val.replace(",", ""))
                f *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(u, 1.0)
                val = "%.2f" % f
            d[v] = val
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    if a.title:
        print("# " + a.title + "\n")
    if a.launches:
        L = launches(a.launches)
        agg = OrderedDict()
        for n, t in L:
            agg.setdefault(n, []).append(t)
        def is_eval(k):   # per-evaluation kernels (setup kernels and torch's own are excluded)
            return not k.startswith(("void at::", "at::", "k_z0", "k_cbox", "k_c4x", "k_b4", "k_pgf", "k_spec")) \
                and "<double" not in k
        tot = sum(sum(v) for k, v in agg.items() if is_eval(k))
        print("## Launch list (ncu gpu__time_duration.sum, cold-cache, serialised)\n")
        print("| kernel | launches | mean us | share of one evaluation |")
        print("|---|---|---|---|")
        for k, v in agg.items():
            share = sum(v) / tot if is_eval(k) else 0
            print("| %s | %d | %.2f | %.1f%% |" % (k, len(v), sum(v) / len(v), 100 * share))
        print()
    if a.rep:
        R = rep(a.rep)
        if R:
            keys = list(R[0].keys())
            print("## ncu --set full (per launch)\n")
            print("| " + " | ".join(keys) + " |")
            print("|" + "---|" * len(keys))
            for d in R:
                print("| " + " | ".join(str(d.get(k, "")) for k in keys) + " |")


if __name__ == "__main__":
    main()
