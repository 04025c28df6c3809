"""Record per-launch DRAM traffic of the hot-path kernels from an `ncu --set full` report into
profiles/traffic.json, which bench.py reports as roofline.traffic (dram__bytes_read.sum +
dram__bytes_write.sum of the dominant kernel, per launch).

    python scripts/ncu_traffic.py --rep gpurun_out/prof_c2.ncu-rep --config C2 [--note "..."]
"""
import argparse
import csv
import io
import json
import os
import subprocess

KMAP = {"k1_local_in": "K1_local_in", "k2_tile": "K2_anterp", "k4_interp_corr": "K4_interp_corr", "k4_win": "K4_interp_corr",
        "k5_grad_sum": "K5_grad_sum", "fft_yz_fused": "K3_fft_yz_fused", "fft_x_forward<float>": "K3_fft_x_forward",
        "fft_x_inverse<float>": "K3_fft_x_inverse", "fft_strided<float": "K3_fft_strided"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--config", required=True)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    out = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    units = rows[1]
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
    db = json.load(open(path)) if os.path.exists(path) else {}
    ent = db.setdefault(a.config, {})
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        key = next((v for k, v in KMAP.items() if k in name), None)
        if key is None:
            continue
        rd = float(r[h.index("dram__bytes_read.sum")]) * scale[units[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")]) * scale[units[h.index("dram__bytes_write.sum")]]
        tu = units[h.index("gpu__time_duration.sum")]
        us = float(r[h.index("gpu__time_duration.sum")]) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(tu, 1.0)
        ent[key] = {"dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr, "ncu_us": us,
                    "report": os.path.basename(a.rep), "note": a.note}
        print(a.config, key, "%.1f MB" % ((rd + wr) / 1e6), "%.1f us" % us)
    json.dump(db, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
