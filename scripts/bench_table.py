"""Markdown table of per-kernel times and HBM fractions from bench.py JSON lines.

    python scripts/bench_table.py profiles/r01_bench_c2_vN.json ...
"""
import json
import sys

KS = ["K1_local_in", "K2_anterp", "K3_fft_conv", "K4_interp_corr", "K5_grad_sum"]
print("| config | N' | ms/eval | evals/s | " + " | ".join("%s ms (%% HBM)" % k.split("_")[0] for k in KS) +
      " | C_box | clocks |")
print("|---" * (6 + len(KS)) + "|")
for p in sys.argv[1:]:
    d = json.loads(open(p).read().strip().splitlines()[-1])
    c = d["config"]
    peak = d["roofline"]["peak"]
    cells = []
    for k in KS:
        v = d["kernels"][k]
        cells.append("%.3f (%d %%)" % (v["ms"], round(100 * v["GBps"] / peak)) if v["GBps"] else "%.3f" % v["ms"])
    print("| %s | %.2fM | %.3f | %.0f | %s | %s | %s MHz |" % (
        c["workload"].split(":")[0], c["n_parents"] / 1e6, d["ms_per_step"], d["value"], " | ".join(cells),
        c.get("cbox_format", "CSR"), d["clocks"]["sm_mhz"]))
