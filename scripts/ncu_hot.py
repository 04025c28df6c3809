"""Top SASS lines of one kernel in an .ncu-rep by warp-stall samples (with executed counts).

    python scripts/ncu_hot.py REP KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(r for r in rows if "Address" in r)
d = [r for r in rows if len(r) == len(h) and r[0].startswith("0x")]
si, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
f = lambda x: int(x) if x.strip() else 0
half = len(d) // 2 if len(d) % 2 == 0 and d[:len(d) // 2] == d[len(d) // 2:] else len(d)
d = d[:half]
print("samples", sum(f(r[si]) for r in d), "warp instructions", sum(f(r[ie]) for r in d), "sass lines", len(d))
for i, r in sorted(enumerate(d), key=lambda x: -f(x[1][si]))[:n]:
    print("%5d %6s %10s  %s" % (i, r[si], r[ie], r[1][:100]))
