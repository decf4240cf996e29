"""Per-opcode executed-instruction histogram (normalised per unit) from an ncu report's source page.

    python tools/ncu_ophist.py report.ncu-rep units [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
op, st = collections.Counter(), collections.Counter()
tot_e = tot_w = 0
for r in rows[2:]:
    if not r[iE].isdigit():
        continue
    m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS])
    if not m:
        continue
    e, w = int(r[iE]), int(r[iW] or 0)
    op[m.group(2)] += e
    st[m.group(2)] += w
    tot_e += e
    tot_w += w
print(f"total {tot_e / units:.1f} warp-instructions per unit")
for k, v in op.most_common(top):
    print(f"{k:10s} {v / units:8.1f}   stall-samples {100.0 * st[k] / tot_w:5.1f}%")
