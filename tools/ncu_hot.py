"""Top stalled SASS instructions of an ncu report (source page), with per-warp-block execution counts.

    python tools/ncu_hot.py report.ncu-rep [units_for_normalisation] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
iS, iE, iW = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_") or "Stall" in c and i not in (iW,)]
tot = sum(int(r[iW] or 0) for r in data if r[iW].isdigit())
rowsx = []
for idx, r in enumerate(data):
    w = int(r[iW]) if r[iW].isdigit() else 0
    rowsx.append((w, idx, r))
print("columns:", [h[i] for i in stall_cols][:30])
for w, idx, r in sorted(rowsx, reverse=True)[:top]:
    e = int(r[iE]) if r[iE].isdigit() else 0
    print(f"{idx:5d} {100.0 * w / tot:5.1f}% ex/unit={e / units:7.2f}  {r[iS].strip()[:90]}")
