"""Per-source-line stall samples, top stall reasons and instruction counts
from an ncu report, per source file (development aid):
python tools/ncu_stall_lines.py report.ncu-rep [N] [sort: smp|inst]"""
import csv
import os
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 18
key = sys.argv[3] if len(sys.argv) > 3 else "smp"
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, h, fname = [], None, "?"
for x in csv.reader(out.splitlines()):
    if x and x[0] == "File Path":
        fname = os.path.basename(x[1])
    elif x and x[0] == "Line No":
        h = x
    elif h and len(x) > 7 and x[2] == "-":
        rows.append((fname, x))
iI = h.index("Instructions Executed")
iS = h.index("Warp Stall Sampling (All Samples)")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(float(x[iS] or 0) for _, x in rows)
ti = sum(float(x[iI] or 0) for _, x in rows)
print(f"samples {tot:.0f}  instructions {ti:.3e}")
k = iS if key == "smp" else iI
for f, x in sorted(rows, key=lambda r: -float(r[1][k] or 0))[:n]:
    st = sorted(((float(x[h.index(c)] or 0), c) for c in cols), reverse=True)[:3]
    print(f"{f[:14]:>14}:{x[0]:<5} smp {100 * float(x[iS] or 0) / tot:5.1f}% inst {100 * float(x[iI] or 0) / ti:5.1f}% "
          f"{' '.join(f'{c[6:]}={v:.0f}' for v, c in st)} | {x[1].strip()[:60]}")
