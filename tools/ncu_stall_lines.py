"""Per-source-line stall samples with the top stall reasons and instruction
counts from an ncu report (development aid):
python tools/ncu_stall_lines.py report.ncu-rep [N]"""
import csv
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 18
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hi = next(i for i, x in enumerate(r) if x and x[0] == "Line No")
h = r[hi]
iI = h.index("Instructions Executed")
iS = h.index("Warp Stall Sampling (All Samples)")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
rows = [x for x in r[hi + 1:] if len(x) > iI and x[2] == "-"]
tot = sum(float(x[iS] or 0) for x in rows)
ti = sum(float(x[iI] or 0) for x in rows)
print(f"samples {tot:.0f}  instructions {ti:.3e}")
for x in sorted(rows, key=lambda x: -float(x[iS] or 0))[:n]:
    st = sorted(((float(x[h.index(c)] or 0), c) for c in cols), reverse=True)[:3]
    print(f"{x[0]:>5} {100 * float(x[iS] or 0) / tot:5.1f}% inst {float(x[iI] or 0):9.2e} "
          f"{' '.join(f'{c[6:]}={v:.0f}' for v, c in st)} | {x[1].strip()[:60]}")
