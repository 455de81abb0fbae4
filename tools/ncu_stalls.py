"""Per-source-line stall samples, top stall reasons and instruction share
from an ncu report (development aid): python tools/ncu_stalls.py rep [N]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hi = next(i for i, x in enumerate(r) if x and x[0] == "Line No")
h = r[hi]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
iI = h.index("Instructions Executed")
iS = h.index("Warp Stall Sampling (All Samples)")
rows = [x for x in r[hi + 1:] if len(x) > iI and x[2] == "-"]
tot = sum(float(x[iS] or 0) for x in rows)
ti = sum(float(x[iI] or 0) for x in rows)
print(f"instructions {ti:.3e}, stall samples {tot:.0f}")
agg = {c: sum(float(x[h.index(c)] or 0) for x in rows) for c in cols}
print("  ".join(f"{k[6:]}={v / tot * 100:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
for x in sorted(rows, key=lambda x: -float(x[iS] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    d = {c: float(x[h.index(c)] or 0) for c in cols}
    top = sorted(d.items(), key=lambda kv: -kv[1])[:3]
    print(f"{x[0]:>5} smp {float(x[iS]) / tot * 100:4.1f}% ins {float(x[iI] or 0) / ti * 100:4.1f}% "
          f"{' '.join(f'{k[6:]}={v:.0f}' for k, v in top)} | {x[1].strip()[:60]}")
