"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by
kernel: python tools/launch_summary.py launches.csv "<command>" > summary.txt"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iK, iM, iV, iU = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = defaultdict(float)
cnt = defaultdict(int)
for r in rows[1:]:
    if r[iM] != "gpu__time_duration.sum":
        continue
    v = float(r[iV].replace(",", ""))
    v = v / 1e3 if r[iU] == "us" else (v / 1e6 if r[iU] == "ns" else v)
    tot[r[iK]] += v
    cnt[r[iK]] += 1
S = sum(tot.values())
print(f"ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised) over `{sys.argv[2]}`")
print("total_ms  launches  avg_ms  share  kernel")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{v:9.3f} {cnt[k]:6d} {v / cnt[k]:9.4f} {100 * v / S:5.1f}%  {k[:90]}")
