"""Top stalled SASS instructions of an ncu report with their CUDA source line
(development aid): python tools/ncu_sass_lines.py report.ncu-rep [N]"""
import csv
import io
import re
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
src = open(re.search(r'"File Path","([^"]+)"', out).group(1)).read().split("\n")
line = None
addr_line = {}
for x in csv.reader(io.StringIO(out)):
    if len(x) > 2 and x[0].isdigit():
        line = int(x[0])
    for f in x:
        if re.fullmatch(r"0x[0-9a-f]+", f):
            addr_line[f] = line
            break
out2 = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                      capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out2)))
h = r[1]
rows = []
for x in r[2:]:  # first kernel of the report only
    if x and x[0] in ("Kernel Name", "Address"):
        break
    rows.append(x)
iS, iN = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
sc = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(float(x[iN] or 0) for x in rows)
by_line = {}
for x in rows:
    ln = addr_line.get(x[0])
    by_line[ln] = by_line.get(ln, 0) + float(x[iN] or 0)
print("by source line:")
for ln, v in sorted(by_line.items(), key=lambda kv: -kv[1])[:n]:
    s = src[ln - 1].strip()[:80] if ln else "?"
    print(f"  {ln!s:>5} {100 * v / tot:5.1f}%  {s}")
print("top SASS:")
for x in sorted(rows, key=lambda x: -float(x[iN] or 0))[:n]:
    st = sorted(((float(x[i] or 0), h[i][6:]) for i in sc), reverse=True)[:2]
    ln = addr_line.get(x[0])
    print(f"  {100 * float(x[iN]) / tot:5.2f}% L{ln!s:>4} {x[iS].strip()[:44]:44s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")
