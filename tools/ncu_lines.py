"""Per-source-line shared-memory wavefronts / stall samples from an ncu report
(development aid): python tools/ncu_lines.py report.ncu-rep [N]"""

import csv
import io
import subprocess
import sys


def main(path, n=30):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hi = next(i for i, x in enumerate(r) if x and x[0] == "Line No")
    h = r[hi]
    iE = h.index("L1 Wavefronts Shared Excessive")
    iW = h.index("L1 Wavefronts Shared")
    iN = h.index("Warp Stall Sampling (All Samples)")
    rows = [x for x in r[hi + 1:] if len(x) > iE and x[2] == "-"]
    tw = sum(float(x[iW] or 0) for x in rows)
    te = sum(float(x[iE] or 0) for x in rows)
    ts = sum(float(x[iN] or 0) for x in rows)
    print(f"shared wavefronts {tw:.3e} (excessive {te:.3e}); stall samples {ts:.0f}")
    print("by shared wavefronts:")
    for x in sorted(rows, key=lambda x: -float(x[iW] or 0))[:n]:
        print(f"  {x[0]:>5} {float(x[iW] or 0):10.3e} exc {float(x[iE] or 0):9.2e} smp {x[iN]:>6}  {x[1].strip()[:70]}")
    print("by stall samples:")
    for x in sorted(rows, key=lambda x: -float(x[iN] or 0))[:n]:
        print(f"  {x[0]:>5} smp {x[iN]:>6} ({100 * float(x[iN]) / ts:4.1f}%)  {x[1].strip()[:80]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
