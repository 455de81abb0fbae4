"""3D assembly at p = 5, 6: the three-pass path (x pass -> G chunk, y sweep
-> H, z sweep -> CSR) against the fused stage-1/2 path (IGS_FLAG_TWO_PASS)
and the generic kernels on small ragged meshes, then timings at 64^3
(development aid)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import sumfac, workloads  # noqa: E402
from tools.sanitize import problem, rel  # noqa: E402

TWO_PASS, GENERIC = 8, 1
if "check" in sys.argv or len(sys.argv) == 1:
    for p, K, kind in [(5, (4, 3, 2), 3), (5, (6, 7, 5), 2), (5, (30, 9, 4), 3), (5, (2, 1, 1), 1), (6, (2, 2, 3), 3),
                       (6, (5, 4, 6), 2), (6, (23, 3, 2), 3), (6, (1, 1, 1), 3)]:
        prob = problem(p, K, kind, seed=10 + p)
        A = sumfac.assemble(prob).values_np()
        A2 = sumfac.assemble(prob, flags=TWO_PASS).values_np()
        Ag = sumfac.assemble(prob, flags=GENERIC).values_np()
        print(f"asm p={p} K={K} kind={kind} path={sumfac.fused_path(prob)} vs stage12 {rel(A, A2):.2e} "
              f"vs generic {rel(A, Ag):.2e}", flush=True)
if "time" in sys.argv or len(sys.argv) == 1:
    from tools.time_asm import run
    for c in [(3, 5, 64, 3, 0), (3, 5, 64, 3, 8), (3, 6, 64, 3, 0), (3, 6, 64, 3, 8)]:
        r = run(*c, reps=3)
        print(json.dumps(r), flush=True)
    # values at size: three-pass (several G chunks) vs stage-1/2
    prob = workloads.make_problem(3, 5, 64, 3)
    a = sumfac.assemble(prob).values
    b = sumfac.assemble(prob, flags=TWO_PASS).values
    print("p5 64^3 three-pass vs stage12:", float(torch.linalg.norm(a - b) / torch.linalg.norm(b)))
