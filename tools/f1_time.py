"""f1 at the C4 point grid (p=6, 128^3 elements, 768^3 Gauss points): the
twisted box pulled back (Laplace) by the fused kernel and by the two-step
pipeline, then one apply on the pulled-back planes.  Prints times and peak
device memory.  python tools/f1_time.py [K]"""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])

from paper_1809_05471_b200 import geometry as G  # noqa: E402
from paper_1809_05471_b200 import matfree, sumfac, workloads  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3, out


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    p = 6
    bases, quad = workloads.spaces(3, p, K)
    geo, pde = G.twisted_box(), G.pde_laplace()
    npts = quad.num_points
    torch.cuda.reset_peak_memory_stats()
    ms_f, field = timed(lambda: G.pull_back_fused(geo, quad, pde))
    peak_f = torch.cuda.max_memory_allocated() / 1e9
    planes_gb = field.planes.numel() * 8 / 1e9
    print(f"K={K} points={npts}: fused pullback {ms_f:.2f} ms, {planes_gb:.2f} GB planes "
          f"-> {planes_gb / ms_f:.2f} TB/s written, peak mem {peak_f:.1f} GB, planes {field.n_planes}", flush=True)
    prob = sumfac.AssemblyProblem(bases, bases, quad, field)
    op = matfree.MatrixFreeOperator(prob)
    x = torch.randn(prob.shape[1], dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    ms_a, _ = timed(lambda: op.apply_device(x, y), reps=5)
    print(f"apply on the pulled-back planes: {ms_a:.3f} ms ({prob.shape[1] / ms_a / 1e3:.1f} MDoF/s), "
          f"fused={op.fused}", flush=True)
    del field, prob, op
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    try:
        ms_t, f2 = timed(lambda: G.build_coefficient_field(G.eval_geometry(geo, quad), pde), reps=1)
        peak_t = torch.cuda.max_memory_allocated() / 1e9
        print(f"two-step (Alg. 3 field arrays + pullback): {ms_t:.2f} ms, peak mem {peak_t:.1f} GB", flush=True)
    except torch.cuda.OutOfMemoryError as exc:
        print(f"two-step: out of memory ({exc.__class__.__name__})")


if __name__ == "__main__":
    main()
