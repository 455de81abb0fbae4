"""Quick device timing of the fused apply / assembly (development aid)."""

import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import matfree, sumfac, workloads  # noqa: E402


def time_apply(name, K=None, reps=10, generic=False):
    c = workloads.CONFIGS[name]
    K = K or c["K"]
    t0 = time.time()
    prob = workloads.make_problem(c["d"], c["p"], K, c["kind"])
    op = matfree.MatrixFreeOperator(prob, force_generic=generic)
    n = prob.shape[1]
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        op.apply_device(x, y)
    torch.cuda.synchronize()
    setup = time.time() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        op.apply_device(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    f = prob.coeff
    npts = prob.quad.num_points
    balg = 8 * f.n_planes * npts + 16 * n
    print(f"{name} K={K} fused={op.fused and not generic}: {ms:.3f} ms/apply, {n / ms / 1e3:.1f} MDoF/s, "
          f"B_alg {balg / 1e9:.2f} GB -> {balg / ms / 1e6:.0f} GB/s (setup {setup:.1f}s)", flush=True)


def time_assemble(name, K=None, reps=10):
    c = workloads.CONFIGS[name]
    prob = workloads.make_problem(c["d"], c["p"], K or c["K"], c["kind"])
    for _ in range(3):
        A = sumfac.assemble(prob)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        A = sumfac.assemble(prob)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name} assemble fused={sumfac.fused_path(prob)}: {ms:.3f} ms, {A.nnz / ms / 1e6:.2f} Gnnz/s", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["C4", "C5"]
    for w in what:
        if w.startswith("asm"):
            time_assemble(w[3:])
        elif w.endswith("g"):
            time_apply(w[:-1], K=32, generic=True)
        else:
            time_apply(w)
