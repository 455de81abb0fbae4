"""Fused apply across spline orders at 128³ elements (p Gauss points per
direction): device ms per apply, DoF/s and B_alg/(t·6544 GB/s), for
stiffness and mass+stiffness.  Also the fused assembly at 64³ for p=2..6.
python tools/order_sweep.py > profiles/r01/order_sweep.txt"""

import sys

import torch

sys.path.insert(0, ".")
from paper_1809_05471_b200 import matfree, sumfac, workloads  # noqa: E402

BW = 6544.3e9
P64 = 37.14e12  # sustained DMMA peak, profiles/fp64_peak.json


def _ref_frac(prob, A, ms):
    """Reference-equivalent roofline fraction of an assembly:
    max(F_ref / (t·P64), B_alg / (t·BW)) with F_ref = 2 x the reference
    FlopCounter's block-update MACs and B_alg = planes read + values written."""
    c = sumfac.FlopCounter()
    sumfac.assemble(prob, counter=c)
    t = ms / 1e3
    f_ref = 2.0 * c.block_update
    b_alg = 8.0 * prob.coeff.n_planes * prob.quad.num_points + 8.0 * A.nnz
    return f_ref, max(f_ref / t / P64, b_alg / t / BW)


def apply_row(p, kind, K=128, reps=10):
    prob = workloads.make_problem(3, p, K, kind)
    op = matfree.MatrixFreeOperator(prob)
    n = prob.shape[1]
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        op.apply_device(x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        op.apply_device(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    balg = 8 * prob.coeff.n_planes * prob.quad.num_points + 16 * n
    print(f"apply p={p} kind={'K' if kind == 2 else 'M+K'} 128^3: {ms:8.3f} ms  {n / ms / 1e3:7.1f} MDoF/s  "
          f"B_alg {balg / 1e9:6.2f} GB  frac {balg / (ms / 1e3) / BW:.3f}  fused={op.fused}", flush=True)
    del prob, op, x, y
    torch.cuda.empty_cache()


def asm_row(p, kind, K=64, reps=10):
    prob = workloads.make_problem(3, p, K, kind, max_nnz=1 << 40)
    for _ in range(3):  # warm: allocator, launch data, clocks
        A = sumfac.assemble(prob)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        A = sumfac.assemble(prob)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    f_ref, frac = _ref_frac(prob, A, ms)
    print(f"assemble p={p} kind={'K' if kind == 2 else 'M+K'} 64^3: {ms:8.3f} ms  {A.nnz / ms / 1e6:6.2f} G nnz/s  "
          f"nnz {A.nnz}  F_ref {f_ref / 1e9:7.2f} GFLOP  frac_ref {frac:.3f}  fused={sumfac.fused_path(prob)}", flush=True)
    del prob, A
    torch.cuda.empty_cache()


def asm2_row(p, kind, K=256, reps=20):
    prob = workloads.make_problem(2, p, K, kind, max_nnz=1 << 40)
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
    f_ref, frac = _ref_frac(prob, A, ms)
    print(f"assemble2d p={p} kind={'K' if kind == 2 else 'M+K'} 256^2: {ms:8.3f} ms  {A.nnz / ms / 1e6:6.2f} G nnz/s  "
          f"nnz {A.nnz}  F_ref {f_ref / 1e9:7.2f} GFLOP  frac_ref {frac:.3f}  fused={sumfac.fused_path(prob)}", flush=True)
    del prob, A
    torch.cuda.empty_cache()


if __name__ == "__main__":
    # small assemblies first (the large apply problems fragment the allocator)
    for p in range(2, 7):
        asm2_row(p, 2)
    for p in range(2, 7):
        asm_row(p, 3)
    for kind in (2, 3):
        for p in range(2, 9):
            apply_row(p, kind)
