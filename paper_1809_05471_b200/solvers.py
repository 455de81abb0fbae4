"""Conjugate gradients on the matrix-free operator.

The reference names Krylov solvers as the caller of the apply
but ships none.  This CG runs entirely on the device: one fused apply
(K4) per iteration plus a few vector updates; with a slab-partitioned
operator (sharded.ShardedApply) the dot products are all-reduced over the
process group (NCCL), which is the only collective the solver adds.
"""

import torch
import torch.distributed as dist


def _dot(a, b, group):
    s = torch.dot(a, b)
    if group is not None:
        dist.all_reduce(s, group=group)
    return s


def cg(apply, b, x0=None, tol=1e-10, maxiter=500, group=None):
    """Solve A x = b for SPD A given as `apply(x, out)`.

    Returns (x, iterations, relative residual).  `group` (a process group)
    makes the inner products global for slab-partitioned vectors.
    """
    x = torch.zeros_like(b) if x0 is None else x0.clone()
    r = b.clone()
    if x0 is not None:
        ax = torch.empty_like(b)
        apply(x, ax)
        r -= ax
    p = r.clone()
    ap = torch.empty_like(b)
    rr = _dot(r, r, group)
    bb = _dot(b, b, group)
    target = (tol * tol) * bb
    it = 0
    while it < maxiter and bool(rr > target):
        apply(p, ap)
        alpha = rr / _dot(p, ap, group)
        x.add_(alpha * p)
        r.sub_(alpha * ap)
        rr_new = _dot(r, r, group)
        p.mul_(rr_new / rr).add_(r)
        rr = rr_new
        it += 1
    return x, it, float(torch.sqrt(rr / bb))
