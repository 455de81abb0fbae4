"""Parity at BASELINE.json's full sizes (C2 / C3 assembly, C4 / C5 applies).

The oracle cannot run these sizes whole, so the checks are the
size-independent properties the domain offers, plus a full-width spot check
against the oracle on a z-slab:
  * symmetry  v·(A u) = u·(A v) (the operators are symmetric),
  * linearity A(αu + βv) = αAu + βAv,
  * positivity u·(A u) > 0 (SPD / SPSD coefficients),
  * the fused slab apply at the full x-y size (every point of the first
    element layer(s), the slab path the multi-GPU partition uses) against
    the oracle's apply_slab on the same planes, 1e-12 relative,
  * C3: the fused assembly against the independent stage-by-stage kernels,
    and 1ᵀA1 = Σ_x w(x)·c(x) (the stiffness part annihilates constants).
"""

import numpy as np
import pytest

from oracle import igs_oracle as O

pytestmark = pytest.mark.gpu


def _mods():
    from paper_1809_05471_b200 import matfree, sumfac, workloads

    return matfree, sumfac, workloads


@pytest.mark.parametrize("name,p,kind,slab_elems", [("C4", 6, 2, 2), ("C5", 8, 3, 1)])
def test_full_size_apply_properties_and_slab_spot_check(cuda, name, p, kind, slab_elems):
    torch = cuda
    matfree, sumfac, workloads = _mods()
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    K, d = 128, 3
    bases, quad = workloads.spaces(d, p, K)
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=0)
    prob = AssemblyProblem(bases, bases, quad, workloads.field_from_planes(d, kind, planes, quad.shape))
    op = matfree.MatrixFreeOperator(prob)
    assert op.fused
    n = prob.shape[1]
    g = torch.Generator(device="cuda").manual_seed(21)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    Au = op.apply_device(u)
    Av = op.apply_device(v)
    nrm = float(torch.linalg.vector_norm(u) * torch.linalg.vector_norm(Av))
    assert abs(float(torch.dot(v, Au) - torch.dot(u, Av))) <= 1e-12 * nrm
    w = 0.75 * u - 1.25 * v
    Aw = op.apply_device(w)
    lin = float(torch.linalg.vector_norm(Aw - (0.75 * Au - 1.25 * Av)) / torch.linalg.vector_norm(Aw))
    assert lin <= 1e-12
    assert float(torch.dot(u, Au)) > 0.0
    # full-width spot check on the first element layers (the slab path)
    layer_pts = quad.num_points // quad.shape[-1]
    layer_n = n // (K + p - 1)
    e0, e1 = 0, slab_elems
    sl = planes[:, e0 * p * layer_pts: e1 * p * layer_pts].contiguous()
    sop = matfree.MatrixFreeOperator(AssemblyProblem(
        bases, bases, quad, workloads.field_from_planes(d, kind, sl, quad.shape, slab=(e0, e1))))
    assert sop.fused
    xl = u[e0 * layer_n: (e1 + p - 1) * layer_n].contiguous()
    y_gpu = sop.apply_device(xl).cpu().numpy()
    sp = [O.uniform_space(p, K) for _ in range(d)]
    ths = O.first_order_set(d)
    x_full = u.cpu().numpy()
    y_ref = O.apply_slab(sp, p, ths, ths, O.plane_map(d, kind), sl.cpu().numpy(), x_full, e0, e1)
    assert np.linalg.norm(y_gpu - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
    del planes, prob, op, sop
    torch.cuda.empty_cache()


def test_full_size_c3_assembly_fused_vs_generic_and_measure(cuda):
    torch = cuda
    matfree, sumfac, workloads = _mods()
    prob = workloads.make_problem(3, 4, 64, workloads.MASS_STIFF, seed=0)
    A = sumfac.assemble(prob)
    assert sumfac.fused_path(prob) == 1
    assert A.nnz == 95_443_993
    B = sumfac.assemble(prob, flags=1)  # stage-by-stage kernels, independent of the fused family
    err = float(torch.linalg.vector_norm(A.values - B.values) / torch.linalg.vector_norm(B.values))
    assert err <= 1e-12
    del B
    n = prob.shape[1]
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    total = float(torch.dot(one, A.matvec(one)))
    c = prob.coeff.planes[0]
    w = torch.as_tensor(prob.quad.flat_weights(), device="cuda")
    assert abs(total - float(torch.dot(w, c))) <= 1e-10
    g = torch.Generator(device="cuda").manual_seed(3)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    Au, Av = A.matvec(u), A.matvec(v)
    nrm = float(torch.linalg.vector_norm(u) * torch.linalg.vector_norm(Av))
    assert abs(float(torch.dot(v, Au) - torch.dot(u, Av))) <= 1e-12 * nrm


def test_full_size_c2_assembly_fused_vs_generic(cuda):
    """C2 (d=2, p=5, 256², stiffness): the fused 2D path at a GPU-filling
    grid (shared precomputed band tables) against the stage kernels."""
    torch = cuda
    matfree, sumfac, workloads = _mods()
    prob = workloads.make_problem(2, 5, 256, workloads.STIFF, seed=0)
    A = sumfac.assemble(prob)
    assert sumfac.fused_path(prob) == 1
    assert A.nnz == 5_382_400
    B = sumfac.assemble(prob, flags=1)
    err = float(torch.linalg.vector_norm(A.values - B.values) / torch.linalg.vector_norm(B.values))
    assert err <= 1e-12
    n = prob.shape[1]
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    assert float(torch.linalg.vector_norm(A.matvec(one))) <= 1e-11 * float(torch.linalg.vector_norm(A.values))
