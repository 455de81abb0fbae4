"""Parity at BASELINE.json's full sizes (C2 / C3 assembly, C4 / C5 applies).

Every configuration is checked against the pinned oracle at its full size
(oracle/igs_oracle.py, on the same planes): C2 / C3 pattern identical and
values within 1e-12, C4 / C5 the whole production apply within 1e-12.
Besides, the size-independent properties the domain offers and a
full-width spot check of the slab path:
  * symmetry  v·(A u) = u·(A v) (the operators are symmetric),
  * linearity A(αu + βv) = αAu + βAv,
  * positivity u·(A u) > 0 (SPD / SPSD coefficients),
  * the fused slab apply at the full x-y size (every point of the first
    element layer(s), the slab path the multi-GPU partition uses) against
    the oracle's apply_slab on the same planes, 1e-12 relative,
  * C2 / C3: 1ᵀA1 = Σ_x w(x)·c(x) (the stiffness part annihilates
    constants); C3 also against the two-kernel fused path.
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


def _oracle_csr(d, p, K):
    sp = [O.uniform_space(p, K) for _ in range(d)]
    pairs = [O.pattern_1d(s.lo, s.hi, s.lo, s.hi, s.points) for s in sp]
    n = [s.num_basis for s in sp]
    indptr, indices = O.tensor_csr(pairs, n, n)
    return sp, indptr, indices


@pytest.mark.parametrize("name,d,p,K,kind,nnz", [("C2", 2, 5, 256, 2, 5_382_400),
                                                 ("C3", 3, 4, 64, 3, 95_443_993)])
def test_full_size_assembly_vs_oracle(cuda, name, d, p, K, kind, nnz):
    """BASELINE C2 / C3 at full size against the oracle's Alg. 1 restatement
    (oracle.assemble_sumfac: the reference's direction-by-direction scipy
    CSR x dense contraction, sumfac.py:200-229) on the same coefficient
    planes: CSR indptr / indices identical to the oracle's lexsorted tensor
    pattern (tensorspace.py:262-338), values within 1e-12 relative Frobenius.
    C3 runs the one-pass symmetric kernel, C2 the 2D fused path (its
    shared-band-table branch is taken at this size)."""
    torch = cuda
    matfree, sumfac, workloads = _mods()
    prob = workloads.make_problem(d, p, K, kind, seed=0)
    A = sumfac.assemble(prob)
    assert sumfac.fused_path(prob) == 1
    assert A.nnz == nnz
    sp, indptr, indices = _oracle_csr(d, p, K)
    pat = prob.pattern()
    np.testing.assert_array_equal(pat.indptr, indptr)
    np.testing.assert_array_equal(pat.indices, indices)
    del indices
    planes = prob.coeff.planes.cpu().numpy()
    ths = O.first_order_set(d)
    ref = O.assemble_sumfac(sp, sp, ths, ths, planes, O.plane_map(d, kind))
    vals = A.values_np()
    err = np.linalg.norm(vals - ref) / np.linalg.norm(ref)
    assert err <= 1e-12, f"{name}: rel Frobenius {err:.3e}"
    if d == 3:
        # the two-kernel fused path on the same problem (H through HBM)
        B = sumfac.assemble(prob, flags=8)
        err2 = float(torch.linalg.vector_norm(A.values - B.values) / torch.linalg.vector_norm(B.values))
        assert err2 <= 1e-12
        del B
    # measure identity 1ᵀA1 = Σ w c (mass part; the stiffness part annihilates constants)
    n = prob.shape[1]
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    total = float(torch.dot(one, A.matvec(one)))
    if kind & 1:
        w = torch.as_tensor(prob.quad.flat_weights(), device="cuda")
        assert abs(total - float(torch.dot(w, prob.coeff.planes[0]))) <= 1e-10
    else:
        assert abs(total) <= 1e-10 * float(torch.linalg.vector_norm(A.values))
    del A, prob
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name,p,kind", [("C4", 6, 2), ("C5", 8, 3)])
def test_full_size_apply_vs_oracle(cuda, name, p, kind):
    """BASELINE C4 / C5 at full size (128^3 elements) through the production
    multi-chunk fused apply (apply3d_kernel + apply_reduce_kernel) against the
    oracle's slab-wise Alg. 2/3 apply on the same planes,
    streamed to the host slab by slab: relative l2 <= 1e-12."""
    torch = cuda
    matfree, sumfac, workloads = _mods()
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    K, d = 128, 3
    bases, quad = workloads.spaces(d, p, K)
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=0)
    prob = AssemblyProblem(bases, bases, quad, workloads.field_from_planes(d, kind, planes, quad.shape))
    op = matfree.MatrixFreeOperator(prob)
    assert op.fused
    x = O.recipe_x(prob.shape[1], seed=0)
    y = op.apply_device(torch.as_tensor(x, device="cuda")).cpu().numpy()
    layer_pts = quad.num_points // quad.shape[-1]
    sp = [O.uniform_space(p, K) for _ in range(d)]
    ths = O.first_order_set(d)

    def slab(z0, z1):
        return planes[:, z0 * p * layer_pts: z1 * p * layer_pts].cpu().numpy()

    y_ref = O.apply(sp, p, ths, ths, O.plane_map(d, kind), None, x, slab=2, planes_fn=slab)
    err = np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref)
    assert err <= 1e-12, f"{name}: rel l2 {err:.3e}"
    del planes, prob, op
    torch.cuda.empty_cache()
