"""3D assembly at p = 5, 6 — the three-pass path (csrc/assemble3d.cu: x pass
on DMMA over chunks of z layers, y sweep, z sweep; one direction per pass
like the reference's recursion, sumfac.py:200-213) against

* the oracle's independent Kronecker assembly (pattern identical, values
  within 1e-12 relative Frobenius) on tiny and ragged meshes,
* the fused stage-1/2 kernel (IGS_FLAG_TWO_PASS) and the generic kernels,
* itself on row ranges (partial layers, whole layers, single rows) and on
  slab coefficient fields (SURVEY §8e assembly partition),
* the stage-1/2 kernel at 64^3 (several G chunks).
"""

import ctypes

import numpy as np
import pytest

from oracle import igs_oracle as O

pytestmark = pytest.mark.gpu

TWO_PASS, GENERIC, THREE_PASS = 8, 1, 32


def _mods():
    from paper_1809_05471_b200 import sumfac, workloads

    return sumfac, workloads


def _problem(p, K, kind, seed):
    sumfac, workloads = _mods()
    from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule

    bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=seed)
    return sumfac.AssemblyProblem(bases, bases, quad, workloads.field_from_planes(3, kind, planes, quad.shape)), planes


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# (x points p·K0 even: the TMA row pitch must be a 16-byte multiple)
@pytest.mark.parametrize("p,K,kind", [
    (5, (2, 1, 1), 1), (5, (4, 3, 2), 3), (5, (6, 7, 5), 2), (5, (14, 3, 4), 3), (5, (2, 9, 3), 2),
    (6, (1, 1, 1), 3), (6, (2, 2, 3), 3), (6, (5, 4, 3), 2), (6, (9, 2, 2), 3), (6, (3, 7, 2), 1),
    # p = 3: the symmetric three-pass path is the default for whole symmetric matrices
    (3, (2, 1, 1), 3), (3, (8, 6, 7), 2), (3, (14, 5, 9), 3), (3, (4, 13, 2), 1),
])
def test_three_pass_vs_oracle_stage12_generic(cuda, p, K, kind):
    sumfac, workloads = _mods()
    prob, planes = _problem(p, K, kind, seed=61)
    assert sumfac.fused_path(prob) == 1
    va = sumfac.assemble(prob).values_np()
    vb = sumfac.assemble(prob, flags=TWO_PASS).values_np()
    vg = sumfac.assemble(prob, flags=GENERIC).values_np()
    sp = [O.uniform_space(p, k) for k in K]
    ths = O.first_order_set(3)
    Ar = O.assemble_kron(sp, sp, ths, ths, O.dense_field(planes.cpu().numpy(), O.plane_map(3, kind)))
    pairs = [O.pattern_1d(s.lo, s.hi, s.lo, s.hi, s.points) for s in sp]
    indptr, indices = O.tensor_csr(pairs, [s.num_basis for s in sp], [s.num_basis for s in sp])
    np.testing.assert_array_equal(prob.pattern().indptr, indptr)
    np.testing.assert_array_equal(prob.pattern().indices, indices)
    ref = O.values_on_pattern(Ar, indptr, indices)
    assert np.all(np.isfinite(va))
    assert _rel(va, ref) <= 1e-12
    assert _rel(va, vb) <= 1e-12
    assert _rel(va, vg) <= 1e-12


def test_three_pass_workspace_holds_the_g_chunk(cuda):
    sumfac, workloads = _mods()
    from paper_1809_05471_b200 import _lib

    prob, _ = _problem(5, (6, 5, 4), 3, seed=1)
    lib = _lib.load()
    st, keep = prob.struct(None)
    ws = lib.igs_workspace_bytes(ctypes.byref(st), _lib.OP_ASSEMBLE, 0)
    # H (4 groups) + one G chunk (9 groups, all z layers here) at least
    ns = [b.num_basis * 9 for b in prob.trial]
    assert ws >= 8 * (ns[0] * ns[1] * 20 * 4 + ns[0] * 25 * 20 * 9)


@pytest.mark.parametrize("p,K,kind", [(5, (4, 5, 9), 3), (6, (3, 2, 8), 2)])
def test_three_pass_row_ranges(cuda, p, K, kind):
    sumfac, workloads = _mods()
    from paper_1809_05471_b200.sumfac import _run_assembly

    prob, _ = _problem(p, K, kind, seed=62)
    full = sumfac.assemble(prob).values_np()
    pat = prob.pattern()
    nrows = pat.shape[0]
    layer = nrows // (K[-1] + p - 1)
    for cuts in ([0, nrows // 3, (2 * nrows) // 3, nrows], [0, 2 * layer, 5 * layer, nrows], [0, 1, nrows - 1, nrows]):
        parts = []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            vals = _run_assembly(prob, None, None, None, 0, (lo, hi)).cpu().numpy()
            parts.append(vals[: pat.indptr[hi] - pat.indptr[lo]])
        got = np.concatenate(parts)
        assert np.all(np.isfinite(got))
        assert _rel(got, full) <= 1e-13


@pytest.mark.parametrize("p,K,kind,world", [(5, 8, 3, 2), (6, 12, 2, 2)])
def test_three_pass_slab_assembly_matches_full(cuda, p, K, kind, world):
    sumfac, workloads = _mods()
    from paper_1809_05471_b200.sharded import SlabAssembly, SlabPartition
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    bases, quad = workloads.spaces(3, p, K)
    full_planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=9)
    full = AssemblyProblem(bases, bases, quad, workloads.field_from_planes(3, kind, full_planes, quad.shape))
    A = sumfac.assemble(full)
    layer_pts = quad.num_points // quad.shape[-1]
    part = SlabPartition(K, p, world)
    vals = []
    for r in range(world):
        sa = SlabAssembly(part, r)
        lo, hi = sa.halo_elements()
        planes = full_planes[:, lo * p * layer_pts: hi * p * layer_pts].contiguous()
        field = workloads.field_from_planes(3, kind, planes, quad.shape, slab=(lo, hi))
        v, ip, ix = sa.assemble(AssemblyProblem(bases, bases, quad, field))
        vals.append(v.cpu().numpy())
    got = np.concatenate(vals)
    assert got.shape == A.values_np().shape
    assert _rel(got, A.values_np()) <= 1e-13


def test_three_pass_full_size_p5_chunks_vs_stage12(cuda):
    """64^3 at p = 5 (207 M nnz): G goes through several z-layer chunks; the
    values equal the fused stage-1/2 kernel's to rounding and A = Aᵀ on a
    sample of entries."""
    import torch

    sumfac, workloads = _mods()
    prob = workloads.make_problem(3, 5, 64, 3, seed=4)
    a = sumfac.assemble(prob).values
    b = sumfac.assemble(prob, flags=TWO_PASS).values
    assert bool(torch.isfinite(a).all())
    assert float(torch.linalg.norm(a - b) / torch.linalg.norm(b)) <= 1e-13


@pytest.mark.parametrize("p,K", [(5, (4, 3, 2)), (6, (2, 3, 2))])
def test_three_pass_nonsymmetric_field(cuda, p, K):
    """A full first-order coefficient field with 16 distinct planes
    (reaction + convection in both slots + non-symmetric diffusion: A != Aᵀ):
    the three-pass path takes any block plan whose stage-2 groups hold at
    most 4 stage-1 groups; checked against the oracle's Kronecker assembly."""
    import torch

    sumfac, workloads = _mods()
    from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots
    from paper_1809_05471_b200.geometry import CoefficientField, first_order_derivative_set
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule

    bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    npts = int(np.prod(quad.shape))
    rng = np.random.default_rng(77)
    planes_np = 1.0 + 0.3 * rng.standard_normal((16, npts))
    plane_of = [[4 * i + j for j in range(4)] for i in range(4)]
    ths = first_order_derivative_set(3)
    field = CoefficientField.from_planes(ths, ths, torch.as_tensor(planes_np, device="cuda"), plane_of, quad.shape)
    prob = sumfac.AssemblyProblem(bases, bases, quad, field)
    assert sumfac.fused_path(prob) == 1
    va = sumfac.assemble(prob).values_np()
    vb = sumfac.assemble(prob, flags=TWO_PASS).values_np()
    sp = [O.uniform_space(p, k) for k in K]
    oths = O.first_order_set(3)
    Ar = O.assemble_kron(sp, sp, oths, oths, O.dense_field(planes_np, plane_of))
    pat = prob.pattern()
    ref = O.values_on_pattern(Ar, pat.indptr, pat.indices)
    assert _rel(va, ref) <= 1e-12
    assert _rel(va, vb) <= 1e-12
    S = sumfac.SparseMatrix(pat, torch.as_tensor(va, device="cuda")).to_scipy()
    assert (S - S.T).count_nonzero() > 0  # genuinely non-symmetric


@pytest.mark.parametrize("p,K,kind", [(3, (8, 5, 6), 3), (4, (6, 5, 7), 3), (4, (13, 4, 6), 2), (5, (4, 3, 2), 3)])
def test_three_pass_flag_forces_the_path(cuda, p, K, kind):
    """IGS_FLAG_THREE_PASS: the three-pass path at every instantiated order
    (p = 4 defaults to the one-pass kernel) equals the default path."""
    sumfac, workloads = _mods()
    prob, _ = _problem(p, K, kind, seed=63)
    va = sumfac.assemble(prob).values_np()
    vt = sumfac.assemble(prob, flags=THREE_PASS).values_np()
    vb = sumfac.assemble(prob, flags=TWO_PASS).values_np()
    assert np.all(np.isfinite(vt))
    assert _rel(vt, va) <= 1e-12
    assert _rel(vt, vb) <= 1e-12
