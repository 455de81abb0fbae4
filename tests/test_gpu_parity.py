"""GPU parity: the CUDA path (through the C-ABI) against the reference's own
outputs (tests/golden, made by oracle/make_golden.py from the reference
package) and against the oracle restatement.

Tolerances: tables 1e-14 absolute; assembled values and applies 1e-12
relative (north_star); CSR patterns identical.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import igs_oracle as O

pytestmark = pytest.mark.gpu


def _pkg():
    from paper_1809_05471_b200 import bspline, matfree, quadrature, sumfac, tensorspace, workloads

    return bspline, quadrature, tensorspace, sumfac, matfree, workloads


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den else 1.0)


# ---------------------------------------------------------------- K1 ------

def test_gauss_rules_match_reference(cuda):
    _, quadrature, *_ = _pkg()
    g = golden("gauss")
    for k in range(1, 17):
        r = quadrature.gauss_legendre(k)
        assert np.max(np.abs(r.nodes - g[f"nodes_{k}"])) <= 1e-15
        assert np.max(np.abs(r.weights - g[f"weights_{k}"])) <= 1e-14
    r = quadrature.per_element_rule([0.0, 0.25, 0.5, 0.75, 1.0], 3)
    assert np.max(np.abs(r.points - g["pe_points"])) <= 1e-15
    assert np.max(np.abs(r.weights - g["pe_weights"])) <= 1e-15


def test_tabulate_matches_reference(cuda):
    bspline, *_ = _pkg()
    g = golden("tabulate")
    for c in range(int(g["ncases"][0])):
        p, K, md = g[f"c{c}_meta"]
        kv = bspline.KnotVector(int(p), g[f"c{c}_knots"])
        b = bspline.UnivariateBasis(kv)
        t = bspline.tabulate(b, g[f"c{c}_points"], int(md))
        np.testing.assert_array_equal(t.first_active_np(), g[f"c{c}_first"])
        scale = np.maximum(1.0, np.abs(g[f"c{c}_values"]))
        assert np.max(np.abs(t.values_np() - g[f"c{c}_values"]) / scale) <= 1e-13, c


def test_tabulate_errors(cuda):
    bspline, *_ = _pkg()
    from paper_1809_05471_b200.errors import DomainError, UnsupportedDerivativeError

    b = bspline.UnivariateBasis(bspline.uniform_open_knots(3, 4))
    with pytest.raises(DomainError):
        bspline.tabulate(b, [0.5, 1.5], 1)
    with pytest.raises(UnsupportedDerivativeError):
        bspline.tabulate(b, [0.5], 3)
    with pytest.raises(ValueError):
        bspline.tabulate(b, [0.6, 0.5], 1)


def test_eval_all_derivs_known_answer(cuda):
    bspline, *_ = _pkg()
    b = bspline.UnivariateBasis(bspline.KnotVector(2, [0.0, 0.0, 1.0, 1.0]))
    first, ders = bspline.eval_all_derivs(b, 0.5, 1)
    assert first == 0
    np.testing.assert_allclose(ders[0], [0.5, 0.5], atol=0)
    np.testing.assert_allclose(ders[1], [-1.0, 1.0], atol=0)


# ---------------------------------------------------------------- K2 ------

def test_pattern_1d_matches_reference(cuda):
    bspline, quadrature, tensorspace, *_ = _pkg()
    g = golden("pattern")
    for c in range(int(g["ncases"][0])):
        pt, Kt, ps, Ks, mt, ms, k = (int(v) for v in g[f"c{c}_meta"])
        bt = bspline.UnivariateBasis(bspline.uniform_open_knots(pt, Kt, interior_multiplicity=mt))
        bs = bspline.UnivariateBasis(bspline.uniform_open_knots(ps, Ks, interior_multiplicity=ms))
        rule = quadrature.per_element_rule(np.union1d(bt.breakpoints, bs.breakpoints), k)
        pairs = tensorspace.nnz_pattern_1d(bt, bs, rule)
        np.testing.assert_array_equal(pairs, g[f"c{c}_pairs"])
        assert tensorspace.nnz_count_exact(bt, bs) == int(g[f"c{c}_count"][0])


# ---------------------------------------------------------------- K3 ------

ASM_CASES = ["c1_full", "c2_reduced", "c3_reduced", "d1_mk", "d3_p2"]


def _golden_problem(g, workloads):
    d, p, K, kind = (int(v) for v in g["meta"])
    bases, quad = workloads.spaces(d, p, K)
    planes = O.recipe_planes(d, list(quad.shape), p, kind)
    np.testing.assert_allclose([planes.sum(), (planes ** 2).sum()], g["planes_sum"], rtol=1e-13)
    return workloads.make_problem(d, p, K, kind, planes=planes), planes


@pytest.mark.parametrize("name", ASM_CASES)
@pytest.mark.parametrize("generic", [False, True])
def test_assembly_matches_reference(cuda, name, generic):
    *_, sumfac, matfree, workloads = _pkg()
    g = golden(f"asm_{name}")
    prob, _ = _golden_problem(g, workloads)
    counter = sumfac.FlopCounter()
    A = sumfac.assemble(prob, counter, flags=1 if generic else 0)
    pat = prob.pattern()
    np.testing.assert_array_equal(pat.indptr, g["indptr"])
    np.testing.assert_array_equal(pat.indices, g["indices"])
    assert rel(A.values_np(), g["values"]) <= 1e-12
    assert counter.as_tuple() == tuple(int(v) for v in g["counter"])


def test_assemble_block_and_dir_order(cuda):
    *_, sumfac, matfree, workloads = _pkg()
    from paper_1809_05471_b200.geometry import first_order_derivative_set

    g = golden("blocks_d3_p3")
    d, p, K, kind = (int(v) for v in g["meta"])
    bases, quad = workloads.spaces(d, p, K)
    planes = O.recipe_planes(d, list(quad.shape), p, kind)
    prob = workloads.make_problem(d, p, K, kind, planes=planes)
    ths = first_order_derivative_set(3)
    blk = sumfac.assemble_block(prob, ths[1], ths[2])
    assert rel(blk.values_np(), g["block_12"]) <= 1e-12
    perm = sumfac.assemble(prob, dir_order=(2, 0, 1))
    assert rel(perm.values_np(), g["perm_201"]) <= 1e-12


# ---------------------------------------------------------------- K4 ------

APPLY_CASES = ["c4_reduced", "c5_reduced", "c3_small", "d2_stiff"]


@pytest.mark.parametrize("name", APPLY_CASES)
@pytest.mark.parametrize("generic", [False, True])
def test_apply_matches_reference_matvec(cuda, name, generic):
    *_, sumfac, matfree, workloads = _pkg()
    g = golden(f"apply_{name}")
    prob, _ = _golden_problem(g, workloads)
    op = matfree.MatrixFreeOperator(prob, force_generic=generic)
    y = matfree.apply(op, g["x"])
    assert rel(y, g["y"]) <= 1e-12


def test_apply_zero_and_mass_identity(cuda):
    *_, sumfac, matfree, workloads = _pkg()
    torch = cuda
    prob = workloads.make_problem(3, 4, 6, workloads.MASS_STIFF)
    op = matfree.MatrixFreeOperator(prob)
    n = prob.shape[1]
    y0 = matfree.apply(op, torch.zeros(n, dtype=torch.float64, device="cuda"))
    assert float(torch.abs(y0).max()) == 0.0
    # pure mass with c = 1: sum of A·1 = measure of the unit cube
    bases, quad = workloads.spaces(3, 4, 6)
    ones = torch.ones((1, quad.num_points), dtype=torch.float64, device="cuda")
    pm = workloads.field_from_planes(3, workloads.MASS, ones, quad.shape)
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    mp = AssemblyProblem(bases, bases, quad, pm)
    v = matfree.apply(matfree.MatrixFreeOperator(mp), np.ones(mp.shape[1]))
    assert abs(v.sum() - 1.0) <= 1e-12


def test_apply_linearity(cuda):
    *_, sumfac, matfree, workloads = _pkg()
    torch = cuda
    prob = workloads.make_problem(3, 6, 8, workloads.STIFF)
    op = matfree.MatrixFreeOperator(prob)
    n = prob.shape[1]
    gen = torch.Generator(device="cuda").manual_seed(3)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    w = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    a, b = 0.7, -1.3
    lhs = op.apply_device(a * u + b * w)
    rhs = a * op.apply_device(u) + b * op.apply_device(w)
    assert float(torch.linalg.vector_norm(lhs - rhs) / torch.linalg.vector_norm(rhs)) <= 1e-12


def test_apply_against_oracle_synthetic(cuda):
    """Device-generated coefficients, regenerated on the host by the oracle's
    mirror of the counter RNG; compare with the oracle's slab-wise apply."""
    *_, sumfac, matfree, workloads = _pkg()
    for (d, p, K, kind) in [(3, 6, 10, 2), (3, 8, 6, 3), (3, 4, 9, 3)]:
        prob = workloads.make_problem(d, p, K, kind, seed=11)
        op = matfree.MatrixFreeOperator(prob)
        x = O.recipe_x(prob.shape[1], seed=5)
        y = matfree.apply(op, x)
        sp = [O.uniform_space(p, K) for _ in range(d)]
        shape = [p * K] * d
        planes = O.synthetic_planes(d, shape, 0, shape[-1], kind, seed=11)
        np.testing.assert_allclose(planes, prob.coeff.planes.cpu().numpy(), rtol=1e-14, atol=1e-15)
        ths = O.first_order_set(d)
        y_ref = O.apply(sp, p, ths, ths, O.plane_map(d, kind), planes, x)
        assert rel(y, y_ref) <= 1e-12


@pytest.mark.parametrize("p", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("kind", [1, 2, 3])
def test_fused_apply_all_orders_vs_oracle(cuda, p, kind):
    """Every fused instantiation (orders 2..8, mass / stiffness / both) on a
    mesh whose element counts are not multiples of the tile, against the
    oracle; also checks the fused path was actually taken when supported."""
    *_, sumfac, matfree, workloads = _pkg()
    K = (11, 6, 9)
    from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=21)
    field = workloads.field_from_planes(3, kind, planes, quad.shape)
    prob = AssemblyProblem(bases, bases, quad, field)
    op = matfree.MatrixFreeOperator(prob)
    x = O.recipe_x(prob.shape[1], seed=6)
    y = matfree.apply(op, x)
    sp = [O.uniform_space(p, k) for k in K]
    ths = O.first_order_set(3)
    y_ref = O.apply(sp, p, ths, ths, O.plane_map(3, kind), planes.cpu().numpy(), x)
    assert rel(y, y_ref) <= 1e-12
    # TMA needs 16-byte rows: the fused kernel serves every order except 7
    # whenever the x point count is even (else the generic kernels run)
    if p != 7 and (p * K[0]) % 2 == 0:
        assert op.fused, f"fused path expected for p={p}"


@pytest.mark.parametrize("p,K", [(2, (1, 1, 1)), (4, (1, 2, 3)), (6, (2, 1, 5)), (8, (3, 2, 1)), (7, (2, 4, 2)),
                                 (6, (24, 17, 2))])
@pytest.mark.parametrize("kind", [2, 3])
def test_apply_tiny_and_ragged_meshes_vs_oracle(cuda, p, K, kind):
    """Meshes smaller than one tile (every element masked but one) and tiles
    cut by the mesh edge in every direction: fused (when the x rows are
    16-byte aligned) and generic paths against the oracle."""
    *_, sumfac, matfree, workloads = _pkg()
    from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=31)
    prob = AssemblyProblem(bases, bases, quad, workloads.field_from_planes(3, kind, planes, quad.shape))
    x = O.recipe_x(prob.shape[1], seed=8)
    sp = [O.uniform_space(p, k) for k in K]
    ths = O.first_order_set(3)
    y_ref = O.apply(sp, p, ths, ths, O.plane_map(3, kind), planes.cpu().numpy(), x)
    for generic in (False, True):
        op = matfree.MatrixFreeOperator(prob, force_generic=generic)
        assert rel(matfree.apply(op, x), y_ref) <= 1e-12
        if not generic and (p * K[0]) % 2 == 0:
            assert op.fused


@pytest.mark.parametrize("d,p,K,kind", [(3, 2, (1, 1, 1), 3), (3, 4, (1, 2, 3), 3), (3, 3, (2, 5, 1), 2),
                                        (3, 5, (2, 1, 2), 3), (3, 6, (1, 1, 2), 2), (2, 5, (1, 3), 3),
                                        (2, 4, (9, 1), 1), (3, 3, (14, 9, 3), 3), (3, 2, (13, 21, 2), 3),
                                        (3, 4, (9, 6, 3), 3)])
def test_assembly_tiny_and_ragged_meshes_vs_oracle(cuda, d, p, K, kind):
    """Assembly on meshes smaller than one row tile and on ragged multi-tile
    meshes (the wide p = 2, 3 tiles included), fused and generic, against
    the oracle's independent Kronecker assembly (pattern identical)."""
    *_, sumfac, matfree, workloads = _pkg()
    from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=41)
    prob = AssemblyProblem(bases, bases, quad, workloads.field_from_planes(d, kind, planes, quad.shape))
    sp = [O.uniform_space(p, k) for k in K]
    ths = O.first_order_set(d)
    F = O.dense_field(planes.cpu().numpy(), O.plane_map(d, kind))
    Ar = O.assemble_kron(sp, sp, ths, ths, F)
    pairs = [O.pattern_1d(s.lo, s.hi, s.lo, s.hi, s.points) for s in sp]
    indptr, indices = O.tensor_csr(pairs, [s.num_basis for s in sp], [s.num_basis for s in sp])
    ref = O.values_on_pattern(Ar, indptr, indices)
    for generic in (False, True):
        A = sumfac._run_assembly(prob, None, None, None, 1 if generic else 0)
        np.testing.assert_array_equal(prob.pattern().indptr, indptr)
        assert rel(A.cpu().numpy(), ref) <= 1e-12
