"""GPU tests of SPEC properties and edge cases beyond the golden vectors:
general spaces on the generic kernels (Petrov-Galerkin, reduced smoothness,
custom rules, convection), symmetry, measure identities, row-range and
slab (multi-GPU partition) execution, error behaviour."""

import numpy as np
import pytest

from oracle import igs_oracle as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den else 1.0)


def _mods():
    from paper_1809_05471_b200 import (bspline, geometry, matfree, quadrature, sumfac, tensorspace,
                                       workloads)

    return bspline, quadrature, tensorspace, geometry, sumfac, matfree, workloads


def _oracle_space(order, knots, points, weights):
    return O.Space1D(order, knots, points, weights, max_deriv=1)


def _dense_problem(trial_kv, test_kv, rules, F, theta, eta):
    bspline, quadrature, tensorspace, geometry, sumfac, matfree, workloads = _mods()
    trial = [bspline.UnivariateBasis(kv) for kv in trial_kv]
    test = [bspline.UnivariateBasis(kv) for kv in test_kv]
    quad = quadrature.TensorQuadrature(rules)
    field = geometry.CoefficientField(theta, eta, F, quad.shape)
    return sumfac.AssemblyProblem(trial, test, quad, field)


def _check_against_kron(prob, F, theta, eta):
    bspline, quadrature, tensorspace, geometry, sumfac, matfree, workloads = _mods()
    A = sumfac.assemble(prob)
    pat = prob.pattern()
    tr = [_oracle_space(b.order, b.kv.knots, r.points, r.weights) for b, r in zip(prob.trial, prob.quad.rules)]
    te = [_oracle_space(b.order, b.kv.knots, r.points, r.weights) for b, r in zip(prob.test, prob.quad.rules)]
    pairs = [O.pattern_1d(t.lo, t.hi, s.lo, s.hi, t.points) for t, s in zip(tr, te)]
    indptr, indices = O.tensor_csr(pairs, [t.num_basis for t in tr], [s.num_basis for s in te])
    np.testing.assert_array_equal(pat.indptr, indptr)
    np.testing.assert_array_equal(pat.indices, indices)
    Ar = O.assemble_kron(tr, te, theta, eta, F)
    vals = O.values_on_pattern(Ar, indptr, indices)
    assert rel(A.values_np(), vals) <= 1e-12
    return A, Ar


def test_petrov_galerkin_reduced_smoothness_and_convection(cuda):
    """Trial order 3 with double interior knots, test order 2, 2D, full
    first-order coupling with a non-symmetric F (convection)."""
    bspline, quadrature, *_ = _mods()
    tk = [bspline.uniform_open_knots(3, 4, interior_multiplicity=2), bspline.uniform_open_knots(3, 3)]
    sk = [bspline.uniform_open_knots(2, 4), bspline.uniform_open_knots(2, 3)]
    rules = [quadrature.per_element_rule(np.unique(k.knots), 3) for k in tk]
    theta = [(0, 0), (1, 0), (0, 1)]
    eta = [(0, 0), (1, 0), (0, 1)]
    npts = rules[0].num_points * rules[1].num_points
    F = np.random.default_rng(3).uniform(-1, 1, (npts, 3, 3))
    prob = _dense_problem(tk, sk, rules, F, theta, eta)
    _check_against_kron(prob, F, theta, eta)


def test_custom_rule_and_dir_order(cuda):
    bspline, quadrature, tensorspace, geometry, sumfac, *_ = _mods()
    kv = bspline.uniform_open_knots(3, 3)
    # trapezoid-like custom rule: still assembles, generic path
    pts = np.linspace(0.02, 0.98, 13)
    w = np.full(13, 1.0 / 13)
    rules = [quadrature.custom_rule(pts, w), quadrature.per_element_rule(np.unique(kv.knots), 2)]
    theta = eta = geometry.first_order_derivative_set(2)
    npts = 13 * rules[1].num_points
    F = np.zeros((npts, 3, 3))
    F[:, 0, 0] = 1.0
    F[:, 1, 1] = F[:, 2, 2] = 2.0
    prob = _dense_problem([kv, kv], [kv, kv], rules, F, theta, eta)
    A, _ = _check_against_kron(prob, F, theta, eta)
    B = sumfac.assemble(prob, dir_order=(1, 0))
    assert rel(B.values_np(), A.values_np()) <= 1e-13


@pytest.mark.parametrize("d,p,K,kind", [(2, 5, 12, 2), (3, 4, 6, 3), (2, 3, 9, 1), (3, 3, 5, 2)])
def test_symmetry_and_mass_total(cuda, d, p, K, kind):
    *_, sumfac, matfree, workloads = _mods()
    prob = workloads.make_problem(d, p, K, kind, seed=4)
    A = sumfac.assemble(prob).to_scipy()
    asym = (A - A.T)
    assert np.sqrt((asym.data ** 2).sum()) / np.sqrt((A.data ** 2).sum()) <= 1e-12
    if kind == 1:
        # c ~ U[0.5, 1.5] mass: 1ᵀ M 1 = ∫ c over the unit cube (quadrature)
        planes = prob.coeff.planes.cpu().numpy()[0]
        w = prob.quad.flat_weights()
        one = np.ones(A.shape[0])
        assert abs(one @ (A @ one) - np.dot(w, planes)) <= 1e-12


def test_assembly_row_ranges_match_full(cuda):
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    from paper_1809_05471_b200.sumfac import _run_assembly

    for (d, p, K, kind) in [(3, 4, 5, 3), (2, 5, 9, 2)]:
        prob = workloads.make_problem(d, p, K, kind, seed=8)
        full = sumfac.assemble(prob).values_np()
        pat = prob.pattern()
        nrows = pat.shape[0]
        cut = [0, nrows // 3, (2 * nrows) // 3, nrows]
        parts = []
        for lo, hi in zip(cut[:-1], cut[1:]):
            vals = _run_assembly(prob, None, None, None, 0, (lo, hi)).cpu().numpy()
            a, b = pat.indptr[lo], pat.indptr[hi]
            parts.append(vals[: b - a])
        np.testing.assert_array_equal(np.concatenate(parts), full)
    del torch


def test_max_nnz_capacity_error(cuda):
    *_, sumfac, matfree, workloads = _mods()
    from paper_1809_05471_b200.errors import CapacityError

    prob = workloads.make_problem(3, 4, 5, 3, max_nnz=1000)
    with pytest.raises(CapacityError):
        prob.pattern()


def test_apply_1d_and_2d_generic_against_oracle(cuda):
    *_, sumfac, matfree, workloads = _mods()
    for (d, p, K, kind) in [(1, 5, 20, 3), (2, 4, 10, 3)]:
        prob = workloads.make_problem(d, p, K, kind, seed=2)
        op = matfree.MatrixFreeOperator(prob)
        assert not op.fused
        x = O.recipe_x(prob.shape[1], seed=1)
        y = matfree.apply(op, x)
        sp = [O.uniform_space(p, K) for _ in range(d)]
        ths = O.first_order_set(d)
        y_ref = O.apply(sp, p, ths, ths, O.plane_map(d, kind), prob.coeff.planes.cpu().numpy(), x)
        assert rel(y, y_ref) <= 1e-12


@pytest.mark.parametrize("p,kind,world", [(6, 2, 3), (8, 3, 2), (4, 3, 4)])
def test_slab_partition_on_one_gpu(cuda, p, kind, world):
    """The multi-GPU decomposition executed slab by slab on one GPU with the
    halo exchange replaced by device copies: must equal the full apply."""
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    from paper_1809_05471_b200.sharded import SlabPartition
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    K = 16
    bases, quad = workloads.spaces(3, p, K)
    full_planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=5)
    full = AssemblyProblem(bases, bases, quad, workloads.field_from_planes(3, kind, full_planes, quad.shape))
    n = full.shape[1]
    layer_n = n // (K + p - 1)
    gen = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    y_full = matfree.MatrixFreeOperator(full).apply_device(x)
    part = SlabPartition(K, p, world)
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    layer_pts = quad.num_points // quad.shape[-1]
    for r in range(world):
        lo, hi = part.elements(r)
        planes = full_planes[:, lo * p * layer_pts: hi * p * layer_pts].contiguous()
        field = workloads.field_from_planes(3, kind, planes, quad.shape, slab=(lo, hi))
        prob = AssemblyProblem(bases, bases, quad, field)
        op = matfree.MatrixFreeOperator(prob)
        assert op.fused
        xl = x[lo * layer_n: (hi + p - 1) * layer_n].contiguous()
        yl = op.apply_device(xl)
        y[lo * layer_n: (hi + p - 1) * layer_n] += yl   # ghost reduce
    err = float(torch.linalg.vector_norm(y - y_full) / torch.linalg.vector_norm(y_full))
    assert err <= 1e-13


def test_apply_accumulate_flag_and_determinism(cuda):
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    prob = workloads.make_problem(3, 6, 9, 2, seed=12)
    op = matfree.MatrixFreeOperator(prob)
    n = prob.shape[1]
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    y1 = op.apply_device(x)
    y2 = op.apply_device(x)
    assert torch.equal(y1, y2), "fixed summation order: bit-reproducible"
    y3 = y1.clone()
    op.apply_device(x, y3, accumulate=True)
    assert torch.allclose(y3, 2 * y1, rtol=1e-15, atol=0)


def test_eval_field_partition_of_unity(cuda):
    *_, sumfac, matfree, workloads = _mods()
    torch = cuda
    prob = workloads.make_problem(3, 4, 5, 3)
    n = prob.shape[1]
    u = matfree.eval_field(prob, torch.ones(n, dtype=torch.float64, device="cuda"), (0, 0, 0))
    assert float(torch.abs(u - 1).max()) <= 1e-14
    du = matfree.eval_field(prob, torch.ones(n, dtype=torch.float64, device="cuda"), (1, 0, 0))
    assert float(torch.abs(du).max()) <= 1e-11


def test_cg_on_matrix_free_operator_and_matrix_market(cuda, tmp_path):
    """CG with the fused apply converges to the solution of the assembled
    system; the assembled matrix round-trips through MatrixMarket."""
    torch = cuda
    import scipy.io
    import scipy.sparse.linalg

    *_, sumfac, matfree, workloads = _mods()
    from paper_1809_05471_b200.solvers import cg

    prob = workloads.make_problem(3, 4, 6, workloads.MASS_STIFF, seed=3)
    op = matfree.MatrixFreeOperator(prob)
    assert op.fused
    n = prob.shape[1]
    b = torch.from_numpy(O.recipe_x(n, seed=9)).cuda()
    x, it, res = cg(lambda v, out: op.apply_device(v, out), b, tol=1e-11, maxiter=2000)
    assert res <= 1e-11 and it < 2000
    A = sumfac.assemble(prob)
    path = tmp_path / "c3_small.mtx"
    A.write_matrix_market(path)
    M = scipy.io.mmread(str(path)).tocsr()
    assert abs(M - A.to_scipy()).max() == 0.0
    r = M @ x.cpu().numpy() - b.cpu().numpy()
    assert np.linalg.norm(r) / np.linalg.norm(b.cpu().numpy()) <= 1e-10


@pytest.mark.parametrize("p,K,kind,world", [(4, 12, 3, 2), (4, 10, 3, 3), (3, 10, 2, 4)])
def test_slab_assembly_matches_full(cuda, p, K, kind, world):
    """SURVEY §8(e) assembly partition: each rank assembles its DoF-layer row
    block from the coefficients of its slab plus a (p-1)-element halo; the
    concatenated slices are bit-identical to the full assembly by the same
    kernels."""
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    from paper_1809_05471_b200.sharded import SlabAssembly, SlabPartition
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    bases, quad = workloads.spaces(3, p, K)
    full_planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=9)
    full = AssemblyProblem(bases, bases, quad, workloads.field_from_planes(3, kind, full_planes, quad.shape))
    A = sumfac.assemble(full)
    layer_pts = quad.num_points // quad.shape[-1]
    part = SlabPartition(K, p, world)
    vals, ptrs, cols = [], [], []
    for r in range(world):
        sa = SlabAssembly(part, r)
        lo, hi = sa.halo_elements()
        planes = full_planes[:, lo * p * layer_pts: hi * p * layer_pts].contiguous()
        field = workloads.field_from_planes(3, kind, planes, quad.shape, slab=(lo, hi))
        v, ip, ix = sa.assemble(AssemblyProblem(bases, bases, quad, field))
        vals.append(v.cpu().numpy())
        ptrs.append(ip.cpu().numpy() + (ptrs[-1][-1] if ptrs else 0))
        cols.append(ix.cpu().numpy())
    got = np.concatenate(vals)
    if p == 3:
        # whole symmetric matrices at p = 3 run the symmetric three-pass path,
        # row blocks the stage-1/2 kernels: bit-identical to the latter, equal
        # to rounding to the former
        np.testing.assert_array_equal(got, sumfac.assemble(full, flags=8).values_np())
        assert np.linalg.norm(got - A.values_np()) <= 1e-13 * np.linalg.norm(got)
    else:
        np.testing.assert_array_equal(got, A.values_np())
    indptr = np.concatenate([ptrs[0]] + [q[1:] for q in ptrs[1:]])
    np.testing.assert_array_equal(indptr, A.pattern.indptr)
    np.testing.assert_array_equal(np.concatenate(cols), A.pattern.indices)
    # a row range needing elements outside the slab is rejected
    sa = SlabAssembly(part, world - 1)
    lo, hi = sa.halo_elements()
    planes = full_planes[:, lo * p * layer_pts: (hi - 1) * p * layer_pts].contiguous()
    field = workloads.field_from_planes(3, kind, planes, quad.shape, slab=(lo, hi - 1))
    with pytest.raises(ValueError):
        sa.assemble(AssemblyProblem(bases, bases, quad, field))
    del torch


@pytest.mark.parametrize("p,kind", [(6, 2), (8, 3), (4, 3)])
def test_slab_interior_boundary_split_equals_slab_apply(cuda, p, kind):
    """The overlapped multi-GPU step computes a rank's slab as interior
    elements [lo, hi-p+1) (own x only) plus boundary elements [hi-p+1, hi)
    accumulated after the ghosts land; on planes views of one slab this
    must equal the slab apply."""
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    K, lo, hi = 16, 3, 13
    bases, quad = workloads.spaces(3, p, K)
    layer_pts = quad.num_points // quad.shape[-1]
    planes = workloads.synthetic_planes(3, list(quad.shape), kind, seed=6, z_range=(lo * p, hi * p))

    def op_on(a, b):
        view = planes[:, (a - lo) * p * layer_pts: (b - lo) * p * layer_pts]
        field = workloads.field_from_planes(3, kind, view, quad.shape, slab=(a, b))
        op = matfree.MatrixFreeOperator(AssemblyProblem(bases, bases, quad, field))
        assert op.fused
        return op

    layer_n = int(np.prod([b.num_basis for b in bases[:-1]]))
    n_loc = (hi - lo + p - 1) * layer_n
    gen = torch.Generator(device="cuda").manual_seed(3)
    x = torch.randn(n_loc, dtype=torch.float64, device="cuda", generator=gen)
    y_ref = op_on(lo, hi).apply_device(x)
    cut = hi - p + 1
    y = torch.zeros(n_loc, dtype=torch.float64, device="cuda")
    n_own = (hi - lo) * layer_n
    op_on(lo, cut).apply_device(x[:n_own], y[:n_own])
    b0 = (cut - lo) * layer_n
    op_on(cut, hi).apply_device(x[b0:], y[b0:], accumulate=True)
    err = float(torch.linalg.vector_norm(y - y_ref) / torch.linalg.vector_norm(y_ref))
    assert err <= 1e-13


def test_host_pipeline_matches_sequential_applies(cuda):
    """Overlapped host transfers (copy streams) give the same results as
    one apply after another."""
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    prob = workloads.make_problem(3, 4, 8, 3, seed=5)
    op = matfree.MatrixFreeOperator(prob)
    n = prob.shape[1]
    xs = [torch.randn(n, dtype=torch.float64).pin_memory() for _ in range(5)]
    ys = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(5)]
    pipe = matfree.HostPipeline(lambda x, y: op.apply_device(x, y), n, n)
    pipe.run(xs, ys)
    torch.cuda.synchronize()
    for xh, yh in zip(xs, ys):
        ref = op.apply_device(xh.cuda()).cpu()
        assert torch.equal(yh, ref)


def test_layers_copy_kernel_and_single_rank_sharded_apply(cuda):
    """K5 halo kernel (igs_layers_copy) behind sharded.layers_copy, and a
    world-1 ShardedApply (no exchange) equal to the plain apply."""
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    from paper_1809_05471_b200.sharded import ShardedApply, SlabPartition, layers_copy

    g = torch.Generator(device="cuda").manual_seed(5)
    a = torch.randn(1000, dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn(1000, dtype=torch.float64, device="cuda", generator=g)
    ref = a + b
    layers_copy(b, a, add=True)
    assert torch.equal(b, ref)
    layers_copy(b[:10], a[:10])
    assert torch.equal(b[:10], a[:10]) and torch.equal(b[10:], ref[10:])
    d, p, K = 3, 4, 5
    prob = workloads.make_problem(d, p, K, 3, seed=2)
    op = matfree.MatrixFreeOperator(prob)
    N = prob.shape[1]
    layer = N // (K + p - 1)
    x = torch.randn(N, dtype=torch.float64, device="cuda", generator=g)
    sh = ShardedApply(SlabPartition(K, p, 1), 0, layer, lambda xl, yl: op.apply_device(xl, yl), "cuda")
    y = torch.empty_like(x)
    sh.apply(x, y)
    assert torch.equal(y, op.apply_device(x, torch.empty_like(x)))


def test_assembly_kernel_only_flag(cuda):
    """IGS_FLAG_KERNEL_ONLY (measurement) runs the dominant assembly kernel
    alone and returns; the next full assembly is unaffected."""
    torch = cuda
    *_, sumfac, matfree, workloads = _mods()
    for d, p, K in [(3, 4, 6), (2, 5, 12)]:
        prob = workloads.make_problem(d, p, K, 3 if d == 3 else 2, seed=8)
        ref = sumfac.assemble(prob, flags=1).values_np()
        sumfac.assemble(prob, flags=4)
        torch.cuda.synchronize()
        assert rel(sumfac.assemble(prob).values_np(), ref) <= 1e-12
