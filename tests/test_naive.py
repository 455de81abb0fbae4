"""the reference's comparison oracles assemble_naive and
assemble_kronecker_dense (sumfac.py:388-509), on the device.

CPU: the oracle restatement of the dense Kronecker product and of the
naive update counter, pinned to the reference's own outputs
(tests/golden/naive_*, oracle/make_golden.py golden_naive).
GPU: igs_assemble_naive (direct quadrature per CSR entry) against the same
vectors, against Alg. 1 (fused and generic K3), and the budget guards.
Tolerance 1e-12 relative (north_star); counters exact."""

import numpy as np
import pytest

from conftest import golden
from oracle import igs_oracle as O


def rel(a, b):
    den = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (den if den else 1.0)


def _pg_spaces():
    tk = [O.uniform_open_knots(3, 4, interior_multiplicity=2), O.uniform_open_knots(3, 3)]
    sk = [O.uniform_open_knots(2, 4), O.uniform_open_knots(2, 3)]
    r0 = O.per_element_rule(np.unique(tk[0]), 3)
    r1 = (np.linspace(0.01, 0.99, 11), np.full(11, 1.0 / 11))
    tr = [O.Space1D(3, tk[0], *r0), O.Space1D(3, tk[1], *r1)]
    te = [O.Space1D(2, sk[0], *r0), O.Space1D(2, sk[1], *r1)]
    return tk, sk, tr, te


THETA = [(0, 0), (1, 0), (0, 1)]


def test_oracle_kron_and_counter_match_reference_pg():
    g = golden("naive_d2_pg")
    _, _, tr, te = _pg_spaces()
    A = O.assemble_kron(tr, te, THETA, THETA, g["F"])
    assert rel(A.toarray(), g["dense"]) <= 1e-13
    assert rel(O.values_on_pattern(A, g["indptr"], g["indices"]), g["values"]) <= 1e-13
    nb = int(np.sum(np.any(g["F"] != 0.0, axis=0)))
    assert O.naive_update_count(tr, te, g["indptr"], g["indices"], nb) == int(g["counter"][0])


def test_oracle_counter_matches_reference_d3():
    g = golden("naive_d3_p3")
    d, p, K, kind = (int(v) for v in g["meta"])
    sp = [O.uniform_space(p, K) for _ in range(d)]
    nb = sum(1 for i in range(d + 1) for j in range(d + 1) if O.plane_map(d, kind)[i][j] >= 0)
    assert O.naive_update_count(sp, sp, g["indptr"], g["indices"], nb) == int(g["counter"][0])


def _pkg():
    from paper_1809_05471_b200 import bspline, geometry, quadrature, sumfac, workloads

    return bspline, geometry, quadrature, sumfac, workloads


@pytest.mark.gpu
def test_naive_matches_reference_d3(cuda):
    bspline, geometry, quadrature, sumfac, workloads = _pkg()
    g = golden("naive_d3_p3")
    d, p, K, kind = (int(v) for v in g["meta"])
    bases, quad = workloads.spaces(d, p, K)
    planes = O.recipe_planes(d, list(quad.shape), p, kind)
    prob = workloads.make_problem(d, p, K, kind, planes=planes)
    counter = sumfac.FlopCounter()
    A = sumfac.assemble_naive(prob, counter)
    np.testing.assert_array_equal(A.pattern.indptr, g["indptr"])
    np.testing.assert_array_equal(A.pattern.indices, g["indices"])
    assert rel(A.values_np(), g["values"]) <= 1e-12
    assert counter.as_tuple() == tuple(int(v) for v in g["counter"])
    # independent of Alg. 1: agrees with the fused and the generic K3
    for flags in (0, 1):
        assert rel(sumfac.assemble(prob, flags=flags).values_np(), A.values_np()) <= 1e-12


@pytest.mark.gpu
def test_naive_and_dense_match_reference_petrov_galerkin(cuda):
    bspline, geometry, quadrature, sumfac, workloads = _pkg()
    g = golden("naive_d2_pg")
    tk = [bspline.uniform_open_knots(3, 4, interior_multiplicity=2), bspline.uniform_open_knots(3, 3)]
    sk = [bspline.uniform_open_knots(2, 4), bspline.uniform_open_knots(2, 3)]
    rules = [quadrature.per_element_rule(np.unique(tk[0].knots), 3),
             quadrature.custom_rule(np.linspace(0.01, 0.99, 11), np.full(11, 1.0 / 11))]
    quad = quadrature.TensorQuadrature(rules)
    field = geometry.CoefficientField(THETA, THETA, g["F"], quad.shape)
    prob = sumfac.AssemblyProblem([bspline.UnivariateBasis(k) for k in tk],
                                  [bspline.UnivariateBasis(k) for k in sk], quad, field)
    counter = sumfac.FlopCounter()
    A = sumfac.assemble_naive(prob, counter)
    np.testing.assert_array_equal(A.pattern.indptr, g["indptr"])
    np.testing.assert_array_equal(A.pattern.indices, g["indices"])
    assert rel(A.values_np(), g["values"]) <= 1e-12
    assert counter.as_tuple() == tuple(int(v) for v in g["counter"])
    D = sumfac.assemble_kronecker_dense(prob)
    assert D.shape == g["dense"].shape
    assert rel(D, g["dense"]) <= 1e-12
    assert np.all(D[g["dense"] == 0.0] == 0.0)
    assert rel(sumfac.assemble(prob).values_np(), A.values_np()) <= 1e-12


@pytest.mark.gpu
def test_naive_budgets(cuda):
    bspline, geometry, quadrature, sumfac, workloads = _pkg()
    from paper_1809_05471_b200.errors import CapacityError

    prob = workloads.make_problem(2, 3, 6, 3, seed=1)
    with pytest.raises(CapacityError):
        sumfac.assemble_naive(prob, budget=10)
    with pytest.raises(CapacityError):
        sumfac.assemble_kronecker_dense(prob, budget=10)
    A = sumfac.assemble_naive(prob)
    assert rel(sumfac.assemble(prob).values_np(), A.values_np()) <= 1e-12
    D = sumfac.assemble_kronecker_dense(prob)
    np.testing.assert_allclose(D, sumfac.assemble(prob).toarray(), rtol=0, atol=1e-13 * np.abs(D).max())
