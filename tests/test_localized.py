"""localized sum factorization.

CPU: partitions (strategies, remainders, fallback), the repetition ratio
(Eq. 20) and its Lemma 4.1 / 4.5 bounds, restricted bases.  GPU: localized
assembly and apply reproduce the global ones within 1e-12 for every
strategy (the SPEC's exactness property)."""

import math
import warnings
from fractions import Fraction

import numpy as np
import pytest


def _bases(d, p, K):
    from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots

    K = [K] * d if np.isscalar(K) else K
    return [UnivariateBasis(uniform_open_knots(p, k)) for k in K]


def test_partition_strategies_and_remainders():
    from paper_1809_05471_b200.localized import make_partition

    b = _bases(2, 3, 7)
    assert len(make_partition(_bases(2, 2, 4), "element")) == 16
    macro = make_partition(b, "macro")
    for i in range(len(macro)):
        assert all(s in (3, 4) for s in macro.sizes(i))   # SPEC example: sizes from {3, 4}, each >= 3
    narrow = make_partition(b, "narrow")
    for i in range(len(narrow)):
        s = narrow.sizes(i)
        assert s[1] == 1 and s[0] >= 3
    assert narrow.narrow == 1
    assert len(make_partition(b, "global")) == 1
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        small = make_partition(_bases(2, 4, 2), "macro")
    assert small.fallback and len(small) == 1 and w


def test_repetition_ratio_examples_and_lemma_bounds():
    from paper_1809_05471_b200.localized import RestrictedBasis, make_partition, repetition_ratio

    # SPEC: 1D order 2, 2 elements, per-element -> {phi_1, phi_2}, {phi_2, phi_3}, R = 4/3
    b1 = _bases(1, 2, 2)
    part = make_partition(b1, "element")
    rb = [RestrictedBasis(b1[0], *part.boxes[i][0]) for i in range(2)]
    assert [(r.offset, r.num_basis) for r in rb] == [(0, 2), (1, 2)]
    assert repetition_ratio(part, b1, b1) == Fraction(4, 3)
    assert repetition_ratio(make_partition(b1, "global"), b1, b1) == 1
    rng = np.random.default_rng(0)
    for d in (2, 3):
        for p in range(2, 6):
            bs = _bases(d, p, 3 * p + 1)
            # Example 4.3 / 4.4: per-element R <= p^d, macro (s = p) R <= 2^d
            assert repetition_ratio(make_partition(bs, "element"), bs, bs) <= p ** d
            # Lemma 4.1 for uniform box sizes s (remainders absorbed are >= s)
            for _ in range(3):
                s = [int(v) for v in rng.integers(p, 2 * p + 1, size=d)]
                part = make_partition(bs, "custom", sizes=s)
                if all((3 * p + 1) % v == 0 for v in s):
                    bound = math.prod(math.ceil((v + p - 1) / v) for v in s)
                    assert repetition_ratio(part, bs, bs) <= bound
            # Lemma 4.5: narrow partitions R <= 2^(d-1) d p
            assert repetition_ratio(make_partition(bs, "narrow"), bs, bs) <= 2 ** (d - 1) * d * p


@pytest.mark.gpu
@pytest.mark.parametrize("d,p,K,kind", [(2, 3, 6, 3), (3, 3, 5, 3), (3, 4, (6, 5, 4), 2), (2, 5, (7, 11), 2)])
@pytest.mark.parametrize("strategy", ["element", "macro", "narrow"])
def test_localized_assembly_and_apply_equal_global(cuda, d, p, K, kind, strategy):
    torch = cuda
    from paper_1809_05471_b200 import localized, matfree, sumfac, workloads
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule

    bases = _bases(d, p, K)
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=17)
    prob = sumfac.AssemblyProblem(bases, bases, quad, workloads.field_from_planes(d, kind, planes, quad.shape))
    A = sumfac.assemble(prob)
    part = localized.make_partition(bases, strategy)
    for policy in ("auto", "fixed"):
        B = localized.assemble_localized(prob, part, direction_policy=policy)
        v, w = B.values_np(), A.values_np()
        assert np.linalg.norm(v - w) <= 1e-12 * np.linalg.norm(w)
    n = prob.shape[1]
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    y = matfree.MatrixFreeOperator(prob).apply_device(x)
    yl = localized.apply_localized(prob, part, x)
    assert float(torch.linalg.vector_norm(yl - y) / torch.linalg.vector_norm(y)) <= 1e-12
    assert float(torch.linalg.vector_norm(localized.apply_localized(prob, part, torch.zeros_like(x)))) == 0.0
    # counted MACs: the sum of the per-box applies' counts
    from paper_1809_05471_b200.localized import restrict, _local_field

    c = sumfac.FlopCounter()
    localized.apply_localized(prob, part, x, counter=c)
    want = sumfac.FlopCounter()
    for i in range(len(part)):
        ls = restrict(prob.trial, prob.test, prob.quad, part, i)
        matfree.MatrixFreeOperator(sumfac.AssemblyProblem(ls.trial, ls.test, ls.quad,
                                                          _local_field(prob, ls))).count(want)
    assert c == want and c.total > 0


@pytest.mark.gpu
def test_localized_flop_counts_grow_like_the_paper(cuda):
    """Counted assembly MACs on a fixed 2D mesh: per-element grows ~p^(2d+1),
    macro-standard ~p^(d+2) (Examples 4.3/4.4): the fitted exponents are
    ordered and within the SPEC's ±0.5 window."""
    from paper_1809_05471_b200 import localized, sumfac, workloads
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule

    d, K = 2, 24
    ps = [2, 3, 4, 5, 6]
    costs = {"element": [], "macro": []}
    for p in ps:
        bases = _bases(d, p, K)
        quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
        prob = workloads.make_problem(d, p, K, workloads.MASS)
        for strat in costs:
            c = sumfac.FlopCounter()
            localized.assemble_localized(prob, localized.make_partition(bases, strat), counter=c)
            costs[strat].append(c.block_update)
        del quad
    slope = {s: np.polyfit(np.log(ps), np.log(np.array(v, dtype=float)), 1)[0] for s, v in costs.items()}
    assert abs(slope["element"] - (2 * d + 1)) <= 0.5, slope
    assert abs(slope["macro"] - (d + 2)) <= 0.5, slope
