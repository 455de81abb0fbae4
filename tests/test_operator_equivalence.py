"""SPEC.md:472 operator equivalence and the reference's rel_frobenius.

* For 50 random vectors per configuration, ||apply(u) - A·u|| / ||A·u||
  <= 1e-12, A the assembled matrix (the apply-shaped BASELINE configs at
  reduced K with their own p and coefficient kind, plus C3's shape).
* rel_frobenius (sumfac.py:118-141): value-array distance for a shared
  pattern, densified distance otherwise, 0 / inf for a zero reference.
"""

import numpy as np
import pytest
import scipy.sparse

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("d,p,K,kind", [(3, 6, 6, 2), (3, 8, 4, 3), (3, 4, 7, 3), (2, 5, 12, 2)])
def test_apply_equals_assembled_matvec_50_vectors(cuda, d, p, K, kind):
    torch = cuda
    from paper_1809_05471_b200 import matfree, sumfac, workloads

    prob = workloads.make_problem(d, p, K, kind, seed=77)
    A = sumfac.assemble(prob)
    op = matfree.MatrixFreeOperator(prob)
    n = prob.shape[1]
    g = torch.Generator(device="cuda").manual_seed(5)
    U = torch.randn(n, 50, dtype=torch.float64, device="cuda", generator=g)
    AU = A.pattern.to_torch(A.values) @ U
    worst = 0.0
    for j in range(50):
        y = op.apply_device(U[:, j].contiguous())
        ref = AU[:, j]
        worst = max(worst, float(torch.linalg.vector_norm(y - ref) / torch.linalg.vector_norm(ref)))
    assert worst <= 1e-12, worst


def test_rel_frobenius_semantics(cuda):
    torch = cuda
    from paper_1809_05471_b200 import sumfac, workloads

    prob = workloads.make_problem(3, 3, 4, workloads.MASS_STIFF, seed=2)
    A = sumfac.assemble(prob)
    B = A.copy()
    B.values[::7] *= 1.0 + 1e-9
    # shared pattern: distance of the value arrays
    va, vb = A.values_np(), B.values_np()
    want = np.linalg.norm(va - vb) / np.linalg.norm(vb)
    assert sumfac.rel_frobenius(A, B) == pytest.approx(want, rel=1e-12)
    assert sumfac.rel_frobenius(A, A) == 0.0
    # anything else is densified: scipy and numpy operands give the same number
    Sa, Sb = A.to_scipy(), B.to_scipy()
    dense = np.linalg.norm((Sa - Sb).toarray()) / np.linalg.norm(Sb.toarray())
    assert sumfac.rel_frobenius(Sa, B) == pytest.approx(dense, rel=1e-12)
    assert sumfac.rel_frobenius(A, Sb.toarray()) == pytest.approx(dense, rel=1e-12)
    # zero reference: 0 when equal, inf otherwise
    Z = scipy.sparse.csr_matrix(Sa.shape)
    assert sumfac.rel_frobenius(Z, Z) == 0.0
    assert sumfac.rel_frobenius(Sa, Z) == np.inf
    del torch
