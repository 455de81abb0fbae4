"""The one-pass symmetric assemblies (csrc/asm3_sym.cuh, csrc/asm2_sym.cuh) against the oracle.

For symmetric problems (trial == test, first-order sets, F_{η,θ} = F_{θ,η})
the fused 3D assembly (asm3_sym) forms only the x-pairs with n0 >= m0 and writes each
value to its row and, mirrored, to the transposed entry.  Checked here:
  * pattern identical and values within 1e-12 (relative Frobenius) of the
    oracle's independent Kronecker assembly (sumfac.py:480-509 form) and of
    the two-kernel fused path (IGS_FLAG_TWO_PASS), on tiny and ragged meshes,
    p = 2 and 4, mass / stiffness / mass+stiffness;
  * A == Aᵀ bit for bit (each mirrored value is the same double);
  * any row range (whole or partial z layers, z chunks) equals the same rows
    of the full assembly bit for bit.
"""

import numpy as np
import pytest

from oracle import igs_oracle as O

pytestmark = pytest.mark.gpu

TWO_PASS = 8


def _mods():
    from paper_1809_05471_b200 import sumfac, workloads

    return sumfac, workloads


def _problem(p, K, kind, seed):
    sumfac, workloads = _mods()
    from paper_1809_05471_b200.bspline import UnivariateBasis, uniform_open_knots
    from paper_1809_05471_b200.quadrature import TensorQuadrature, per_element_rule

    d = len(K)
    bases = [UnivariateBasis(uniform_open_knots(p, k)) for k in K]
    quad = TensorQuadrature([per_element_rule(b.breakpoints, p) for b in bases])
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=seed)
    return sumfac.AssemblyProblem(bases, bases, quad, workloads.field_from_planes(d, kind, planes, quad.shape)), planes


def _rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("p,K,kind", [
    (4, (1, 1, 1), 3), (4, (2, 5, 1), 3), (4, (5, 3, 9), 2), (4, (9, 6, 3), 3), (4, (7, 7, 7), 1),
    (4, (13, 4, 6), 3), (4, (17, 9, 5), 2), (2, (13, 21, 2), 3), (2, (1, 3, 5), 1), (2, (8, 10, 9), 2),
    # 2D (asm2_sym: x strips sweeping y in chunks): tiny, ragged strips,
    # many chunks, all orders 2..5, mass / stiffness / mass+stiffness
    # (x points p·K0 even: the TMA row pitch must be a 16-byte multiple)
    (5, (2, 1), 2), (5, (2, 7), 3), (5, (20, 5), 2), (5, (38, 23), 3), (5, (40, 37), 2), (5, (64, 96), 2),
    (4, (1, 6), 1), (4, (24, 25), 3), (4, (31, 50), 2), (3, (64, 64), 1), (3, (34, 9), 3), (3, (70, 41), 2),
    (2, (48, 10), 3), (2, (50, 3), 1), (2, (97, 61), 2),
])
def test_sym_assembly_vs_oracle_and_two_pass(cuda, p, K, kind):
    sumfac, workloads = _mods()
    prob, planes = _problem(p, K, kind, seed=51)
    assert sumfac.fused_path(prob) == 1
    A = sumfac.assemble(prob)
    B = sumfac.assemble(prob, flags=TWO_PASS)
    d = len(K)
    sp = [O.uniform_space(p, k) for k in K]
    ths = O.first_order_set(d)
    Ar = O.assemble_kron(sp, sp, ths, ths, O.dense_field(planes.cpu().numpy(), O.plane_map(d, kind)))
    pairs = [O.pattern_1d(s.lo, s.hi, s.lo, s.hi, s.points) for s in sp]
    indptr, indices = O.tensor_csr(pairs, [s.num_basis for s in sp], [s.num_basis for s in sp])
    np.testing.assert_array_equal(prob.pattern().indptr, indptr)
    np.testing.assert_array_equal(prob.pattern().indices, indices)
    ref = O.values_on_pattern(Ar, indptr, indices)
    va = A.values_np()
    assert np.all(np.isfinite(va))
    assert _rel(va, ref) <= 1e-12
    assert _rel(va, B.values_np()) <= 1e-12
    S = A.to_scipy()
    assert (S - S.T).count_nonzero() == 0  # exactly symmetric


@pytest.mark.parametrize("p,K,kind", [(4, (6, 5, 11), 3), (4, (9, 4, 21), 2), (2, (9, 8, 13), 3)])
def test_sym_assembly_row_ranges_bit_identical(cuda, p, K, kind):
    sumfac, workloads = _mods()
    from paper_1809_05471_b200.sumfac import _run_assembly

    prob, _ = _problem(p, K, kind, seed=52)
    full = sumfac.assemble(prob).values_np()
    pat = prob.pattern()
    nrows = pat.shape[0]
    layer = nrows // (K[-1] + p - 1)
    for cuts in ([0, nrows // 3, (2 * nrows) // 3, nrows],             # partial layers
                 [0, 2 * layer, 5 * layer, nrows],                     # whole layers
                 [0, 1, nrows - 1, nrows]):                            # single rows
        parts = []
        for lo, hi in zip(cuts[:-1], cuts[1:]):
            vals = _run_assembly(prob, None, None, None, 0, (lo, hi)).cpu().numpy()
            a, b = pat.indptr[lo], pat.indptr[hi]
            parts.append(vals[: b - a])
        np.testing.assert_array_equal(np.concatenate(parts), full)


def test_sym_assembly_workspace_is_small_and_two_pass_still_available(cuda):
    """The one-pass kernel needs no intermediate in HBM: its workspace is the
    row-offset scalar; IGS_FLAG_TWO_PASS sizes the H round trip."""
    sumfac, workloads = _mods()
    import ctypes

    from paper_1809_05471_b200 import _lib

    prob = workloads.make_problem(3, 4, 12, workloads.MASS_STIFF, seed=3)
    lib = _lib.load()
    st, keep = prob.struct(None)
    one = lib.igs_workspace_bytes(ctypes.byref(st), _lib.OP_ASSEMBLE, 0)
    two = lib.igs_workspace_bytes(ctypes.byref(st), _lib.OP_ASSEMBLE, TWO_PASS)
    assert one <= 4096 < two
