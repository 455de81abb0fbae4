"""Drop-in surface: every public name of the reference package's modules
(igasum.bspline / errors / geometry / quadrature / sumfac / tensorspace, the
operator API SURVEY §8(b) lists) exists under the same module name here,
plus the SPEC's matrix-free module.  The list was taken from the reference's
module bodies (public top-level functions and classes)."""

import importlib

import pytest

REFERENCE_PUBLIC = {
    "bspline": ["KnotVector", "uniform_open_knots", "UnivariateBasis", "find_span", "eval_all_derivs",
                "overlap_param", "BasisEvalTable", "tabulate"],
    "errors": ["DomainError", "UnsupportedDerivativeError", "CapacityError", "DegenerateGeometryError"],
    "geometry": ["first_order_derivative_set", "GeometryMap", "GeometryEvaluation", "eval_geometry", "PDEData",
                 "pde_mass", "pde_laplace", "pde_convection_diffusion", "named_pde", "CoefficientField",
                 "build_coefficient_field", "PulledBackCoefficient", "box_geometry", "identity_geometry",
                 "affine_geometry", "quarter_annulus", "twisted_box", "named_geometry"],
    "quadrature": ["ReferenceGaussRule", "gauss_legendre", "QuadratureRule1D", "per_element_rule", "custom_rule",
                   "TensorQuadrature"],
    "sumfac": ["FlopCounter", "SparseMatrix", "rel_frobenius", "AssemblyProblem", "assemble_block", "assemble",
               "assemble_naive", "assemble_kronecker_dense", "DEFAULT_NAIVE_BUDGET", "DEFAULT_DENSE_BUDGET"],
    "tensorspace": ["LexOrdering", "TensorGeneratingSystem", "contract_to_points", "nnz_pattern_1d",
                    "nnz_count_exact", "SparsityPattern", "tensor_pattern"],
    # SPEC-only: the matrix-free operator and localized strategies
    "matfree": ["MatrixFreeOperator", "apply", "eval_field"],
    "localized": ["make_partition", "assemble_localized", "apply_localized", "repetition_ratio"],
}


@pytest.mark.parametrize("module", sorted(REFERENCE_PUBLIC))
def test_public_names_present(module):
    mod = importlib.import_module(f"paper_1809_05471_b200.{module}")
    missing = [n for n in REFERENCE_PUBLIC[module] if not hasattr(mod, n)]
    assert not missing, f"{module}: missing {missing}"


def test_budgets_match_reference():
    from paper_1809_05471_b200 import sumfac

    assert sumfac.DEFAULT_NAIVE_BUDGET == 4_000_000_000
    assert sumfac.DEFAULT_DENSE_BUDGET == 100_000_000


# Public methods / properties of the reference's classes (taken from the class
# bodies of igasum.*; dataclass fields are instance attributes, not listed).
REFERENCE_CLASS_MEMBERS = {
    "bspline.KnotVector": ["multiplicity", "num_basis", "num_elements"],
    "bspline.UnivariateBasis": ["breakpoints", "csupp", "domain", "num_elements"],
    "bspline.BasisEvalTable": ["dense", "num_points", "point_matrix", "restrict"],
    "geometry.GeometryMap": ["d", "is_rational"],
    "geometry.GeometryEvaluation": ["d", "num_points"],
    "geometry.CoefficientField": ["block", "is_zero_block", "num_points", "restrict_flat"],
    "geometry.PulledBackCoefficient": ["evaluate"],
    "quadrature.QuadratureRule1D": ["num_points", "restrict"],
    "quadrature.TensorQuadrature": ["dim", "flat_weights", "num_points", "shape"],
    "sumfac.FlopCounter": ["add_block_update", "add_coeff_build", "add_field_eval", "as_tuple", "block_update",
                           "coeff_build", "field_eval", "merge", "total"],
    "sumfac.SparseMatrix": ["copy", "matvec", "nnz", "shape", "to_scipy", "toarray"],
    "sumfac.AssemblyProblem": ["coeff", "coeff_field", "core", "d", "pattern", "shape", "test_tables",
                               "trial_tables"],
    "tensorspace.LexOrdering": ["component", "d", "flatten", "size", "split"],
    "tensorspace.TensorGeneratingSystem": ["d", "dense_factor", "dims", "num_functions", "point_shape"],
    "tensorspace.SparsityPattern": ["d", "nnz", "shape", "to_scipy", "value_perm"],
}


@pytest.mark.parametrize("qual", sorted(REFERENCE_CLASS_MEMBERS))
def test_class_members_present(qual):
    module, cls = qual.split(".")
    mod = importlib.import_module(f"paper_1809_05471_b200.{module}")
    klass = getattr(mod, cls)
    missing = [n for n in REFERENCE_CLASS_MEMBERS[qual] if not hasattr(klass, n)]
    if missing and hasattr(klass, "__dataclass_fields__"):
        missing = [n for n in missing if n not in klass.__dataclass_fields__]
    assert not missing, f"{qual}: missing {missing}"


def test_value_perm_matches_layout():
    """SparsityPattern.value_perm maps the per-direction pair layout (first
    processed direction fastest) to CSR order, as tensorspace.py:324-332."""
    import numpy as np

    from paper_1809_05471_b200.tensorspace import DirectionPairs, SparsityPattern

    class _DP(DirectionPairs):
        def __init__(self, rp, n, nt):
            self._host = (np.asarray(rp), np.asarray(n), np.repeat(np.arange(len(rp) - 1), np.diff(rp)))
            self.num_trial = self.num_test = nt

        @property
        def num_pairs(self):
            return len(self._host[1])

    # 1D patterns |n - m| <= 1 on 3 functions, and on 2 functions (full)
    d0 = _DP([0, 2, 5, 7], [0, 1, 0, 1, 2, 1, 2], 3)
    d1 = _DP([0, 2, 4], [0, 1, 0, 1], 2)
    pat = SparsityPattern.__new__(SparsityPattern)
    from paper_1809_05471_b200.tensorspace import LexOrdering

    pat.dir_pairs = (d0, d1)
    pat.trial_ordering = pat.test_ordering = LexOrdering((3, 2))
    pat._host = {}
    for order in [(0, 1), (1, 0)]:
        perm = pat.value_perm(order)
        # layout entry -> (m_flat, n_flat), then sorted order must be CSR (row, col) ascending
        first, second = order
        mm, nn = [], []
        for a in range(d1.num_pairs if first == 0 else d0.num_pairs):
            for b in range(d0.num_pairs if first == 0 else d1.num_pairs):
                i0, i1 = (b, a) if first == 0 else (a, b)
                mm.append(d0.m[i0] + 3 * d1.m[i1])
                nn.append(d0.n[i0] + 3 * d1.n[i1])
        mm, nn = np.array(mm)[perm], np.array(nn)[perm]
        keys = mm * 6 + nn
        assert np.all(np.diff(keys) > 0) and len(perm) == 28
