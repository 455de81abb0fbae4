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
