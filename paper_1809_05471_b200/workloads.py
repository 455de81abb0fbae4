"""The BASELINE.json workloads (C1..C5) and their seeded synthetic inputs.

C1  d=2 mass assembly,          p=3, 64^2 elements
C2  d=2 stiffness assembly,     p=5, 256^2 elements
C3  d=3 mass+stiffness assembly, p=4, 64^3 elements
C4  d=3 stiffness apply,        p=6, 128^3 elements, 100 applies
C5  d=3 mass+stiffness apply,   p=8, 128^3 elements, 50 applies

Uniform open knots on [0,1], p Gauss points per element and direction.
Coefficients: c ~ U[0.5, 1.5], A = I + 0.05·G·Gᵀ/d, G ~ N(0,1), generated
on the device by igs_fill_synthetic (counter-based, slab-reproducible);
`field_from_planes` wraps host planes (e.g. the SURVEY §8d numpy recipe).
"""

import ctypes

import numpy as np

from . import _lib
from .bspline import UnivariateBasis, uniform_open_knots
from .geometry import CoefficientField, first_order_derivative_set
from .quadrature import TensorQuadrature, per_element_rule
from .sumfac import AssemblyProblem

MASS, STIFF, MASS_STIFF = 1, 2, 3

CONFIGS = {
    "C1": dict(d=2, p=3, K=64, kind=MASS, op="assemble"),
    "C2": dict(d=2, p=5, K=256, kind=STIFF, op="assemble"),
    "C3": dict(d=3, p=4, K=64, kind=MASS_STIFF, op="assemble"),
    "C4": dict(d=3, p=6, K=128, kind=STIFF, op="apply", applies=100),
    "C5": dict(d=3, p=8, K=128, kind=MASS_STIFF, op="apply", applies=50),
}


def plane_map(d, kind):
    """plane_of[eta][theta] over the first-order set: [c], then the diagonal
    a_aa, then the upper triangle a_ab (shared by (a,b) and (b,a))."""
    n = d + 1
    pm = [[-1] * n for _ in range(n)]
    pl = 0
    if kind & MASS:
        pm[0][0] = pl
        pl += 1
    if kind & STIFF:
        for a in range(d):
            pm[1 + a][1 + a] = pl
            pl += 1
        for a in range(d):
            for b in range(a + 1, d):
                pm[1 + a][1 + b] = pm[1 + b][1 + a] = pl
                pl += 1
    return pm, pl


def spaces(d, p, K, k=None):
    k = p if k is None else k
    bases = [UnivariateBasis(uniform_open_knots(p, K)) for _ in range(d)]
    rules = [per_element_rule(b.breakpoints, k) for b in bases]
    return bases, TensorQuadrature(rules)


def synthetic_planes(d, point_dims, kind, seed=0, z_range=None, out=None):
    """Device planes [n_planes, points of layers z_range] via igs_fill_synthetic."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    _, npl = plane_map(d, kind)
    z_lo, z_hi = (0, point_dims[-1]) if z_range is None else z_range
    layer = int(np.prod(point_dims[:-1]))
    n = (z_hi - z_lo) * layer
    if out is None:
        out = torch.empty((npl, n), dtype=torch.float64, device="cuda")
    dims = (ctypes.c_int64 * 3)(*(list(point_dims) + [1] * (3 - d)))
    st = lib.igs_fill_synthetic(d, dims, z_lo, z_hi, kind, seed, _lib.ptr(out), out.stride(0),
                                _lib.stream_handle())
    _lib.check(st, "fill_synthetic")
    return out


def field_from_planes(d, kind, planes, point_shape, slab=None):
    torch = _lib.require_cuda()
    pm, npl = plane_map(d, kind)
    if not isinstance(planes, torch.Tensor):
        planes = torch.as_tensor(np.ascontiguousarray(planes), dtype=torch.float64, device="cuda")
    ths = first_order_derivative_set(d)
    return CoefficientField.from_planes(ths, ths, planes, pm, point_shape, slab=slab)


def make_problem(d, p, K, kind, seed=0, planes=None, max_nnz=1 << 62, k=None):
    """AssemblyProblem on uniform knots with synthetic (or given) planes."""
    bases, quad = spaces(d, p, K, k)
    if planes is None:
        planes = synthetic_planes(d, list(quad.shape), kind, seed)
    field = field_from_planes(d, kind, planes, quad.shape)
    return AssemblyProblem(bases, bases, quad, field, max_nnz=max_nnz)


def config_problem(name, seed=0, K=None):
    c = CONFIGS[name]
    return make_problem(c["d"], c["p"], K or c["K"], c["kind"], seed)
