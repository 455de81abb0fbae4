"""Univariate B-spline bases and banded tabulation (mirror of bspline.py).

Knot vectors and bases are host metadata (validated exactly as the reference
does, bspline.py:28-150); the tabulation itself (bspline.py:314-333) runs on
the GPU through igs_tabulate (K1).  Tables live on the device; `.values` /
`.first_active` are device tensors, `.values_np()` copies them to the host.
"""

import ctypes

import numpy as np

from . import _lib
from .errors import DomainError, UnsupportedDerivativeError

__all__ = (
    "KnotVector",
    "UnivariateBasis",
    "BasisEvalTable",
    "uniform_open_knots",
    "find_span",
    "eval_all_derivs",
    "overlap_param",
    "tabulate",
)


class KnotVector:
    """A validated open knot vector (bspline.py:28-90)."""

    def __init__(self, order, knots):
        order = int(order)
        if order < 1:
            raise ValueError("order must be at least 1")
        knots = np.ascontiguousarray(knots, dtype=float)
        if knots.ndim != 1:
            raise ValueError("knots must be a flat sequence")
        if len(knots) < 2 * order:
            raise ValueError("need at least 2*order knots for a clamped vector")
        if np.any(np.diff(knots) < 0):
            raise ValueError("knots must be non-decreasing")
        a, b = knots[0], knots[-1]
        if not a < b:
            raise ValueError("knot vector spans an empty interval")
        if np.any(knots[:order] != a) or knots[order] == a:
            raise ValueError("first knot must have multiplicity exactly `order`")
        if np.any(knots[-order:] != b) or knots[-order - 1] == b:
            raise ValueError("last knot must have multiplicity exactly `order`")
        values, counts = np.unique(knots, return_counts=True)
        if np.any(counts > order):
            raise ValueError("knot multiplicity exceeds the order")
        self.order = order
        self.knots = knots
        self.knots.setflags(write=False)
        self.a = float(a)
        self.b = float(b)
        self.breakpoints = values
        self.breakpoints.setflags(write=False)
        self._multiplicity = dict(zip(values.tolist(), counts.tolist()))
        self._dev = {}

    @property
    def num_basis(self):
        return len(self.knots) - self.order

    @property
    def num_elements(self):
        return len(self.breakpoints) - 1

    @property
    def max_interior_multiplicity(self):
        inner = [self._multiplicity[v] for v in self.breakpoints[1:-1].tolist()]
        return max(inner) if inner else 1

    def multiplicity(self, xi):
        return self._multiplicity.get(float(xi), 0)

    def device(self, name="knots"):
        """Device copy (cached) of `knots` or `breakpoints`."""
        t = self._dev.get(name)
        if t is None:
            torch = _lib.require_cuda()
            t = torch.tensor(np.asarray(getattr(self, name), dtype=np.float64), device="cuda")
            self._dev[name] = t
        return t

    def __repr__(self):
        return f"KnotVector(order={self.order}, knots={self.knots.tolist()})"


def uniform_open_knots(order, num_elements, a=0.0, b=1.0, interior_multiplicity=1):
    """Open knot vector with uniform breakpoints on [a, b] (bspline.py:93-111)."""
    if num_elements < 1:
        raise ValueError("need at least one element")
    if not 1 <= interior_multiplicity <= order:
        raise ValueError("interior multiplicity must be in [1, order]")
    interior = np.linspace(a, b, num_elements + 1)[1:-1]
    knots = np.concatenate(
        [np.full(order, float(a)), np.repeat(interior, interior_multiplicity), np.full(order, float(b))]
    )
    return KnotVector(order, knots)


class UnivariateBasis:
    """The B-spline basis of a knot vector; csupp(n) = [knots[n], knots[n+order]]."""

    def __init__(self, knot_vector):
        if not isinstance(knot_vector, KnotVector):
            raise TypeError("knot_vector must be a KnotVector")
        self.kv = knot_vector
        self.order = knot_vector.order
        self.num_basis = knot_vector.num_basis
        self.csupp_lo = knot_vector.knots[: self.num_basis].copy()
        self.csupp_hi = knot_vector.knots[self.order:].copy()
        self.csupp_lo.setflags(write=False)
        self.csupp_hi.setflags(write=False)
        self._dev = {}

    @property
    def breakpoints(self):
        return self.kv.breakpoints

    @property
    def num_elements(self):
        return self.kv.num_elements

    @property
    def domain(self):
        return self.kv.a, self.kv.b

    @property
    def max_smoothness(self):
        """True when every interior knot is simple (function e+j active on element e)."""
        return self.kv.max_interior_multiplicity == 1

    def csupp(self, n):
        return float(self.csupp_lo[n]), float(self.csupp_hi[n])

    def device_csupp(self):
        t = self._dev.get("csupp")
        if t is None:
            torch = _lib.require_cuda()
            t = (torch.tensor(self.csupp_lo, dtype=torch.float64, device="cuda"),
                 torch.tensor(self.csupp_hi, dtype=torch.float64, device="cuda"))
            self._dev["csupp"] = t
        return t

    def __repr__(self):
        return f"UnivariateBasis(order={self.order}, N={self.num_basis})"


def find_span(basis, x):
    """Knot-interval index with knots[i] <= x < knots[i+1] (bspline.py:153-166)."""
    kv = basis.kv
    if not kv.a <= x <= kv.b:
        raise DomainError(f"point {x} outside the domain [{kv.a}, {kv.b}]")
    if x >= kv.b:
        return basis.num_basis - 1
    return int(np.searchsorted(kv.knots, x, side="right")) - 1


class BasisEvalTable:
    """Banded table: values[k, j, i] = k-th derivative of function first_active[i]+j.

    `values` and `first_active` are device tensors; `points` is the host
    point array the table was built at (bspline.py:258-311).
    """

    def __init__(self, order, num_functions, points, max_deriv, first_active, values, basis=None,
                 points_dev=None):
        self.order = order
        self.num_functions = num_functions
        self.points = points
        self.max_deriv = max_deriv
        self.first_active = first_active
        self.values = values
        self.basis = basis
        self.points_dev = points_dev
        self._np = None

    @property
    def num_points(self):
        return len(self.points)

    def values_np(self):
        if self._np is None:
            self._np = (self.values.cpu().numpy(), self.first_active.cpu().numpy())
        return self._np[0]

    def first_active_np(self):
        self.values_np()
        return self._np[1]

    def dense(self, deriv=0):
        """Dense (num_functions x num_points) value matrix; zeros off-band."""
        vals = self.values_np()
        fa = self.first_active_np()
        out = np.zeros((self.num_functions, self.num_points))
        cols = np.arange(self.num_points)
        for j in range(self.order):
            out[fa + j, cols] = vals[deriv, j, :]
        return out


    def point_matrix(self, deriv=0):
        """COO triplets (rows = point, cols = function, data) of the band,
        structural zeros kept (bspline.py:287-297)."""
        npts = self.num_points
        rows = np.repeat(np.arange(npts), self.order)
        cols = (self.first_active_np()[:, None] + np.arange(self.order)[None, :]).ravel()
        data = self.values_np()[deriv].T.ravel()
        return rows, cols, data

    def restrict(self, point_slice, fn_lo, num_functions):
        """View of this table on a point range and a function index range
        (bspline.py:299-311); the device arrays are sliced, not copied."""
        first = self.first_active[point_slice] - fn_lo
        if first.numel():
            lo, hi = int(first.min()), int(first.max())
            if lo < 0 or hi + self.order > num_functions:
                raise ValueError("restriction does not cover the active band")
        return BasisEvalTable(self.order, num_functions, self.points[point_slice], self.max_deriv, first,
                              self.values[:, :, point_slice],
                              points_dev=None if self.points_dev is None else self.points_dev[point_slice])


def tabulate(basis, points, max_deriv):
    """Evaluate the basis and derivatives 0..max_deriv at sorted points, on the GPU.

    Same contract as bspline.tabulate (bspline.py:314-333): unsorted points
    raise ValueError, out-of-domain points DomainError, max_deriv >= order
    UnsupportedDerivativeError.
    """
    torch = _lib.require_cuda()
    lib = _lib.load()
    p = basis.order
    if not 0 <= max_deriv < p:
        raise UnsupportedDerivativeError(f"derivative order {max_deriv} not supported for spline order {p}")
    if isinstance(points, torch.Tensor):
        pts_dev = points.to(device="cuda", dtype=torch.float64).contiguous()
        pts_host = pts_dev.cpu().numpy()
    else:
        pts_host = np.array(points, dtype=float, copy=True)
        pts_dev = torch.from_numpy(pts_host).to("cuda")
    npts = len(pts_host)
    values = torch.empty((max_deriv + 1, p, npts), dtype=torch.float64, device="cuda")
    first = torch.empty(npts, dtype=torch.int64, device="cuda")
    knots = basis.kv.device("knots")
    st = lib.igs_tabulate(p, _lib.ptr(knots), len(basis.kv.knots), _lib.ptr(pts_dev), npts, max_deriv,
                          _lib.ptr(values), _lib.ptr(first), _lib.stream_handle())
    _lib.check(st, "tabulate")
    return BasisEvalTable(p, basis.num_basis, pts_host, max_deriv, first, values, basis=basis,
                          points_dev=pts_dev)


def eval_all_derivs(basis, x, max_deriv):
    """(first, ders[k, j]) of the order functions active at x (bspline.py:169-239)."""
    tab = tabulate(basis, [float(x)], max_deriv)
    return int(tab.first_active_np()[0]), tab.values_np()[:, :, 0].copy()


def overlap_param(basis, points):
    """Largest number of csupps containing one point (bspline.py:242-255)."""
    points = np.asarray(points, dtype=float)
    if points.size == 0:
        return 0
    lo, hi = basis.csupp_lo, basis.csupp_hi
    pts = np.atleast_1d(points)
    a = np.searchsorted(hi, pts, side="left")        # first n with hi >= x
    b = np.searchsorted(lo, pts, side="right")       # first n with lo > x
    return int(np.max(b - a))
