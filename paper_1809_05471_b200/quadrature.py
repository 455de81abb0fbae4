"""Gauss-Legendre rules per element and tensor quadrature (mirror of quadrature.py).

The Newton iteration and the affine element map run on the GPU
(igs_gauss_rule, K1); rules are immutable host/device pairs.
"""

import numpy as np

from . import _lib

__all__ = (
    "ReferenceGaussRule",
    "QuadratureRule1D",
    "TensorQuadrature",
    "gauss_legendre",
    "per_element_rule",
    "custom_rule",
)

_MAX_GAUSS_NODES = 64


class ReferenceGaussRule:
    """Gauss-Legendre rule on [-1, 1] (quadrature.py:25-31)."""

    def __init__(self, k, nodes, weights):
        self.k = k
        self.nodes = nodes
        self.weights = weights


class QuadratureRule1D:
    """Sorted quadrature points with aligned weights (quadrature.py:68-84).

    `elements` / `points_per_element` are set for per-element rules so the
    fused kernels can use the element structure; custom rules leave them 0.
    """

    def __init__(self, points, weights, elements=0, points_per_element=0):
        self.points = points
        self.weights = weights
        self.elements = int(elements)
        self.points_per_element = int(points_per_element)
        self.breakpoints = None
        self._dev = None

    @property
    def num_points(self):
        return len(self.points)

    def __len__(self):
        return len(self.points)

    def restrict(self, lo, hi):
        return QuadratureRule1D(self.points[lo:hi], self.weights[lo:hi])

    def device(self):
        """(points, weights) as device tensors (cached)."""
        if self._dev is None:
            torch = _lib.require_cuda()
            self._dev = (torch.as_tensor(np.ascontiguousarray(self.points), device="cuda"),
                         torch.as_tensor(np.ascontiguousarray(self.weights), device="cuda"))
        return self._dev


def _device_rule(k, breakpoints):
    torch = _lib.require_cuda()
    lib = _lib.load()
    bp = torch.as_tensor(np.ascontiguousarray(breakpoints, dtype=float), device="cuda")
    n = (len(breakpoints) - 1) * k
    pts = torch.empty(n, dtype=torch.float64, device="cuda")
    wts = torch.empty(n, dtype=torch.float64, device="cuda")
    st = lib.igs_gauss_rule(k, _lib.ptr(bp), len(breakpoints), _lib.ptr(pts), _lib.ptr(wts),
                            _lib.stream_handle())
    _lib.check(st, "gauss_rule")
    return pts, wts


def gauss_legendre(k):
    """Gauss-Legendre nodes/weights on [-1, 1] for 1 <= k <= 64 (quadrature.py:34-65)."""
    if not 1 <= k <= _MAX_GAUSS_NODES:
        raise ValueError(f"node count {k} outside [1, {_MAX_GAUSS_NODES}]")
    pts, wts = _device_rule(k, [-1.0, 1.0])
    nodes = pts.cpu().numpy()
    weights = wts.cpu().numpy()
    nodes.setflags(write=False)
    weights.setflags(write=False)
    return ReferenceGaussRule(k, nodes, weights)


def per_element_rule(breakpoints, k):
    """k-point Gauss rule mapped into every element (quadrature.py:87-106)."""
    breakpoints = np.unique(np.asarray(breakpoints, dtype=float))
    if len(breakpoints) < 2:
        raise ValueError("need at least 2 distinct breakpoints")
    if not 1 <= k <= _MAX_GAUSS_NODES:
        raise ValueError(f"node count {k} outside [1, {_MAX_GAUSS_NODES}]")
    pts, wts = _device_rule(k, breakpoints)
    points = pts.cpu().numpy()
    weights = wts.cpu().numpy()
    points.setflags(write=False)
    weights.setflags(write=False)
    rule = QuadratureRule1D(points, weights, elements=len(breakpoints) - 1, points_per_element=k)
    rule.breakpoints = breakpoints
    rule._dev = (pts, wts)
    return rule


def custom_rule(points, weights):
    """Wrap user-supplied points/weights unchanged (quadrature.py:109-119)."""
    points = np.ascontiguousarray(points, dtype=float)
    weights = np.ascontiguousarray(weights, dtype=float)
    if points.shape != weights.shape or points.ndim != 1:
        raise ValueError("points and weights must be flat sequences of equal length")
    if np.any(np.diff(points) < 0):
        raise ValueError("points must be sorted ascending")
    points.setflags(write=False)
    weights.setflags(write=False)
    return QuadratureRule1D(points, weights)


class TensorQuadrature:
    """One QuadratureRule1D per direction (quadrature.py:122-151)."""

    def __init__(self, rules):
        self.rules = tuple(rules)
        if not self.rules:
            raise ValueError("need at least one direction")

    @property
    def dim(self):
        return len(self.rules)

    @property
    def shape(self):
        return tuple(r.num_points for r in self.rules)

    @property
    def num_points(self):
        n = 1
        for r in self.rules:
            n *= r.num_points
        return n

    def flat_weights(self):
        """Tensor weights, direction 1 fastest (host; used by oracles/tests)."""
        w = np.ones(1)
        for rule in self.rules:
            w = (rule.weights[:, None] * w[None, :]).ravel()
        return w
