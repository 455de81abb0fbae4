"""Coefficient fields at quadrature points (the input layout of the hot path).

Mirror of CoefficientField / first_order_derivative_set (geometry.py:48-55,
279-312).  On the device the field is stored as SoA planes
`planes[plane, x]` (x flat, direction 1 fastest) with a map
`plane_of[eta_i][theta_j]` -> plane index, -1 marking an exactly-zero block
(geometry.py:296: zero blocks are detected exactly, never thresholded).
Blocks that are exactly equal (F symmetric) share one plane, so a symmetric
3D mass+stiffness field streams 7 planes instead of 16.

Geometry maps and the PDE pullback (geometry.py:58-276, 315-451) are the
step before this path and are not part of it.
"""

import numpy as np

from . import _lib

__all__ = ("CoefficientField", "first_order_derivative_set")


def first_order_derivative_set(d):
    """Multi-indices of total order <= 1: the value plus one per direction."""
    out = [(0,) * d]
    for delta in range(d):
        e = [0] * d
        e[delta] = 1
        out.append(tuple(e))
    return tuple(out)


class CoefficientField:
    """Matrix-valued coefficient at every quadrature point.

    ``CoefficientField(theta_set, eta_set, values, point_shape)`` accepts the
    reference's dense ``values[x, i(eta), j(theta)]`` (numpy or torch); the
    planes are built on the device.  ``CoefficientField.from_planes`` wraps
    planes that already live on the device (the BASELINE workloads generate
    them there).
    """

    def __init__(self, theta_set, eta_set, values, point_shape):
        torch = _lib.require_cuda()
        self.theta_set = tuple(tuple(int(v) for v in t) for t in theta_set)
        self.eta_set = tuple(tuple(int(v) for v in t) for t in eta_set)
        vals = torch.as_tensor(values, dtype=torch.float64, device="cuda")
        if vals.dim() != 3 or tuple(vals.shape[1:]) != (len(self.eta_set), len(self.theta_set)):
            raise ValueError("coefficient array shape does not match the index sets")
        npts = vals.shape[0]
        nonzero = (vals != 0).any(dim=0).cpu().numpy()
        planes = []
        plane_of = [[-1] * len(self.theta_set) for _ in self.eta_set]
        for i in range(len(self.eta_set)):
            for j in range(len(self.theta_set)):
                if not nonzero[i, j]:
                    continue
                col = vals[:, i, j]
                # share the plane of an exactly equal transposed block
                if j < len(self.eta_set) and i < len(self.theta_set) and plane_of[j][i] >= 0 \
                        and j < i and torch.equal(col, planes[plane_of[j][i]]):
                    plane_of[i][j] = plane_of[j][i]
                    continue
                plane_of[i][j] = len(planes)
                planes.append(col.contiguous())
        if planes:
            self.planes = torch.stack(planes, dim=0).contiguous()
        else:
            self.planes = torch.zeros((0, npts), dtype=torch.float64, device="cuda")
        self.plane_of = tuple(tuple(r) for r in plane_of)
        self.point_shape = tuple(point_shape)
        self._num_points = int(npts)
        self.slab = None

    @classmethod
    def from_planes(cls, theta_set, eta_set, planes, plane_of, point_shape, slab=None):
        """Wrap device planes [n_planes, npts] with an explicit plane map.

        `slab=(lo, hi)`: the planes hold only the points of elements
        [lo, hi) of the last direction (one rank's part of a slab-
        partitioned apply, sharded.py); `point_shape` stays the full grid.
        """
        torch = _lib.require_cuda()
        self = cls.__new__(cls)
        self.theta_set = tuple(tuple(int(v) for v in t) for t in theta_set)
        self.eta_set = tuple(tuple(int(v) for v in t) for t in eta_set)
        if planes.device.type != "cuda" or planes.dtype != torch.float64 or planes.dim() != 2:
            raise ValueError("planes must be a float64 CUDA tensor [n_planes, npts]")
        self.planes = planes if planes.stride(1) == 1 else planes.contiguous()
        self.plane_of = tuple(tuple(int(v) for v in r) for r in plane_of)
        if len(self.plane_of) != len(self.eta_set) or any(len(r) != len(self.theta_set) for r in self.plane_of):
            raise ValueError("plane_of must be [len(eta_set)][len(theta_set)]")
        self.point_shape = tuple(point_shape)
        self._num_points = int(planes.shape[1])
        self.slab = None if slab is None else (int(slab[0]), int(slab[1]))
        return self

    @property
    def num_points(self):
        return self._num_points

    @property
    def n_planes(self):
        return int(self.planes.shape[0])

    @property
    def plane_stride(self):
        return int(self.planes.stride(0)) if self.n_planes else self._num_points

    def block(self, eta_idx, theta_idx):
        torch = _lib.require_cuda()
        pl = self.plane_of[eta_idx][theta_idx]
        if pl < 0:
            return torch.zeros(self._num_points, dtype=torch.float64, device="cuda")
        return self.planes[pl]

    def is_zero_block(self, eta_idx, theta_idx):
        return self.plane_of[eta_idx][theta_idx] < 0

    @property
    def values(self):
        """Dense host copy values[x, i, j] (only for small fields)."""
        out = np.zeros((self._num_points, len(self.eta_set), len(self.theta_set)))
        host = self.planes.cpu().numpy()
        for i in range(len(self.eta_set)):
            for j in range(len(self.theta_set)):
                pl = self.plane_of[i][j]
                if pl >= 0:
                    out[:, i, j] = host[pl]
        return out
