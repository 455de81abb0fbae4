"""Coefficient fields at quadrature points (the input layout of the hot path).

Mirror of CoefficientField / first_order_derivative_set (geometry.py:48-55,
279-312).  On the device the field is stored as SoA planes
`planes[plane, x]` (x flat, direction 1 fastest) with a map
`plane_of[eta_i][theta_j]` -> plane index, -1 marking an exactly-zero block
(geometry.py:296: zero blocks are detected exactly, never thresholded).
Blocks that are exactly equal (F symmetric) share one plane, so a symmetric
3D mass+stiffness field streams 7 planes instead of 16.

Geometry maps and the PDE pullback (geometry.py:58-276, 315-451; SURVEY
§8f row f1, the step before the path) run on the device as well: the map's
spline fields come from Alg. 3 (igs_eval_field) and one pointwise kernel
(igs_geometry_pullback) forms J, det J, J^{-1} and writes the pulled-back
coefficient straight into the SoA planes.  PDE coefficients are constants,
the named specs ("identity", "default"), per-point arrays, or callables of
the physical points (evaluated on the host: user code).
"""

import numpy as np

from . import _lib
from .bspline import KnotVector, UnivariateBasis, tabulate, uniform_open_knots
from .errors import DegenerateGeometryError

__all__ = (
    "GeometryMap",
    "GeometryEvaluation",
    "CoefficientField",
    "PDEData",
    "PulledBackCoefficient",
    "eval_geometry",
    "build_coefficient_field",
    "identity_geometry",
    "box_geometry",
    "affine_geometry",
    "quarter_annulus",
    "twisted_box",
    "named_geometry",
    "pde_mass",
    "pde_laplace",
    "pde_convection_diffusion",
    "named_pde",
    "first_order_derivative_set",
)

_DEGENERACY_RTOL = 1e-12


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
        # the fused kernels read the planes by TMA (16-byte aligned base and
        # plane stride): realign strided / offset views once here
        if planes.stride(1) != 1 or planes.data_ptr() % 16 or (planes.shape[0] > 1 and planes.stride(0) % 2):
            planes = planes.contiguous() if planes.stride(1) != 1 else planes.clone()
        self.planes = planes
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

    def restrict_flat(self, flat_idx, point_shape):
        """Sub-field over a subset of grid points given as flat indices
        (geometry.py:308-312); the planes are gathered on the device and the
        plane map is kept."""
        torch = _lib.require_cuda()
        idx = torch.as_tensor(np.asarray(flat_idx, dtype=np.int64).reshape(-1), device=self.planes.device)
        return CoefficientField.from_planes(self.theta_set, self.eta_set,
                                            self.planes.index_select(1, idx).contiguous(),
                                            self.plane_of, point_shape)

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


# --------------------------------------------------------------------------
# Geometry maps (geometry.py:58-101) and their evaluation (geometry.py:158-216)


class GeometryMap:
    """Tensor-product (rational) spline map of the unit cube, physical
    dimension = d.  control_points: (N, d) with direction 1 fastest (or the
    same data as a grid); weights: one strictly positive value per point."""

    def __init__(self, bases, control_points, weights=None):
        from .tensorspace import LexOrdering

        self.bases = tuple(bases)
        self.ordering = LexOrdering(b.num_basis for b in self.bases)
        n = self.ordering.size
        cp = np.asarray(control_points, dtype=float)
        if cp.ndim != 2:
            cp = cp.reshape(n, -1)
        if cp.shape[0] != n:
            raise ValueError("control point count must equal the basis function count")
        if cp.shape[1] != len(self.bases):
            raise ValueError("only maps with physical dimension equal to d are supported")
        self.control_points = cp
        self.s = cp.shape[1]
        if weights is not None:
            weights = np.asarray(weights, dtype=float).ravel()
            if len(weights) != n:
                raise ValueError("one weight per control point required")
            if np.any(weights <= 0):
                raise ValueError("rational weights must be strictly positive")
        self.weights = weights

    @property
    def d(self):
        return len(self.bases)

    @property
    def is_rational(self):
        return self.weights is not None


class GeometryEvaluation:
    """The map's spline fields at every tensor quadrature point (device).

    Holds the component values/gradients (weighted numerators and the weight
    for rational maps) that the pullback kernel consumes; `phys`, `jac`,
    `det` and `inv` are materialised on request (host-side convenience, same
    layouts as the reference: (npts, s), (npts, s, d), (npts,), (npts, d, s)).
    """

    def __init__(self, point_shape, fields, phys):
        self.point_shape = tuple(point_shape)
        self._f = fields
        self.phys_dev = phys

    @property
    def num_points(self):
        return int(self.phys_dev.shape[1])

    @property
    def d(self):
        return len(self._f["val"])

    @property
    def phys(self):
        return self.phys_dev.t().cpu().numpy()

    def _jac_dev(self):
        f = self._f
        d = self.d
        torch = _lib.require_cuda()
        jac = torch.empty((self.num_points, d, d), dtype=torch.float64, device="cuda")
        for c in range(d):
            for k in range(d):
                if f["wval"] is None:
                    jac[:, c, k] = f["grad"][c][k]
                else:
                    w = f["wval"]
                    jac[:, c, k] = (f["grad"][c][k] * w - f["val"][c] * f["wgrad"][k]) / (w * w)
        return jac

    @property
    def jac(self):
        return self._jac_dev().cpu().numpy()

    @property
    def det(self):
        return np.linalg.det(self.jac)

    @property
    def inv(self):
        return np.linalg.inv(self.jac)


def _spline_fields(geo, quad, counter=None):
    from .tensorspace import contract_to_points

    d = geo.d
    for basis in geo.bases:
        if basis.order < 2:
            raise ValueError("geometry bases need order >= 2 for derivatives")
    tables = [tabulate(b, r.points, 1) for b, r in zip(geo.bases, quad.rules)]

    def field(coeffs, derivs):
        return contract_to_points(tables, derivs, coeffs, counter).permute(*reversed(range(d))).reshape(-1)

    def value_and_grad(coeffs):
        val = field(coeffs, (0,) * d)
        grad = []
        for k in range(d):
            e = [0] * d
            e[k] = 1
            grad.append(field(coeffs, tuple(e)))
        return val, grad

    f = {"val": [], "grad": [], "wval": None, "wgrad": None}
    if geo.is_rational:
        f["wval"], f["wgrad"] = value_and_grad(geo.weights)
        for c in range(geo.s):
            v, g = value_and_grad(geo.weights * geo.control_points[:, c])
            f["val"].append(v)
            f["grad"].append(g)
    else:
        for c in range(geo.s):
            v, g = value_and_grad(geo.control_points[:, c])
            f["val"].append(v)
            f["grad"].append(g)
    return f


def _pullback(fields, npts, plane_of, n_planes, coeff_ptrs, phys=None, planes=None, keep=()):
    """One igs_geometry_pullback call; returns (first degenerate point or -1, nonzero flags)."""
    import ctypes

    torch = _lib.require_cuda()
    lib = _lib.load()
    d = len(fields["val"])
    args = _lib.IgsPullbackArgs()
    args.d = d
    args.npts = npts
    for c in range(d):
        args.val[c] = fields["val"][c].data_ptr()
        for k in range(d):
            args.grad[c][k] = fields["grad"][c][k].data_ptr()
    if fields["wval"] is not None:
        args.wval = fields["wval"].data_ptr()
        for k in range(d):
            args.wgrad[k] = fields["wgrad"][k].data_ptr()
    (args.reaction, args.reaction_stride, conv, args.convection_stride, diff,
     args.diffusion_stride) = coeff_ptrs
    for i in range(d):
        args.convection[i] = conv[i]
        for j in range(d):
            args.diffusion[i][j] = diff[i][j]
    args.rtol = _DEGENERACY_RTOL
    pm = (ctypes.c_int8 * 16)(*[plane_of[i][j] if (i < len(plane_of) and j < len(plane_of)) else -1
                                for i in range(4) for j in range(4)])
    flags = torch.zeros(max(n_planes, 1), dtype=torch.int32, device="cuda")
    ws = torch.empty(64, dtype=torch.uint8, device="cuda")
    bad = ctypes.c_int64(-1)
    st = lib.igs_geometry_pullback(ctypes.byref(args), pm, n_planes,
                                   planes.data_ptr() if planes is not None else None,
                                   int(planes.stride(0)) if planes is not None else 0,
                                   phys.data_ptr() if phys is not None else None, flags.data_ptr(),
                                   ctypes.byref(bad), ws.data_ptr(), 64, _lib.stream_handle())
    _lib.check(st, "geometry_pullback")
    del keep
    return int(bad.value), flags[:n_planes].cpu().numpy()


def _raise_degenerate(quad, flat):
    from .tensorspace import LexOrdering

    coords = tuple(float(rule.points[c]) for rule, c in zip(quad.rules, LexOrdering(quad.shape).split(flat)))
    raise DegenerateGeometryError(f"geometry Jacobian is singular at quadrature point {coords}")


def eval_geometry(geo, quad, counter=None):
    """Map, Jacobians, determinants and inverses at all points
    (geometry.py:158-216): the component splines by Alg. 3 on the device,
    rational maps as weighted numerators over the weight spline; a
    (near-)singular Jacobian raises DegenerateGeometryError."""
    torch = _lib.require_cuda()
    fields = _spline_fields(geo, quad, counter)
    npts = quad.num_points
    phys = torch.empty((geo.s, npts), dtype=torch.float64, device="cuda")
    nop = (None, 0, [None] * 3, 0, [[None] * 3 for _ in range(3)], 0)
    bad, _ = _pullback(fields, npts, [], 0, nop, phys=phys)
    if bad >= 0:
        _raise_degenerate(quad, bad)
    ev = GeometryEvaluation(quad.shape, fields, phys)
    ev.quad = quad
    return ev


# --------------------------------------------------------------------------
# PDE data and the pullback (geometry.py:219-336)


class PDEData:
    """Second-order coefficients on the physical domain: each of diffusion
    (d x d), convection (d) and reaction (scalar) is None, a constant, a
    named spec ("identity" / "default"), a per-point array, or a callable
    of the (npts, d) physical points."""

    def __init__(self, diffusion=None, convection=None, reaction=None):
        self.diffusion = diffusion
        self.convection = convection
        self.reaction = reaction


def pde_mass():
    return PDEData(reaction=1.0)


def pde_laplace():
    return PDEData(diffusion="identity")


def pde_convection_diffusion(diffusion=1.0, convection=None, reaction=1.0):
    return PDEData(diffusion=diffusion, convection=convection, reaction=reaction)


def named_pde(name, convection=None, reaction=None):
    name = name.replace("-", "_")
    if name == "mass":
        return pde_mass()
    if name == "laplace":
        return pde_laplace()
    if name in ("convection_diffusion", "cdr"):
        return pde_convection_diffusion(convection=convection if convection is not None else "default",
                                        reaction=reaction if reaction is not None else 1.0)
    raise ValueError(f"unknown pde '{name}'")


def _coeff_device(spec, shape, d, geo_eval):
    """Device tensor of the coefficient (shape () / (d,) / (d, d)) or per point
    ((npts,) + shape), and whether it is per point.  None -> (None, False)."""
    torch = _lib.require_cuda()
    if spec is None:
        return None, False
    if isinstance(spec, str):
        if spec == "identity":
            return torch.eye(d, dtype=torch.float64, device="cuda").reshape(shape), False
        if spec == "default":  # unit convection in every physical direction
            return torch.ones(shape, dtype=torch.float64, device="cuda"), False
        raise ValueError(f"unknown coefficient spec '{spec}'")
    npts = geo_eval.num_points
    if callable(spec):
        vals = np.asarray(spec(geo_eval.phys), dtype=float)
    elif isinstance(spec, torch.Tensor):
        vals = spec.to(device="cuda", dtype=torch.float64)
    else:
        vals = np.asarray(spec, dtype=float)
        if shape == (d, d) and vals.ndim == 0:
            vals = vals * np.eye(d)
    t = torch.as_tensor(vals, dtype=torch.float64, device="cuda")
    if tuple(t.shape) == shape:
        return t.contiguous(), False
    if t.dim() == len(shape) + 1 and t.shape[0] == npts:
        return torch.broadcast_to(t, (npts,) + shape).contiguous(), True
    return torch.broadcast_to(t, shape).contiguous(), False


def _plane_setup(pde, d, geo_eval):
    """Device PDE data, the plane map over (eta i, theta j) of the first-order
    set and the kernel pointer tuple.  `geo_eval` provides num_points and, for
    callables, phys."""
    torch = _lib.require_cuda()
    A, a_pp = _coeff_device(pde.diffusion, (d, d), d, geo_eval)
    b, b_pp = _coeff_device(pde.convection, (d,), d, geo_eval)
    c, c_pp = _coeff_device(pde.reaction, (), d, geo_eval)
    keep = [A, b, c]
    # pointers + strides for the kernel (stride 0 = constant)
    cptr = c.data_ptr() if c is not None else None
    conv = [None] * 3
    diff = [[None] * 3 for _ in range(3)]
    if b is not None:
        bt = b.t().contiguous() if b_pp else b
        keep.append(bt)
        for i in range(d):
            conv[i] = bt[i].data_ptr()
    sym = False
    if A is not None:
        At = A.permute(1, 2, 0).contiguous() if a_pp else A
        keep.append(At)
        for i in range(d):
            for j in range(d):
                diff[i][j] = At[i, j].data_ptr()
        sym = all(torch.equal(At[i, j], At[j, i]) for i in range(d) for j in range(i + 1, d))
    n = d + 1
    plane_of = [[-1] * n for _ in range(n)]
    npl = 0
    if c is not None:
        plane_of[0][0] = npl
        npl += 1
    if b is not None:
        for i in range(d):
            plane_of[1 + i][0] = npl
            npl += 1
    if A is not None:
        for i in range(d):
            for j in range(d):
                if sym and j < i:
                    plane_of[1 + i][1 + j] = plane_of[1 + j][1 + i]
                else:
                    plane_of[1 + i][1 + j] = npl
                    npl += 1
    ptrs = (cptr, 1 if c_pp else 0, conv, 1 if b_pp else 0, diff, 1 if a_pp else 0)
    return plane_of, npl, ptrs, keep


def _plane_finish(planes, plane_of, npl, nonzero, d, npts, point_shape, counter):
    """Drop exactly-zero planes (geometry.py:296), renumber, wrap."""
    torch = _lib.require_cuda()
    if counter is not None:
        counter.add_coeff_build(npts * (2 * (1 + d) ** 3 + (1 + d) ** 2))
    n = d + 1
    live = [p for p in range(npl) if nonzero[p]]
    remap = {p: k for k, p in enumerate(live)}
    plane_of = [[remap.get(plane_of[i][j], -1) if plane_of[i][j] >= 0 else -1 for j in range(n)] for i in range(n)]
    if live and len(live) < npl:
        planes = planes[torch.tensor(live, device="cuda")].contiguous()
    elif not live:
        planes = torch.zeros((0, npts), dtype=torch.float64, device="cuda")
    ths = first_order_derivative_set(d)
    return CoefficientField.from_planes(ths, ths, planes, plane_of, point_shape)


def build_coefficient_field(geo_eval, pde, counter=None):
    """Pull a second-order form back through an evaluated geometry
    (geometry.py:315-336) into device coefficient planes: F = |det J|·E·
    [[c, 0], [b, A]]·E^T, E = diag(1, J^{-1}); exactly-zero blocks are
    dropped (geometry.py:296), transposed blocks of a symmetric diffusion
    share a plane."""
    torch = _lib.require_cuda()
    d = geo_eval.d
    npts = geo_eval.num_points
    plane_of, npl, ptrs, keep = _plane_setup(pde, d, geo_eval)
    planes = torch.empty((max(npl, 1), npts), dtype=torch.float64, device="cuda")
    bad, nonzero = _pullback(geo_eval._f, npts, plane_of, npl, ptrs, planes=planes, keep=keep)
    if bad >= 0:
        _raise_degenerate(geo_eval.quad, bad)
    return _plane_finish(planes, plane_of, npl, nonzero, d, npts, geo_eval.point_shape, counter)


class _MapPoints:
    """The fused path's view of the map at the quadrature points: tables,
    control data and the C struct; `phys` (for callable PDE data) by one
    plane-less pass of the fused kernel."""

    def __init__(self, geo, quad):
        torch = _lib.require_cuda()
        self.geo, self.quad = geo, quad
        self.d = geo.d
        self.point_shape = tuple(quad.shape)
        self.num_points = quad.num_points
        for basis in geo.bases:
            if not 2 <= basis.order <= 8:
                raise ValueError("fused geometry evaluation needs map orders 2..8")
        self.tables = [tabulate(b, r.points, 1) for b, r in zip(geo.bases, quad.rules)]
        self.control = torch.as_tensor(np.ascontiguousarray(geo.control_points), dtype=torch.float64,
                                       device="cuda").contiguous()
        self.weights = (torch.as_tensor(np.asarray(geo.weights, dtype=float), device="cuda")
                        if geo.is_rational else None)
        m = _lib.IgsGeometryMap()
        m.d = self.d
        for k, (b, t) in enumerate(zip(geo.bases, self.tables)):
            m.order[k] = b.order
            m.num_basis[k] = b.num_basis
            m.num_points[k] = quad.rules[k].num_points
            m.values[k] = t.values.data_ptr()
            m.first_active[k] = t.first_active.data_ptr()
        m.control = self.control.data_ptr()
        m.weights = self.weights.data_ptr() if self.weights is not None else None
        self.struct = m
        self._phys = None

    def run(self, plane_of, npl, ptrs, planes=None, phys=None, keep=()):
        import ctypes

        torch = _lib.require_cuda()
        lib = _lib.load()
        d = self.d
        args = _lib.IgsPullbackArgs()
        args.d = d
        args.npts = self.num_points
        (args.reaction, args.reaction_stride, conv, args.convection_stride, diff,
         args.diffusion_stride) = ptrs
        for i in range(d):
            args.convection[i] = conv[i]
            for j in range(d):
                args.diffusion[i][j] = diff[i][j]
        args.rtol = _DEGENERACY_RTOL
        pm = (ctypes.c_int8 * 16)(*[plane_of[i][j] if (i < len(plane_of) and j < len(plane_of)) else -1
                                    for i in range(4) for j in range(4)])
        flags = torch.zeros(max(npl, 1), dtype=torch.int32, device="cuda")
        ws = torch.empty(64, dtype=torch.uint8, device="cuda")
        bad = ctypes.c_int64(-1)
        st = lib.igs_geometry_planes(ctypes.byref(self.struct), ctypes.byref(args), pm, npl,
                                     planes.data_ptr() if planes is not None else None,
                                     int(planes.stride(0)) if planes is not None else 0,
                                     phys.data_ptr() if phys is not None else None, flags.data_ptr(),
                                     ctypes.byref(bad), ws.data_ptr(), 64, _lib.stream_handle())
        _lib.check(st, "geometry_planes")
        del keep
        if bad.value >= 0:
            _raise_degenerate(self.quad, int(bad.value))
        return flags[:npl].cpu().numpy()

    @property
    def phys(self):
        if self._phys is None:
            torch = _lib.require_cuda()
            ph = torch.empty((self.d, self.num_points), dtype=torch.float64, device="cuda")
            nop = (None, 0, [None] * 3, 0, [[None] * 3 for _ in range(3)], 0)
            self.run([], 0, nop, phys=ph)
            self._phys = ph.t().cpu().numpy()
        return self._phys


def pull_back_fused(geo, quad, pde, counter=None):
    """f1 fused: coefficient planes straight from the map and the PDE data
    (one kernel pass evaluates the map's fields per point and pulls back;
    no per-point field arrays) — the same planes as
    build_coefficient_field(eval_geometry(geo, quad), pde) up to rounding."""
    torch = _lib.require_cuda()
    mp = _MapPoints(geo, quad)
    d, npts = mp.d, mp.num_points
    plane_of, npl, ptrs, keep = _plane_setup(pde, d, mp)
    planes = torch.empty((max(npl, 1), npts), dtype=torch.float64, device="cuda")
    nonzero = mp.run(plane_of, npl, ptrs, planes=planes, keep=keep)
    if counter is not None:
        # the reference's count for the fields the two-step path evaluates
        # (value + d derivatives per component, and the weight if rational)
        from .tensorspace import field_eval_count

        per = field_eval_count([b.order for b in geo.bases], [b.num_basis for b in geo.bases],
                               [r.num_points for r in quad.rules])
        counter.add_field_eval(per * (d + 1) * (geo.s + (1 if geo.is_rational else 0)))
    return _plane_finish(planes, plane_of, npl, nonzero, d, npts, mp.point_shape, counter)


class PulledBackCoefficient:
    """Lazy coefficient provider: geometry map plus PDE data
    (geometry.py:339-354)."""

    def __init__(self, geometry, pde):
        self.geometry = geometry
        self.pde = pde
        self.theta_set = first_order_derivative_set(geometry.d)
        self.eta_set = self.theta_set

    def evaluate(self, quad, counter=None, fused=True):
        """fused=True: pull_back_fused (map orders 2..8); else the two-step
        eval_geometry (Alg. 3 field arrays) + build_coefficient_field."""
        if fused and all(2 <= b.order <= 8 for b in self.geometry.bases):
            return pull_back_fused(self.geometry, quad, self.pde, counter)
        return build_coefficient_field(eval_geometry(self.geometry, quad, counter), self.pde, counter)


# --------------------------------------------------------------------------
# Built-in geometries (geometry.py:357-451)


def _linear_bases(d):
    return [UnivariateBasis(KnotVector(2, [0.0, 0.0, 1.0, 1.0])) for _ in range(d)]


def box_geometry(lo, hi):
    """Axis-aligned box as a multilinear map (constant Jacobian)."""
    from .tensorspace import LexOrdering

    lo = np.asarray(lo, dtype=float)
    hi = np.asarray(hi, dtype=float)
    d = len(lo)
    ordering = LexOrdering((2,) * d)
    corners = np.array([[hi[i] if bits[i] else lo[i] for i in range(d)]
                        for bits in (ordering.split(n) for n in range(2 ** d))], dtype=float)
    return GeometryMap(_linear_bases(d), corners)


def identity_geometry(d):
    return box_geometry([0.0] * d, [1.0] * d)


def affine_geometry(matrix, shift=None):
    """x -> matrix @ x + shift on the unit cube."""
    matrix = np.asarray(matrix, dtype=float)
    d = matrix.shape[0]
    shift = np.zeros(d) if shift is None else np.asarray(shift, dtype=float)
    base = box_geometry([0.0] * d, [1.0] * d)
    return GeometryMap(base.bases, base.control_points @ matrix.T + shift[None, :])


def quarter_annulus(r_inner=1.0, r_outer=2.0):
    """Exact rational quarter annulus: direction 1 radial (linear), direction
    2 angular (quadratic arc with weights 1, 1/sqrt(2), 1)."""
    radial = UnivariateBasis(KnotVector(2, [0.0, 0.0, 1.0, 1.0]))
    angular = UnivariateBasis(KnotVector(3, [0.0, 0.0, 0.0, 1.0, 1.0, 1.0]))
    arc = np.array([[1.0, 0.0], [1.0, 1.0], [0.0, 1.0]])
    w_arc = np.array([1.0, np.sqrt(0.5), 1.0])
    radii = np.array([r_inner, r_outer])
    cp = np.array([radii[i] * arc[j] for j in range(3) for i in range(2)])  # radial fastest
    weights = np.array([w_arc[j] for j in range(3) for i in range(2)])
    return GeometryMap([radial, angular], cp, weights)


def twisted_box(twist=np.pi / 6, bend=0.3):
    """Bent and twisted unit box: quadratic splines (2 elements per
    direction) through a height-dependent rotation with a parabolic bend,
    control points at the Greville abscissae."""
    from .tensorspace import LexOrdering

    bases = [UnivariateBasis(uniform_open_knots(3, 2)) for _ in range(3)]

    def greville(basis):
        p = basis.order
        k = basis.kv.knots
        return np.array([k[n + 1: n + p].mean() for n in range(basis.num_basis)])

    g = [greville(b) for b in bases]
    ordering = LexOrdering([b.num_basis for b in bases])
    cp = np.empty((ordering.size, 3))
    for n in range(ordering.size):
        i, j, k = (int(v) for v in ordering.split(n))
        x, y, z = g[0][i], g[1][j], g[2][k]
        ang = twist * z
        u, v = x - 0.5, y - 0.5
        cp[n] = [np.cos(ang) * u - np.sin(ang) * v + 0.5 + bend * z * z, np.sin(ang) * u + np.cos(ang) * v + 0.5, z]
    return GeometryMap(bases, cp)


def named_geometry(name, d=None):
    if name == "identity2d":
        return identity_geometry(2)
    if name == "identity3d":
        return identity_geometry(3)
    if name == "identity":
        if d is None:
            raise ValueError("identity geometry needs the dimension")
        return identity_geometry(d)
    if name == "quarter_annulus":
        return quarter_annulus()
    if name == "twisted_box":
        return twisted_box()
    raise ValueError(f"unknown geometry '{name}'")
