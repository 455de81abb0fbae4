"""Localized sum factorization (PAPER §4).

The reference package specifies but does not ship this module.  A partition
splits the element grid into disjoint axis-aligned boxes; each box gets its
restricted bases (the global B-splines active on the box, supports clipped
to it), its part of the quadrature and of the coefficient field, and is
assembled / applied by the same device kernels as a global problem (the
fused kernels serve interior boxes of uniform meshes: a box looks like a
small global mesh).  Results are accumulated into the global CSR / vector
in a fixed box order (Eq. 19: A = Σ_D S_Ψ,Dᵀ A_D S_Φ,D), so they are
deterministic; the FLOP counter sees each box's own sum-factorization cost.
"""

import warnings
from fractions import Fraction

import numpy as np

from . import _lib
from .sumfac import AssemblyProblem, FlopCounter, SparseMatrix, assemble

__all__ = ("Partition", "RestrictedBasis", "LocalSystem", "make_partition", "repetition_ratio", "restrict",
           "assemble_localized", "apply_localized")


class Partition:
    """Disjoint boxes of element ranges [lo_δ, hi_δ) covering the grid."""

    def __init__(self, boxes, num_elements, strategy="custom", fallback=False, narrow=None):
        self.boxes = [tuple((int(a), int(b)) for a, b in box) for box in boxes]
        self.num_elements = tuple(int(k) for k in num_elements)
        self.strategy = strategy
        self.fallback = bool(fallback)   # mesh smaller than one macro element: single global box
        self.narrow = narrow             # the size-1 direction of a narrow partition
        self._check()

    def _check(self):
        d = len(self.num_elements)
        seen = np.zeros(self.num_elements[::-1], dtype=np.int8) if d else None
        for box in self.boxes:
            if len(box) != d or any(not 0 <= a < b <= k for (a, b), k in zip(box, self.num_elements)):
                raise ValueError(f"box {box} outside the element grid")
            seen[tuple(slice(a, b) for a, b in reversed(box))] += 1
        if not np.all(seen == 1):
            raise ValueError("boxes must be pairwise disjoint and cover every element")

    def sizes(self, box_index):
        return tuple(b - a for a, b in self.boxes[box_index])

    def __len__(self):
        return len(self.boxes)


def _split(k, s, absorb):
    """[0, k) into runs of s; the remainder is merged into the last run when
    `absorb` (sizes in [s, 2s)), else kept as a shorter trailing run."""
    if s >= k:
        return [(0, k)]
    cuts = list(range(0, k, s))
    runs = [(c, min(k, c + s)) for c in cuts]
    if absorb and runs[-1][1] - runs[-1][0] < s:
        last = runs.pop()
        runs[-1] = (runs[-1][0], last[1])
    return runs


def make_partition(bases, strategy, sizes=None, narrow_dir=None):
    """Partition of the bases' element grid (SPEC.md make_partition).

    strategy: "global" (one box), "element" / "per-element" (Example 4.3),
    "macro" / "macro-standard" (boxes of >= order elements per direction,
    Example 4.4; trailing boxes absorb the remainder), "narrow" /
    "macro-narrow" (one direction, by default the last, of size 1, the
    others >= order, Example 4.7), "custom" (explicit `sizes`).
    """
    ks = [b.num_elements for b in bases]
    orders = [b.order for b in bases]
    d = len(ks)
    strategy = {"per-element": "element", "macro-standard": "macro", "macro-narrow": "narrow"}.get(strategy,
                                                                                                 strategy)
    fallback = False
    narrow = None
    if strategy == "global":
        runs = [[(0, k)] for k in ks]
    elif strategy == "element":
        runs = [[(e, e + 1) for e in range(k)] for k in ks]
    elif strategy in ("macro", "narrow", "custom"):
        if strategy == "custom":
            if sizes is None or len(sizes) != d:
                raise ValueError("custom partitions need one box size per direction")
            s = [int(v) for v in sizes]
        else:
            s = [int(v) for v in sizes] if sizes is not None else list(orders)
        if strategy == "narrow":
            narrow = d - 1 if narrow_dir is None else int(narrow_dir)
            s[narrow] = 1
        if any(v < 1 for v in s):
            raise ValueError("box sizes must be positive")
        if strategy != "custom" and any(k < v for k, v, dd in zip(ks, s, range(d)) if dd != narrow):
            warnings.warn("mesh smaller than one macro element per direction: single global box")
            return Partition([tuple((0, k) for k in ks)], ks, strategy, fallback=True)
        runs = [_split(k, v, absorb=strategy != "custom") for k, v in zip(ks, s)]
    else:
        raise ValueError(f"unknown strategy '{strategy}'")
    boxes = []
    for idx in np.ndindex(*[len(r) for r in reversed(runs)]):
        boxes.append(tuple(runs[dd][idx[d - 1 - dd]] for dd in range(d)))   # direction 0 fastest
    return Partition(boxes, ks, strategy, fallback=fallback, narrow=narrow)


class RestrictedBasis:
    """The global B-splines whose support meets elements [e_lo, e_hi),
    restricted to that box (PAPER §4.2, Φ_D): local index n - offset, support
    clipped to the box, tables = the global tabulation at the box's points."""

    def __init__(self, basis, e_lo, e_hi):
        bp = np.asarray(basis.breakpoints)
        if not 0 <= e_lo < e_hi <= len(bp) - 1:
            raise ValueError("element range outside the basis")
        a, b = float(bp[e_lo]), float(bp[e_hi])
        lo, hi = np.asarray(basis.csupp_lo), np.asarray(basis.csupp_hi)
        active = np.nonzero((lo < b) & (hi > a))[0]
        self.parent = basis
        self.order = basis.order
        self.offset = int(active[0])
        self.num_basis = int(active[-1] + 1 - active[0])
        self.csupp_lo = np.maximum(lo[self.offset: self.offset + self.num_basis], a)
        self.csupp_hi = np.minimum(hi[self.offset: self.offset + self.num_basis], b)
        self._bp = bp[e_lo: e_hi + 1].copy()
        self._max_smooth = basis.max_smoothness
        self._dev = {}

    @property
    def breakpoints(self):
        return self._bp

    @property
    def num_elements(self):
        return len(self._bp) - 1

    @property
    def max_smoothness(self):
        return self._max_smooth

    @property
    def domain(self):
        return float(self._bp[0]), float(self._bp[-1])

    def device_csupp(self):
        t = self._dev.get("csupp")
        if t is None:
            torch = _lib.require_cuda()
            t = (torch.tensor(self.csupp_lo, dtype=torch.float64, device="cuda"),
                 torch.tensor(self.csupp_hi, dtype=torch.float64, device="cuda"))
            self._dev["csupp"] = t
        return t

    def tabulate(self, points, max_deriv):
        from .bspline import BasisEvalTable, tabulate

        t = tabulate(self.parent, points, max_deriv)
        return BasisEvalTable(t.order, self.num_basis, t.points, t.max_deriv, t.first_active - self.offset,
                              t.values, basis=self, points_dev=t.points_dev)


class LocalSystem:
    """One box: restricted trial/test bases, local quadrature, selection
    offsets (the tensor-product S_Φ,D / S_Ψ,D of Eq. 19 are index ranges)."""

    def __init__(self, box, trial, test, quad, point_ranges):
        self.box = box
        self.trial = tuple(trial)
        self.test = tuple(test)
        self.quad = quad
        self.point_ranges = tuple(point_ranges)

    @property
    def trial_ranges(self):
        return tuple((b.offset, b.offset + b.num_basis) for b in self.trial)

    @property
    def test_ranges(self):
        return tuple((b.offset, b.offset + b.num_basis) for b in self.test)

    def selection(self, which="trial"):
        """Flat global indices of the local functions (direction 0 fastest)."""
        ranges = self.trial_ranges if which == "trial" else self.test_ranges
        n_glob = [b.parent.num_basis for b in (self.trial if which == "trial" else self.test)]
        idx = np.zeros(1, dtype=np.int64)
        stride = 1
        for (a, b), n in zip(ranges, n_glob):
            idx = (idx[None, :] + stride * np.arange(a, b, dtype=np.int64)[:, None]).reshape(-1)
            stride *= n
        return idx


def _local_rule(rule, e_lo, e_hi):
    from . import quadrature

    if rule.points_per_element > 0 and getattr(rule, "breakpoints", None) is not None:
        bp = np.asarray(rule.breakpoints)
        return quadrature.per_element_rule(bp[e_lo: e_hi + 1], rule.points_per_element), (
            e_lo * rule.points_per_element, e_hi * rule.points_per_element)
    raise ValueError("localized strategies need per-element quadrature rules")


def restrict(bases_trial, bases_test, quad, partition, box_index):
    """LocalSystem of one box (SPEC.md restrict)."""
    from .quadrature import TensorQuadrature

    box = partition.boxes[box_index]
    rules, ranges = [], []
    for rule, (a, b) in zip(quad.rules, box):
        r, pr = _local_rule(rule, a, b)
        rules.append(r)
        ranges.append(pr)
    trial = [RestrictedBasis(bs, a, b) for bs, (a, b) in zip(bases_trial, box)]
    test = [RestrictedBasis(bs, a, b) for bs, (a, b) in zip(bases_test, box)]
    return LocalSystem(box, trial, test, TensorQuadrature(rules), ranges)


def repetition_ratio(partition, trial, test):
    """R = max(Σ_D N_D / N, Σ_D M_D / M) (Eq. 20), exact."""
    n = int(np.prod([b.num_basis for b in trial]))
    m = int(np.prod([b.num_basis for b in test]))
    sn = sm = 0
    for box in partition.boxes:
        sn += int(np.prod([RestrictedBasis(b, lo, hi).num_basis for b, (lo, hi) in zip(trial, box)]))
        sm += int(np.prod([RestrictedBasis(b, lo, hi).num_basis for b, (lo, hi) in zip(test, box)]))
    return max(Fraction(sn, n), Fraction(sm, m))


def _local_field(problem, ls):
    """The box's coefficient planes (a sub-block of the point grid)."""
    from .geometry import CoefficientField

    torch = _lib.require_cuda()
    f = problem.coeff_field()
    shape = [r.num_points for r in problem.quad.rules]
    grid = f.planes.view([f.n_planes] + shape[::-1])
    sl = tuple(slice(a, b) for a, b in reversed(ls.point_ranges))
    planes = grid[(slice(None),) + sl].contiguous().view(f.n_planes, -1)
    del torch
    return CoefficientField.from_planes(f.theta_set, f.eta_set, planes, f.plane_of, ls.quad.shape)


def _direction_order(partition, d, policy):
    if policy == "auto" and partition.narrow is not None and partition.narrow != d - 1:
        return tuple(k for k in range(d) if k != partition.narrow) + (partition.narrow,)
    return None


def _local_positions(pattern_g, ls, lpat):
    """Global CSR positions of the local pattern's entries.  In a tensor
    pattern row m, column n sits at indptr[m] + ((r_2·w_1 + r_1)·w_0 + r_0)
    with r_δ the offset of n_δ in the 1D row m_δ and w_δ its width."""
    torch = _lib.require_cuda()
    rows = torch.repeat_interleave(torch.arange(lpat.shape[0], device="cuda"), torch.diff(lpat.indptr_dev))
    mrem, nrem = rows, lpat.indices_dev.long()
    m_flat = torch.zeros_like(rows)
    stride = 1
    per_dir = []
    for k, (te, tr) in enumerate(zip(ls.test, ls.trial)):
        m_k = mrem % te.num_basis + te.offset
        n_k = nrem % tr.num_basis + tr.offset
        mrem, nrem = mrem // te.num_basis, nrem // tr.num_basis
        rp, cols = pattern_g.dir_pairs[k].rowptr_dev, pattern_g.dir_pairs[k].cols_dev
        first = rp[m_k]
        per_dir.append((n_k - cols[first], rp[m_k + 1] - first))
        m_flat = m_flat + stride * m_k
        stride *= te.parent.num_basis
    off = torch.zeros_like(rows)
    for r_k, w_k in reversed(per_dir):
        off = off * w_k + r_k
    return pattern_g.indptr_dev[m_flat] + off


def assemble_localized(problem, partition, direction_policy="auto", counter=None):
    """A = Σ_D S_Ψ,Dᵀ A_D S_Φ,D (Eq. 19): every box assembled by the device
    kernels on its LocalSystem, accumulated into the global CSR in box order."""
    torch = _lib.require_cuda()
    pat = problem.pattern()
    values = torch.zeros(pat.nnz, dtype=torch.float64, device="cuda")
    d = problem.d
    order = _direction_order(partition, d, direction_policy)
    for i in range(len(partition)):
        ls = restrict(problem.trial, problem.test, problem.quad, partition, i)
        local = AssemblyProblem(ls.trial, ls.test, ls.quad, _local_field(problem, ls), max_nnz=problem.max_nnz)
        A_loc = assemble(local, counter=counter, dir_order=order)
        pos = _local_positions(pat, ls, local.pattern())
        values.index_add_(0, pos, A_loc.values)  # distinct positions within a box
    return SparseMatrix(pat, values)


def apply_localized(op_or_problem, partition, u, counter=None):
    """v = Σ_D S_Ψ,Dᵀ A_D S_Φ,D u with per-box matrix-free applies (§4.1)."""
    from .matfree import MatrixFreeOperator

    torch = _lib.require_cuda()
    problem = op_or_problem.problem if isinstance(op_or_problem, MatrixFreeOperator) else op_or_problem
    host = not isinstance(u, torch.Tensor)
    x = torch.as_tensor(np.asarray(u, dtype=float) if host else u, dtype=torch.float64, device="cuda")
    m, n = problem.shape
    if x.numel() != n:
        raise ValueError("vector length does not match the trial space")
    y = torch.zeros(m, dtype=torch.float64, device="cuda")
    xg = x.view([b.num_basis for b in reversed(problem.trial)])
    yg = y.view([b.num_basis for b in reversed(problem.test)])
    for i in range(len(partition)):
        ls = restrict(problem.trial, problem.test, problem.quad, partition, i)
        local = AssemblyProblem(ls.trial, ls.test, ls.quad, _local_field(problem, ls))
        op = MatrixFreeOperator(local)
        xs = xg[tuple(slice(a, b) for a, b in reversed(ls.trial_ranges))].contiguous().view(-1)
        ys = op.apply_device(xs)
        yg[tuple(slice(a, b) for a, b in reversed(ls.test_ranges))] += ys.view(
            [b.num_basis for b in reversed(ls.test)])
        if counter is not None:
            op.count(counter)  # adds this box's apply MACs in place
    return y.cpu().numpy() if host else y


del FlopCounter
