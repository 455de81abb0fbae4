"""Global sum-factorized assembly on the GPU (mirror of sumfac.py).

`assemble` / `assemble_block` keep the reference's signatures
(sumfac.py:358-379) and return a `SparseMatrix` over a shared
`SparsityPattern` (CSR, rows = test functions, ascending columns, band zeros
stored).  The values are computed by igs_assemble_values (K3): the fused
sm_100a kernel for the BASELINE shapes, else the stage-by-stage kernels.
`FlopCounter` is filled analytically with exactly the counts the reference
records (Eq. 13, sumfac.py:211) so the SPEC's FLOP law holds.
"""

import ctypes

import numpy as np

from . import _lib
from ._problem import problem_struct
from .bspline import tabulate
from .errors import CapacityError, UnsupportedDerivativeError
from .geometry import CoefficientField
from .tensorspace import DEFAULT_MAX_PATTERN_NNZ, tensor_pattern

__all__ = (
    "FlopCounter",
    "SparseMatrix",
    "AssemblyProblem",
    "assemble",
    "assemble_block",
    "rel_frobenius",
    "assemble_naive",
    "assemble_kronecker_dense",
    "DEFAULT_NAIVE_BUDGET",
    "DEFAULT_DENSE_BUDGET",
)

# nominal-work guards of the comparison oracles (sumfac.py:43-44)
DEFAULT_NAIVE_BUDGET = 4_000_000_000
DEFAULT_DENSE_BUDGET = 100_000_000


class FlopCounter:
    """Deterministic multiply-add counters (sumfac.py:47-85)."""

    __slots__ = ("block_update", "field_eval", "coeff_build")

    def __init__(self):
        self.block_update = 0
        self.field_eval = 0
        self.coeff_build = 0

    def add_block_update(self, n):
        self.block_update += int(n)

    def add_field_eval(self, n):
        self.field_eval += int(n)

    def add_coeff_build(self, n):
        self.coeff_build += int(n)

    def merge(self, other):
        self.block_update += other.block_update
        self.field_eval += other.field_eval
        self.coeff_build += other.coeff_build

    @property
    def total(self):
        return self.block_update + self.field_eval + self.coeff_build

    def as_tuple(self):
        return (self.block_update, self.field_eval, self.coeff_build)

    def __eq__(self, other):
        return isinstance(other, FlopCounter) and self.as_tuple() == other.as_tuple()

    def __repr__(self):
        return (f"FlopCounter(block_update={self.block_update}, field_eval={self.field_eval}, "
                f"coeff_build={self.coeff_build})")


class SparseMatrix:
    """CSR values (device tensor) over a shared SparsityPattern (sumfac.py:88-115)."""

    def __init__(self, pattern, values):
        if int(values.shape[0]) != pattern.nnz:
            raise ValueError("values not aligned with the pattern")
        self.pattern = pattern
        self.values = values

    @property
    def shape(self):
        return self.pattern.shape

    @property
    def nnz(self):
        return self.pattern.nnz

    def values_np(self):
        return self.values.cpu().numpy() if hasattr(self.values, "cpu") else np.asarray(self.values)

    def to_scipy(self):
        return self.pattern.to_scipy(self.values_np())

    def toarray(self):
        return self.to_scipy().toarray()

    def matvec(self, u):
        """A @ u on the device (cuSPARSE through torch); numpy in -> numpy out."""
        torch = _lib.require_cuda()
        host = not isinstance(u, torch.Tensor)
        x = torch.as_tensor(np.asarray(u, dtype=float) if host else u, dtype=torch.float64,
                            device="cuda").reshape(-1, 1)
        y = (self.pattern.to_torch(self.values) @ x).reshape(-1)
        return y.cpu().numpy() if host else y

    def copy(self):
        return SparseMatrix(self.pattern, self.values.clone())

    def write_matrix_market(self, path):
        """MatrixMarket coordinate export (1-based, 17 significant digits,
        SPEC.md:426); the CSR arrays are copied to the host once."""
        lib = _lib.load()
        indptr = np.ascontiguousarray(self.pattern.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(self.pattern.indices, dtype=np.int64)
        values = np.ascontiguousarray(self.values_np(), dtype=np.float64)
        m, n = self.shape
        st = lib.igs_write_matrix_market(str(path).encode(), m, n, indptr.ctypes.data, indices.ctypes.data,
                                         values.ctypes.data)
        _lib.check(st, "write_matrix_market")


def rel_frobenius(a, b):
    """Relative Frobenius distance ||a - b||_F / ||b||_F (sumfac.py:118-141).

    Same-pattern SparseMatrix pairs compare their value arrays (on the
    device); anything else is densified on the host like the reference.
    """
    if isinstance(a, SparseMatrix) and isinstance(b, SparseMatrix) and (
            a.pattern is b.pattern or (a.pattern.nnz == b.pattern.nnz and a.shape == b.shape
                                       and np.array_equal(a.pattern.indptr, b.pattern.indptr)
                                       and np.array_equal(a.pattern.indices, b.pattern.indices))):
        torch = _lib.require_cuda()
        va = torch.as_tensor(a.values, device="cuda")
        vb = torch.as_tensor(b.values, device="cuda")
        num = float(torch.linalg.vector_norm(va - vb))
        den = float(torch.linalg.vector_norm(vb))
    else:
        def dense(x):
            if isinstance(x, SparseMatrix):
                return x.toarray()
            if hasattr(x, "toarray"):
                return x.toarray()
            if hasattr(x, "cpu"):
                return x.cpu().numpy()
            return np.asarray(x, dtype=float)

        da, db = dense(a), dense(b)
        num = float(np.linalg.norm(da - db))
        den = float(np.linalg.norm(db))
    if den == 0.0:
        return 0.0 if num == 0.0 else np.inf
    return num / den


class AssemblyProblem:
    """Trial/test spaces, a tensor quadrature and a coefficient field (sumfac.py:232-337)."""

    def __init__(self, trial, test, quad, coeff, max_nnz=DEFAULT_MAX_PATTERN_NNZ):
        self.trial = tuple(trial)
        self.test = tuple(test)
        self.quad = quad
        if not len(self.trial) == len(self.test) == quad.dim:
            raise ValueError("trial, test and quadrature dimensions differ")
        self.theta_set = tuple(tuple(t) for t in coeff.theta_set)
        self.eta_set = tuple(tuple(t) for t in coeff.eta_set)
        self.max_nnz = max_nnz
        for delta, basis in enumerate(self.trial):
            if max(t[delta] for t in self.theta_set) >= basis.order:
                raise UnsupportedDerivativeError(f"trial derivative exceeds order in direction {delta}")
        for delta, basis in enumerate(self.test):
            if max(t[delta] for t in self.eta_set) >= basis.order:
                raise UnsupportedDerivativeError(f"test derivative exceeds order in direction {delta}")
        if not isinstance(coeff, CoefficientField):
            raise TypeError("coeff must be a CoefficientField (lazy geometry providers are out of scope)")
        slab = getattr(coeff, "slab", None)
        if slab is None:
            if coeff.num_points != quad.num_points:
                raise ValueError("coefficient field does not match the point grid")
        else:
            rule = quad.rules[-1]
            if rule.points_per_element <= 0:
                raise ValueError("slab fields need a per-element rule in the last direction")
            want = quad.num_points // rule.num_points * (slab[1] - slab[0]) * rule.points_per_element
            if coeff.num_points != want:
                raise ValueError("slab coefficient field does not match the slab's points")
        self.slab = slab
        self._field = coeff
        self._cache = {}

    @property
    def d(self):
        return len(self.trial)

    @property
    def shape(self):
        m = n = 1
        for b in self.test:
            m *= b.num_basis
        for b in self.trial:
            n *= b.num_basis
        return m, n

    def coeff_field(self, counter=None):
        return self._field

    @property
    def coeff(self):
        return self._field

    def trial_tables(self):
        tabs = self._cache.get("trial_tables")
        if tabs is None:
            md = max(max(t) for t in self.theta_set)
            tabs = tuple(_tabulate(b, r.points, min(md, b.order - 1)) for b, r in zip(self.trial, self.quad.rules))
            self._cache["trial_tables"] = tabs
        return tabs

    def test_tables(self):
        tabs = self._cache.get("test_tables")
        if tabs is None:
            if self.test == self.trial and self.eta_set == self.theta_set:
                tabs = self.trial_tables()
            else:
                md = max(max(t) for t in self.eta_set)
                tabs = tuple(_tabulate(b, r.points, min(md, b.order - 1)) for b, r in zip(self.test, self.quad.rules))
            self._cache["test_tables"] = tabs
        return tabs

    def pattern(self):
        pat = self._cache.get("pattern")
        if pat is None:
            pat = tensor_pattern(self.trial, self.test, self.quad, max_nnz=self.max_nnz)
            self._cache["pattern"] = pat
        return pat

    def core(self, dir_order=None):
        """The assembly engine for one direction order (sumfac.py:325-337);
        here a thin handle over the device kernels (see _DeviceCore)."""
        key = ("core", tuple(dir_order) if dir_order is not None else None)
        core = self._cache.get(key)
        if core is None:
            core = _DeviceCore(self, dir_order)
            self._cache[key] = core
        return core

    def struct(self, dir_order=None, slab=None, with_pattern=True):
        """The C igs_problem for this problem (cached per dir_order/slab)."""
        key = ("struct", tuple(dir_order) if dir_order is not None else None,
               tuple(slab) if slab is not None else None, with_pattern)
        hit = self._cache.get(key)
        if hit is None:
            f = self._field
            num_pairs = [dp.num_pairs for dp in self.pattern().dir_pairs] if with_pattern else None
            hit = problem_struct(self.trial, self.test, self.quad.rules, self.trial_tables(),
                                 self.test_tables(), self.theta_set, self.eta_set, f.plane_of,
                                 f.n_planes, f.plane_stride, dir_order=dir_order, num_pairs=num_pairs,
                                 slab=slab)
            self._cache[key] = hit
        return hit


class _DeviceCore:
    """Device counterpart of the reference's _Core (sumfac.py:143-229): the
    tables, pattern and direction order are fixed by the problem; values
    come back in CSR order from igs_assemble_values."""

    def __init__(self, problem, dir_order=None):
        d = problem.d
        self.problem = problem
        self.dir_order = tuple(dir_order) if dir_order is not None else tuple(range(d))
        if sorted(self.dir_order) != list(range(d)):
            raise ValueError("dir_order must be a permutation of the directions")
        self.pattern = problem.pattern()
        self.d = d

    def assemble_values(self, counter=None):
        """CSR-ordered values of the summed non-zero blocks (device tensor)."""
        return _run_assembly(self.problem, None, counter, self.dir_order)

    def block_values_csr(self, theta, eta, counter=None):
        """One derivative block's values in CSR order (device tensor)."""
        theta, eta = _check_block_indices(self.problem, theta, eta)
        i, j = self.problem.eta_set.index(eta), self.problem.theta_set.index(theta)
        torch = _lib.require_cuda()
        if self.problem.coeff_field().is_zero_block(i, j) or self.pattern.nnz == 0:
            return torch.zeros(self.pattern.nnz, dtype=torch.float64, device="cuda")
        return _run_assembly(self.problem, (i, j), counter, self.dir_order)


def _tabulate(basis, points, max_deriv):
    # restricted bases (localized.RestrictedBasis) tabulate through their parent
    if hasattr(basis, "tabulate"):
        return basis.tabulate(points, max_deriv)
    return tabulate(basis, points, max_deriv)


def _check_block_indices(problem, theta, eta):
    theta = tuple(theta)
    eta = tuple(eta)
    for delta, basis in enumerate(problem.trial):
        if theta[delta] >= basis.order:
            raise UnsupportedDerivativeError(f"trial derivative {theta[delta]} >= order {basis.order}")
    for delta, basis in enumerate(problem.test):
        if eta[delta] >= basis.order:
            raise UnsupportedDerivativeError(f"test derivative {eta[delta]} >= order {basis.order}")
    if theta not in problem.theta_set or eta not in problem.eta_set:
        raise ValueError("derivative multi-index not in the problem's index sets")
    return theta, eta


def block_update_count(problem, theta, eta, dir_order=None):
    """The reference's block_update MACs for one (theta, eta) block (Eq. 13)."""
    d = problem.d
    order = tuple(range(d)) if dir_order is None else tuple(dir_order)
    pat = problem.pattern()
    dims = list(problem.quad.shape)
    total = 0
    for delta in order:
        p = problem.trial[delta].order
        q = problem.test[delta].order
        x = problem.quad.shape[delta]
        w_nnz = p * q * x if dims[delta] and pat.dir_pairs[delta].num_pairs else 0
        other = 1
        for j, v in enumerate(dims):
            if j != delta:
                other *= v
        total += w_nnz * other
        dims[delta] = pat.dir_pairs[delta].num_pairs
    return total


def _run_assembly(problem, block, counter, dir_order, flags=0, row_range=None, out=None):
    """Values of rows [lo, hi) (default: all) in CSR order.  With a slab
    coefficient field (elements [slab_lo, slab_hi) of the last direction,
    SURVEY §8(e)) the rows must only need slab elements; the result then
    holds the range's entries at the front (nnz of the range), as for any
    row range."""
    torch = _lib.require_cuda()
    lib = _lib.load()
    pat = problem.pattern()
    prob, keep = problem.struct(dir_order, slab=problem.slab)
    nrows = pat.shape[0]
    if row_range is None and problem.slab is not None:
        raise ValueError("a slab coefficient field assembles row ranges only (see sharded.SlabAssembly)")
    lo, hi = (0, nrows) if row_range is None else row_range
    if row_range is None:
        n_out = pat.nnz
    else:
        ip = pat.indptr
        n_out = int(ip[hi] - ip[lo])
    # per-(block, dir_order, flags) launch data, cached on the problem like the
    # reference's lazily built tables/core (sumfac.py:296-337): the fused-path
    # test, the workspace, the 1D pattern pointer arrays and the analytic
    # FlopCounter increments (warm calls then cost one C-ABI call)
    key = ("asm_launch", block, None if dir_order is None else tuple(dir_order), flags)
    lc = problem._cache.get(key)
    if lc is None:
        fused = bool(block is None and not (flags & _lib.FLAG_FORCE_GENERIC)
                     and lib.igs_fused_path(ctypes.byref(prob), _lib.OP_ASSEMBLE))
        ws_bytes = lib.igs_workspace_bytes(ctypes.byref(prob), _lib.OP_ASSEMBLE, flags)
        ws = problem._cache.get(("ws_asm", ws_bytes))
        if ws is None:
            ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
            problem._cache[("ws_asm", ws_bytes)] = ws
        d = problem.d
        rp = (ctypes.c_void_p * 3)(*[dp.rowptr_dev.data_ptr() for dp in pat.dir_pairs] + [0] * (3 - d))
        cl = (ctypes.c_void_p * 3)(*[dp.cols_dev.data_ptr() for dp in pat.dir_pairs] + [0] * (3 - d))
        bi, bj = block if block is not None else (-1, -1)
        f = problem.coeff_field()
        updates = 0
        for j, th in enumerate(problem.theta_set):
            for i, et in enumerate(problem.eta_set):
                if block is not None and (i, j) != (bi, bj):
                    continue
                if f.is_zero_block(i, j):
                    continue
                updates += block_update_count(problem, th, et, dir_order)
        lc = (fused, ws_bytes, ws, rp, cl, bi, bj, updates)
        problem._cache[key] = lc
    fused, ws_bytes, ws, rp, cl, bi, bj, updates = lc
    # the fused kernels write every entry of the range (band zeros included)
    if out is not None:
        # caller-provided value storage (contiguous float64 CUDA, >= n_out entries)
        if out.dtype != torch.float64 or out.device.type != "cuda" or not out.is_contiguous() or out.numel() < n_out:
            raise ValueError(f"out must be a contiguous float64 CUDA tensor with >= {n_out} entries")
        values = out.reshape(-1)[:n_out]
        if not fused:
            values.zero_()
    else:
        values = (torch.empty if fused else torch.zeros)(n_out, dtype=torch.float64, device="cuda")
    if n_out == 0:
        return values
    f = problem.coeff_field()
    st = lib.igs_assemble_values(ctypes.byref(prob), rp, cl, lo, hi, bi, bj, _lib.ptr(f.planes),
                                 _lib.ptr(values), _lib.ptr(ws), ws_bytes, flags, _lib.stream_handle())
    _lib.check(st, "assemble_values")
    if counter is not None:
        counter.add_block_update(updates)
    return values


def assemble_block(problem, theta, eta, counter=None, dir_order=None):
    """Assemble the single derivative block (theta, eta) on the shared pattern."""
    torch = _lib.require_cuda()
    counter = counter if counter is not None else FlopCounter()
    theta, eta = _check_block_indices(problem, theta, eta)
    pattern = problem.pattern()
    i = problem.eta_set.index(eta)
    j = problem.theta_set.index(theta)
    if problem.coeff_field().is_zero_block(i, j) or pattern.nnz == 0:
        return SparseMatrix(pattern, torch.zeros(pattern.nnz, dtype=torch.float64, device="cuda"))
    return SparseMatrix(pattern, _run_assembly(problem, (i, j), counter, dir_order))


def assemble(problem, counter=None, dir_order=None, flags=0):
    """Assemble the full matrix: the sum of all derivative blocks (sumfac.py:373-379)."""
    counter = counter if counter is not None else FlopCounter()
    vals = _run_assembly(problem, None, counter, dir_order, flags)
    return SparseMatrix(problem.pattern(), vals)


def fused_path(problem, op="assemble", dir_order=None):
    """1 when the fused sm_100a kernel serves this problem, 0 for the generic kernels."""
    lib = _lib.load()
    prob, keep = problem.struct(dir_order)
    return int(lib.igs_fused_path(ctypes.byref(prob), _lib.OP_ASSEMBLE if op == "assemble" else _lib.OP_APPLY))


def _naive_values(problem, counter):
    torch = _lib.require_cuda()
    lib = _lib.load()
    pat = problem.pattern()
    values = torch.zeros(pat.nnz, dtype=torch.float64, device="cuda")
    if pat.nnz == 0 or problem.quad.num_points == 0:
        return values
    if problem.slab is not None:
        raise ValueError("the naive oracle takes whole coefficient fields (no slab)")
    prob, keep = problem.struct(None)
    f = problem.coeff_field()
    updates = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = lib.igs_assemble_naive(ctypes.byref(prob), _lib.ptr(pat.indptr_dev), _lib.ptr(pat.indices_dev),
                                pat.indices_dev.element_size(), 0, pat.shape[0], 0, pat.nnz,
                                _lib.ptr(f.planes), _lib.ptr(values), _lib.ptr(updates), _lib.stream_handle())
    _lib.check(st, "assemble_naive")
    if counter is not None:
        counter.add_block_update(int(updates.item()))
    return values


def assemble_naive(problem, counter=None, budget=DEFAULT_NAIVE_BUDGET):
    """Direct quadrature sum per pattern entry: the comparison oracle
    (sumfac.py:388-477), one device thread per CSR entry (igs_assemble_naive).

    Same guard as the reference: pattern nnz x points x derivative blocks
    above `budget` raises CapacityError; the counter gets the reference's
    block_update count (the support-overlap box of every entry and block).
    """
    counter = counter if counter is not None else FlopCounter()
    pattern = problem.pattern()
    n_blocks = len(problem.theta_set) * len(problem.eta_set)
    nominal = pattern.nnz * problem.quad.num_points * n_blocks
    if nominal > budget:
        raise CapacityError(f"naive assembly would take {nominal} nominal operations, above {budget}")
    return SparseMatrix(pattern, _naive_values(problem, counter))


def assemble_kronecker_dense(problem, budget=DEFAULT_DENSE_BUDGET):
    """Dense (test x trial) numpy matrix of the full operator (sumfac.py:480-509).

    The reference materialises Kronecker products of the dense 1D tables;
    every entry outside the tensor pattern is an exact zero of that product,
    so the device computes the pattern entries by direct quadrature
    (igs_assemble_naive) and scatters them into the dense array.
    """
    m_total, n_total = problem.shape
    npts = problem.quad.num_points
    if m_total * n_total * max(npts, 1) > budget:
        raise CapacityError("instance too large for the dense Kronecker oracle")
    out = np.zeros((m_total, n_total))
    pat = problem.pattern()
    if pat.nnz == 0:
        return out
    vals = _naive_values(problem, None).cpu().numpy()
    rows = np.repeat(np.arange(m_total), np.diff(pat.indptr))
    out[rows, pat.indices] = vals
    return out


__all__ += ("block_update_count", "fused_path")
