"""Lexicographic tensor indexing, sparsity patterns and Alg. 3 (mirror of tensorspace.py).

Flat indices put direction 1 fastest (tensorspace.py:3-5).  The 1D
interaction patterns (Lemma 3.1) and the tensor CSR pattern are computed on
the GPU (igs_pattern_1d / igs_pattern, K2); `contract_to_points` (Alg. 3)
runs through igs_eval_field.
"""

import numpy as np

from . import _lib
from .errors import CapacityError

__all__ = (
    "LexOrdering",
    "TensorGeneratingSystem",
    "SparsityPattern",
    "nnz_pattern_1d",
    "nnz_count_exact",
    "tensor_pattern",
    "contract_to_points",
    "DEFAULT_MAX_PATTERN_NNZ",
)

DEFAULT_MAX_PATTERN_NNZ = 1 << 26


class LexOrdering:
    """Bijection between flat indices and multi-indices, direction 1 fastest (tensorspace.py:33-72)."""

    def __init__(self, dims):
        self.dims = tuple(int(n) for n in dims)
        if any(n < 0 for n in self.dims):
            raise ValueError("dimensions must be non-negative")
        strides = [1]
        for n in self.dims[:-1]:
            strides.append(strides[-1] * n)
        self.strides = tuple(strides)

    @property
    def d(self):
        return len(self.dims)

    @property
    def size(self):
        n = 1
        for v in self.dims:
            n *= v
        return n

    def flatten(self, multi):
        flat = 0
        for idx, stride in zip(multi, self.strides):
            flat = flat + np.asarray(idx) * stride
        return flat

    def split(self, flat):
        flat = np.asarray(flat)
        return tuple((flat // stride) % dim for stride, dim in zip(self.strides, self.dims))

    def component(self, delta, flat):
        return (np.asarray(flat) // self.strides[delta]) % self.dims[delta]


class TensorGeneratingSystem:
    """Per-direction evaluation tables at chosen derivative levels (tensorspace.py:75-112)."""

    def __init__(self, tables, derivs=None):
        self.tables = tuple(tables)
        if derivs is None:
            derivs = (0,) * len(self.tables)
        self.derivs = tuple(int(k) for k in derivs)
        if len(self.derivs) != len(self.tables):
            raise ValueError("one derivative level per direction required")
        for table, k in zip(self.tables, self.derivs):
            if not 0 <= k <= table.max_deriv:
                raise ValueError(f"table does not hold derivative level {k}")
        self.ordering = LexOrdering(t.num_functions for t in self.tables)

    @property
    def d(self):
        return len(self.tables)

    @property
    def dims(self):
        return self.ordering.dims

    @property
    def num_functions(self):
        return self.ordering.size

    @property
    def point_shape(self):
        return tuple(t.num_points for t in self.tables)

    def dense_factor(self, delta):
        return self.tables[delta].dense(self.derivs[delta])


class DirectionPairs:
    """1D pattern of one direction, m-major (tensorspace.py:230-259); device arrays."""

    def __init__(self, rowptr, cols, num_trial, num_test):
        self.rowptr_dev = rowptr
        self.cols_dev = cols
        self.num_trial = num_trial
        self.num_test = num_test
        self._host = None

    @property
    def num_pairs(self):
        return int(self.cols_dev.numel())

    def _h(self):
        if self._host is None:
            rp = self.rowptr_dev.cpu().numpy()
            n = self.cols_dev.cpu().numpy()
            m = np.repeat(np.arange(self.num_test, dtype=np.int64), np.diff(rp))
            self._host = (rp, n, m)
        return self._host

    @property
    def rowptr(self):
        return self._h()[0]

    @property
    def n(self):
        return self._h()[1]

    @property
    def m(self):
        return self._h()[2]

    @property
    def row_widths(self):
        return np.diff(self.rowptr)


class SparsityPattern:
    """Tensor-product CSR pattern shared by all derivative blocks (tensorspace.py:262-338).

    `indptr_dev` (int64) / `indices_dev` (int32 when the columns fit, else
    int64) are device tensors; `indptr` / `indices` (int64) are host copies
    made on first access.
    """

    def __init__(self, dir_pairs, trial_dims, test_dims, indptr_dev, indices_dev, nnz):
        self.dir_pairs = tuple(dir_pairs)
        self.trial_ordering = LexOrdering(trial_dims)
        self.test_ordering = LexOrdering(test_dims)
        self.indptr_dev = indptr_dev
        self.indices_dev = indices_dev
        self._nnz = int(nnz)
        self._host = {}

    @property
    def d(self):
        return len(self.dir_pairs)

    @property
    def shape(self):
        return self.test_ordering.size, self.trial_ordering.size

    @property
    def nnz(self):
        return self._nnz

    @property
    def indptr(self):
        if "indptr" not in self._host:
            self._host["indptr"] = self.indptr_dev.cpu().numpy()
        return self._host["indptr"]

    @property
    def indices(self):
        if "indices" not in self._host:
            self._host["indices"] = self.indices_dev.cpu().numpy().astype(np.int64, copy=False)
        return self._host["indices"]

    def value_perm(self, dir_order):
        """Permutation from the assembly-value layout (pair index of the
        first processed direction fastest) into CSR value order
        (tensorspace.py:324-332): CSR position k holds layout entry perm[k].
        Host numpy, cached per dir_order; the device kernels write CSR order
        directly and never need it."""
        dir_order = tuple(int(v) for v in dir_order)
        key = ("vperm", dir_order)
        if key not in self._host:
            d = self.d
            # layout axes, slowest first: the last processed direction first
            m_flat = np.zeros(1, dtype=np.int64)
            n_flat = np.zeros(1, dtype=np.int64)
            for delta in reversed(dir_order):
                dp = self.dir_pairs[delta]
                m_flat = (m_flat[:, None] + dp.m[None, :] * self.test_ordering.strides[delta]).ravel()
                n_flat = (n_flat[:, None] + dp.n[None, :] * self.trial_ordering.strides[delta]).ravel()
            del d
            self._host[key] = np.lexsort((n_flat, m_flat))
        return self._host[key]

    def to_scipy(self, values=None):
        import scipy.sparse

        m, n = self.shape
        if values is None:
            values = np.ones(self.nnz)
        if hasattr(values, "cpu"):
            values = values.cpu().numpy()
        return scipy.sparse.csr_matrix((values, self.indices, self.indptr), shape=(m, n))

    def to_torch(self, values):
        torch = _lib.require_cuda()
        m, n = self.shape
        ip, ix = self.indptr_dev, self.indices_dev
        if ip.dtype != ix.dtype:  # cuSPARSE wants one index type
            key = "torch_idx"
            if key not in self._host:
                self._host[key] = (ip.to(torch.int32), ix) if self.nnz < 2 ** 31 else (ip, ix.to(torch.int64))
            ip, ix = self._host[key]
        return torch.sparse_csr_tensor(ip, ix, values, size=(m, n))


def _direction_bases(system):
    if isinstance(system, TensorGeneratingSystem):
        return [t.basis for t in system.tables]
    return list(system)


def _pattern_problem(trial_bases, test_bases, rules):
    """IgsProblem carrying only what the pattern kernels read."""
    from ._problem import problem_struct_for_pattern

    return problem_struct_for_pattern(trial_bases, test_bases, rules)


def _pairs_1d(prob, keep, delta, num_trial, num_test):
    torch = _lib.require_cuda()
    import ctypes

    lib = _lib.load()
    rowptr = torch.empty(num_test + 1, dtype=torch.int64, device="cuda")
    count = ctypes.c_int64(0)
    st = lib.igs_pattern_1d(ctypes.byref(prob), delta, _lib.ptr(rowptr), None, ctypes.byref(count),
                            _lib.stream_handle())
    _lib.check(st, "pattern_1d")
    cols = torch.empty(int(count.value), dtype=torch.int64, device="cuda")
    if count.value:
        st = lib.igs_pattern_1d(ctypes.byref(prob), delta, _lib.ptr(rowptr), _lib.ptr(cols), None,
                                _lib.stream_handle())
        _lib.check(st, "pattern_1d")
    return DirectionPairs(rowptr, cols, num_trial, num_test)


def nnz_pattern_1d(trial, test, rule):
    """All (n, m) pairs whose csupps share a quadrature point, sorted by (m, n)."""
    prob, keep = _pattern_problem([trial], [test], [rule])
    dp = _pairs_1d(prob, keep, 0, trial.num_basis, test.num_basis)
    return np.column_stack([dp.n, dp.m])


def nnz_count_exact(trial, test):
    """Closed-form 1D pair count, Corollary 3.3 (tensorspace.py:211-227)."""
    if trial.domain != test.domain:
        raise ValueError("trial and test bases must share the domain")
    p, q = trial.order, test.order
    big_n, big_m = trial.num_basis, test.num_basis
    xi = np.unique(np.concatenate([trial.breakpoints, test.breakpoints]))
    b = trial.domain[1]
    correction = sum(trial.kv.multiplicity(x) * test.kv.multiplicity(x) for x in xi if x != b)
    return q * big_n + p * big_m - correction


def tensor_pattern(trial, test, quad, max_nnz=DEFAULT_MAX_PATTERN_NNZ):
    """Tensor-product CSR pattern (tensorspace.py:347-369), built on the GPU."""
    import ctypes

    torch = _lib.require_cuda()
    lib = _lib.load()
    trial_bases = _direction_bases(trial)
    test_bases = _direction_bases(test)
    if not len(trial_bases) == len(test_bases) == quad.dim:
        raise ValueError("inconsistent dimensions")
    prob, keep = _pattern_problem(trial_bases, test_bases, quad.rules)
    pairs = [
        _pairs_1d(prob, keep, k, tr.num_basis, te.num_basis)
        for k, (tr, te) in enumerate(zip(trial_bases, test_bases))
    ]
    total = 1
    for dp in pairs:
        total *= dp.num_pairs
    if total > max_nnz:
        raise CapacityError(f"pattern would hold {total} pairs, above the limit {max_nnz}")
    nrows = 1
    for b in test_bases:
        nrows *= b.num_basis
    indptr = torch.empty(nrows + 1, dtype=torch.int64, device="cuda")
    ncols = 1
    for b in trial_bases:
        ncols *= b.num_basis
    # int32 columns whenever they fit (2/3 of the index bytes; the host copy
    # is widened to the reference's int64)
    ib = 4 if ncols < 2 ** 31 else 8
    indices = torch.empty(total, dtype=torch.int32 if ib == 4 else torch.int64, device="cuda")
    rp = (ctypes.c_void_p * 3)(*[dp.rowptr_dev.data_ptr() for dp in pairs] + [0] * (3 - len(pairs)))
    cl = (ctypes.c_void_p * 3)(*[dp.cols_dev.data_ptr() for dp in pairs] + [0] * (3 - len(pairs)))
    for k, dp in enumerate(pairs):
        prob.num_pairs[k] = dp.num_pairs
    st = lib.igs_pattern(ctypes.byref(prob), rp, cl, 0, nrows, 0, _lib.ptr(indptr),
                         _lib.ptr(indices) if total else None, ib, _lib.stream_handle())
    _lib.check(st, "pattern")
    return SparsityPattern(pairs, [b.num_basis for b in trial_bases], [b.num_basis for b in test_bases],
                           indptr, indices, total)


def contract_to_points(tables, derivs, coeffs, counter=None, dir_order=None):
    """Coefficient grid -> values at all tensor points (Alg. 3, tensorspace.py:134-153).

    Returns a device tensor indexed [i_1, ..., i_d] (a permuted view of a
    contiguous buffer whose flat order has direction 1 fastest, i.e. the
    reference's `order="F"` ravel).
    """
    from ._problem import problem_struct_for_tables
    import ctypes

    torch = _lib.require_cuda()
    lib = _lib.load()
    tables = tuple(tables)
    d = len(tables)
    derivs = tuple(int(k) for k in derivs)
    prob, keep = problem_struct_for_tables(tables)
    n = 1
    for t in tables:
        n *= t.num_functions
    c = torch.as_tensor(coeffs, dtype=torch.float64, device="cuda").reshape(-1)
    if c.numel() != n:
        raise ValueError("coefficient length does not match the tables")
    c = c.contiguous()
    npts = 1
    for t in tables:
        npts *= t.num_points
    out = torch.empty(npts, dtype=torch.float64, device="cuda")
    ws_bytes = lib.igs_workspace_bytes(ctypes.byref(prob), _lib.OP_EVAL_FIELD, 0)
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device="cuda")
    dv = (ctypes.c_int8 * 3)(*(list(derivs) + [0] * (3 - d)))
    st = lib.igs_eval_field(ctypes.byref(prob), dv, _lib.ptr(c), _lib.ptr(out), _lib.ptr(ws), ws_bytes,
                            _lib.stream_handle())
    _lib.check(st, "eval_field")
    if counter is not None:
        counter.add_field_eval(field_eval_count([t.order for t in tables],
                                                [t.num_functions for t in tables],
                                                [t.num_points for t in tables], dir_order))
    shape = tuple(t.num_points for t in reversed(tables))
    return out.view(shape).permute(*reversed(range(d)))


def field_eval_count(orders, nfun, npts, dir_order=None):
    """MACs the reference counts for one contract_to_points (tensorspace.py:150-151)."""
    dims = list(nfun)
    total = 0
    order = range(len(orders)) if dir_order is None else dir_order
    for k in order:
        other = 1
        for j, v in enumerate(dims):
            if j != k:
                other *= v
        total += orders[k] * npts[k] * other
        dims[k] = npts[k]
    return total
