"""Slab partition of the matrix-free apply along the last (slowest) direction.

SURVEY §8(e): rank r owns elements [lo_r, hi_r) of the last direction and
the DoF layers [lo_r, hi_r) (the last rank also the trailing order-1
layers).  One apply is

  1. ghost gather : x layers [hi_r, hi_r + p - 1) from rank r+1      (p2p)
  2. local apply  : y_local over DoF layers [lo_r, hi_r + p - 1)     (K4 on the slab)
  3. ghost reduce : trailing p-1 y layers added into rank r+1          (p2p)

The exchanges are point-to-point sends/receives through torch.distributed
(NCCL over NVLink on GPUs, gloo in the CPU tests), issued as one batched
group per step.  Each message is (p-1)·N0·N1 doubles.

The assembly needs no communication (SlabAssembly): rank r owns the rows of
DoF layers [lo_r, hi_r) of the last direction and reads the coefficients of
elements [lo_r - 2(p-1), hi_r + p - 1) — its slab plus the halo the one-pass
symmetric kernel needs for the mirrored half of its rows — and writes its
contiguous CSR slice; global indptr offsets are closed-form.
"""

import torch
import torch.distributed as dist


def layers_copy(dst, src, add=False):
    """dst (+)= src over contiguous DoF layers: the K5 halo kernel
    (igs_layers_copy) on the device, torch on the CPU (gloo tests)."""
    n = src.numel()
    if n == 0:
        return dst
    if dst.is_cuda:
        from . import _lib

        lib = _lib.load()
        _lib.check(lib.igs_layers_copy(_lib.ptr(src), _lib.ptr(dst), n, int(bool(add)), _lib.stream_handle()),
                   "layers_copy")
    elif add:
        dst.add_(src)
    else:
        dst.copy_(src)
    return dst


class SlabPartition:
    """Balanced split of K elements (last direction) over `world` ranks."""

    def __init__(self, num_elements, order, world):
        if world > num_elements:
            raise ValueError("more ranks than element layers")
        self.K = int(num_elements)
        self.p = int(order)
        self.world = int(world)
        base, rem = divmod(self.K, self.world)
        self.bounds = []
        lo = 0
        for r in range(self.world):
            hi = lo + base + (1 if r < rem else 0)
            self.bounds.append((lo, hi))
            lo = hi
        for r in range(self.world - 1):
            lo, hi = self.bounds[r + 1]
            if hi - lo < self.p - 1 and r + 1 < self.world - 1:
                raise ValueError("slabs must hold at least order-1 element layers")

    def elements(self, r):
        return self.bounds[r]

    def own_layers(self, r):
        """DoF layers owned by rank r (disjoint, covering K + p - 1)."""
        lo, hi = self.bounds[r]
        return (lo, hi + self.p - 1) if r == self.world - 1 else (lo, hi)

    def local_layers(self, r):
        """DoF layers touched by rank r's elements (own + ghost)."""
        lo, hi = self.bounds[r]
        return lo, hi + self.p - 1


class ShardedApply:
    """Runs one rank's part of a slab-partitioned apply.

    compute(x_local, y_local) must write the slab's y (DoF layers
    local_layers(rank)) from x on the same layers — e.g.
    MatrixFreeOperator(problem, slab=...).apply_device, or the CPU oracle.
    """

    def __init__(self, part, rank, layer_size, compute, device, dtype=torch.float64, group=None, split=None):
        """split=(interior, boundary): optional overlap of the ghost gather
        with compute.  interior(x, y) writes y over DoF layers [lo, hi) from
        elements [lo, hi-p+1) (own x only); boundary(x, y) ADDS elements
        [hi-p+1, hi) into DoF layers [hi-p+1, hi+p-1) (needs the ghosts).
        Both get views starting at their first DoF layer."""
        self.part = part
        self.rank = int(rank)
        self.layer = int(layer_size)
        self.compute = compute
        self.split = split
        self.group = group
        lo, hi = part.local_layers(self.rank)
        olo, ohi = part.own_layers(self.rank)
        self.n_local = (hi - lo) * self.layer
        self.n_own = (ohi - olo) * self.layer
        self.n_ghost = self.n_local - self.n_own
        self.x_local = torch.zeros(self.n_local, dtype=dtype, device=device)
        self.y_local = torch.zeros(self.n_local, dtype=dtype, device=device)
        self.halo_in = torch.zeros((part.p - 1) * self.layer, dtype=dtype, device=device)

    def _staged(self):
        """Device tensors over a CPU-only backend (gloo): the halo is staged
        through host buffers (the multi-process tests run the CUDA kernels of
        every rank on one GPU this way)."""
        if not self.x_local.is_cuda or not dist.is_initialized():
            return False
        return dist.get_backend(self.group) == "gloo"

    def _start(self, send, recv):
        ops = []
        back = []
        staged = bool(send or recv) and self._staged()
        for buf, peer in send:
            ops.append(dist.P2POp(dist.isend, buf.cpu() if staged else buf, peer, group=self.group))
        for buf, peer in recv:
            tgt = torch.empty(buf.shape, dtype=buf.dtype) if staged else buf
            if staged:
                back.append((tgt, buf))
            ops.append(dist.P2POp(dist.irecv, tgt, peer, group=self.group))
        reqs = dist.batch_isend_irecv(ops) if ops else []
        return _Pending(reqs, back)

    def _exchange(self, send, recv):
        self._start(send, recv).wait()

    def apply(self, x_own, y_own=None):
        """y_own = (A x) restricted to this rank's own DoF layers."""
        r, W, g = self.rank, self.part.world, (self.part.p - 1) * self.layer
        layers_copy(self.x_local[: self.n_own], x_own)
        # 1. ghost gather: my first p-1 own layers go to r-1; r+1's come to me.
        send, recv = [], []
        if r > 0 and g:
            send.append((self.x_local[:g].clone() if self.x_local.device.type == "cpu" else self.x_local[:g], r - 1))
        if r < W - 1 and g:
            recv.append((self.x_local[self.n_own:], r + 1))
        lo, hi = self.part.elements(r)
        p = self.part.p
        if self.split is not None and r < W - 1 and hi - lo > p - 1:
            # 2a. interior elements while the ghosts are in flight
            pending = self._start(send, recv)
            interior, boundary = self.split
            interior(self.x_local[: self.n_own], self.y_local[: self.n_own])
            pending.wait()
            # 2b. the last p-1 elements need the ghost layers
            b0 = (hi - lo - p + 1) * self.layer
            self.y_local[self.n_own:].zero_()
            boundary(self.x_local[b0:], self.y_local[b0:])
        else:
            self._exchange(send, recv)
            # 2. local apply on the slab
            self.compute(self.x_local, self.y_local)
        # 3. ghost reduce: my trailing p-1 partial layers go to r+1.
        send, recv = [], []
        if r < W - 1 and g:
            send.append((self.y_local[self.n_own:], r + 1))
        if r > 0 and g:
            recv.append((self.halo_in, r - 1))
        self._exchange(send, recv)
        out = self.y_local[: self.n_own]
        if r > 0 and g:
            layers_copy(out[:g], self.halo_in, add=True)
        if y_own is not None:
            return layers_copy(y_own, out)
        return out


class _Pending:
    """Outstanding p2p requests; host-staged receives are copied to their
    device buffers once complete."""

    def __init__(self, reqs, back):
        self.reqs = reqs
        self.back = back

    def wait(self):
        for req in self.reqs:
            req.wait()
        for host, dev in self.back:
            dev.copy_(host)


class NcclComm:
    """An NCCL communicator of the library (igs_nccl_comm_init) over the ranks
    of a torch.distributed group: rank 0 draws the unique id, the group
    broadcasts it.  world = 1 needs no torch.distributed."""

    def __init__(self, rank, world, group=None):
        import ctypes

        from . import _lib

        self._lib = _lib
        lib = _lib.load()
        uid = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _lib.check(lib.igs_nccl_unique_id(uid), "nccl_unique_id")
        if world > 1:
            t = torch.tensor(list(bytes(uid)), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0, group=group)
            uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        self.handle = ctypes.c_void_p()
        _lib.check(lib.igs_nccl_comm_init(uid, world, rank, ctypes.byref(self.handle)), "nccl_comm_init")
        self.rank, self.world = int(rank), int(world)

    def check(self, abort=True):
        """Raise RuntimeError (IGS_ENCCL) on an asynchronous communicator error."""
        self._lib.check(self._lib.load().igs_nccl_check(self.handle, int(bool(abort))), "nccl")

    def close(self):
        if self.handle:
            self._lib.check(self._lib.load().igs_nccl_comm_destroy(self.handle), "nccl_comm_destroy")
            self.handle = None


class NcclSlabApply:
    """One rank's slab apply through the C-ABI's NCCL data plane
    (igs_apply_sharded): ghost gather overlapped with the interior elements
    on a communication stream, the boundary elements after it, the ghost
    reduce into the next rank.  `op` is the MatrixFreeOperator of the rank's
    slab problem (coefficients of elements part.elements(rank))."""

    def __init__(self, op, part, rank, comm=None, overlap=True, split_boundary=False):
        import ctypes

        from . import _lib

        self._lib = _lib
        self.op = op
        self.part = part
        self.rank = int(rank)
        self.comm = comm
        if part.world > 1 and comm is None:
            raise ValueError("more than one rank needs an NcclComm")
        lib = _lib.load()
        self.prob, self._keep = op.struct()
        self.flags = (op.flags & _lib.FLAG_FORCE_GENERIC) | (_lib.FLAG_SPLIT_BOUNDARY if split_boundary else 0)
        nbytes = lib.igs_apply_sharded_workspace(ctypes.byref(self.prob), self.rank, part.world, self.flags)
        if nbytes == 0:
            _lib.check(_lib.IGS_EARG, "apply_sharded_workspace")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        self.comm_stream = torch.cuda.Stream() if overlap else None

    def apply(self, x_own, y_own):
        import ctypes

        lib = self._lib.load()
        cs = ctypes.c_void_p(self.comm_stream.cuda_stream) if self.comm_stream is not None else None
        handle = self.comm.handle if self.comm is not None else None
        st = lib.igs_apply_sharded(ctypes.byref(self.prob), self._lib.ptr(self.op.problem.coeff_field().planes),
                                   self._lib.ptr(x_own), self._lib.ptr(y_own), self._lib.ptr(self.ws),
                                   self.ws.numel(), handle, self.rank, self.part.world, self.flags,
                                   self._lib.stream_handle(), cs)
        self._lib.check(st, "apply_sharded")
        return y_own


class SlabAssembly:
    """One rank's row block of a slab-partitioned assembly (no collective).

    Rows are split by DoF layers of the last direction: rank r owns layers
    own_layers(r) of `part` (the last rank also the trailing p-1 layers);
    the coefficient planes it needs are those of elements halo_elements(r).
    """

    def __init__(self, part, rank):
        self.part = part
        self.rank = int(rank)

    def own_layers(self):
        return self.part.own_layers(self.rank)

    def halo_elements(self):
        """Elements whose coefficients the rank's rows need.  The rows of
        DoF layers [a, b) sum elements [a - p + 1, b); the one-pass symmetric
        kernel (csrc/asm3_sym.cuh) also forms the rows within p - 1 layers of
        the block, whose mirrored entries land in it, so it reads elements
        [a - 2(p - 1), b + p - 1) (clamped to the mesh)."""
        a, b = self.own_layers()
        p, K = self.part.p, self.part.K
        return max(0, a - 2 * (p - 1)), min(K, b + p - 1)

    def row_range(self, layer_rows):
        a, b = self.own_layers()
        return a * layer_rows, b * layer_rows

    def assemble(self, problem):
        """Values and CSR slice (indptr relative to the slice, indices) of the
        rank's rows.  `problem` holds the full-grid spaces and a coefficient
        field on the slab halo_elements() (or on the whole grid)."""
        from .sumfac import _run_assembly

        pat = problem.pattern()
        layer_rows = pat.shape[0] // problem.test[-1].num_basis
        lo, hi = self.row_range(layer_rows)
        vals = _run_assembly(problem, None, None, None, 0, (lo, hi))
        bounds = pat.indptr_dev[[lo, hi]].tolist()
        a, b = int(bounds[0]), int(bounds[1])
        indptr = pat.indptr_dev[lo: hi + 1] - a
        return vals[: b - a], indptr, pat.indices_dev[a:b]
