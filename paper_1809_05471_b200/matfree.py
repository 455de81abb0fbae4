"""Matrix-free operator application (Alg. 2 with Alg. 3).

The reference package specifies but does not ship this module
(SPEC.md:440-483).  `apply(op, u)` computes
    v = Σ_eta Q_eta^T · w · Σ_theta F_{eta,theta} · Q_theta · u
on the GPU through igs_apply (K4): the fused sm_100a kernel for the
BASELINE shapes (3D, same order in every direction, per-element Gauss
rules), else the stage-by-stage kernels.  Host (numpy) vectors are copied
to the device and back; device tensors stay on the device.
"""

import ctypes

import numpy as np

from . import _lib
from .sumfac import FlopCounter
from .tensorspace import field_eval_count

__all__ = ("MatrixFreeOperator", "apply", "eval_field", "HostPipeline")


class MatrixFreeOperator:
    """A ready-to-apply operator: problem + device tables + workspace.

    `slab=(lo, hi)` restricts the operator to elements [lo, hi) of the last
    direction (the multi-GPU partition, see sharded.py); the coefficient
    planes then cover only that slab's points and vectors hold DoF layers
    [lo, hi + order - 1).
    """

    def __init__(self, problem, dir_order=None, slab=None, force_generic=False):
        self.problem = problem
        self.dir_order = None if dir_order is None else tuple(dir_order)
        if slab is None:
            slab = getattr(problem, "slab", None)
        self.slab = None if slab is None else (int(slab[0]), int(slab[1]))
        self.flags = _lib.FLAG_FORCE_GENERIC if force_generic else 0
        self._ws = None
        self._prob = None

    @property
    def shape(self):
        if self.slab is None:
            return self.problem.shape
        lo, hi = self.slab
        last_t = self.problem.trial[-1].order
        last_s = self.problem.test[-1].order
        m = n = 1
        for b in self.problem.test[:-1]:
            m *= b.num_basis
        for b in self.problem.trial[:-1]:
            n *= b.num_basis
        return m * (hi - lo + last_s - 1), n * (hi - lo + last_t - 1)

    def struct(self):
        if self._prob is None:
            self._prob = self.problem.struct(self.dir_order, slab=self.slab, with_pattern=False)
        return self._prob

    @property
    def fused(self):
        lib = _lib.load()
        prob, _ = self.struct()
        return bool(lib.igs_fused_path(ctypes.byref(prob), _lib.OP_APPLY)) and not self.flags

    def workspace(self):
        torch = _lib.require_cuda()
        lib = _lib.load()
        prob, _ = self.struct()
        nbytes = lib.igs_workspace_bytes(ctypes.byref(prob), _lib.OP_APPLY, self.flags)
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        return self._ws, nbytes

    def apply_device(self, x, y=None, accumulate=False, stream=None, kernel_only=False):
        """y (+)= A x for device tensors; returns y.  Enqueued on `stream`
        (default: torch's current stream); no host synchronisation.
        `kernel_only` (measurement) runs only the fused main kernel."""
        torch = _lib.require_cuda()
        lib = _lib.load()
        m, n = self.shape
        if x.numel() != n:
            raise ValueError(f"vector length {x.numel()} does not match the trial space ({n})")
        if y is None:
            y = torch.empty(m, dtype=torch.float64, device="cuda")
        prob, _ = self.struct()
        ws, nbytes = self.workspace()
        f = self.problem.coeff_field()
        flags = self.flags | (_lib.FLAG_ACCUMULATE if accumulate else 0) | (4 if kernel_only else 0)
        sh = ctypes.c_void_p(stream.cuda_stream) if stream is not None else _lib.stream_handle()
        st = lib.igs_apply(ctypes.byref(prob), _lib.ptr(f.planes), _lib.ptr(x), _lib.ptr(y), _lib.ptr(ws),
                           nbytes, flags, sh)
        _lib.check(st, "apply")
        return y

    def count(self, counter):
        """Reference-style MAC counts of one apply (see module docstring)."""
        p = self.problem
        orders_t = [b.order for b in p.trial]
        orders_s = [b.order for b in p.test]
        nt = [b.num_basis for b in p.trial]
        ns = [b.num_basis for b in p.test]
        npts = list(p.quad.shape)
        f = p.coeff_field()
        for j, th in enumerate(p.theta_set):
            if all(f.is_zero_block(i, j) for i in range(len(p.eta_set))):
                continue
            counter.add_field_eval(field_eval_count(orders_t, nt, npts))
        for i, et in enumerate(p.eta_set):
            if all(f.is_zero_block(i, j) for j in range(len(p.theta_set))):
                continue
            counter.add_block_update(field_eval_count(orders_s, ns, npts))


def apply(op, u, counter=None):
    """v = A u without forming A.

    numpy input -> numpy output (host copies included); a CUDA tensor stays
    on the device.
    """
    torch = _lib.require_cuda()
    host = not isinstance(u, torch.Tensor)
    if host:
        u_np = np.ascontiguousarray(u, dtype=float).reshape(-1)
        x = torch.from_numpy(u_np).to("cuda", non_blocking=False)
    else:
        x = u.to(device="cuda", dtype=torch.float64).reshape(-1).contiguous()
    y = op.apply_device(x)
    if counter is not None:
        op.count(counter)
    return y.cpu().numpy() if host else y


def eval_field(op, u, theta, counter=None):
    """∂^theta u at every quadrature point (Alg. 3).

    Returns a device tensor indexed [i_1, ..., i_d].
    """
    from .tensorspace import contract_to_points

    p = op.problem if isinstance(op, MatrixFreeOperator) else op
    return contract_to_points(p.trial_tables(), theta, u, counter)



class HostPipeline:
    """Applies to a sequence of pinned host vectors with the transfers
    overlapped (CUDA streams): the upload of vector i+1 and the download of
    result i-1 run on two copy streams while apply i runs on the compute
    stream; device buffers are double-buffered and ordered by events.

    `step(x_dev, y_dev)` enqueues one apply on the current stream (e.g.
    ``op.apply_device`` or a sharded step).  Every vector still crosses the
    bus each step; only the latency of the copies is hidden.
    """

    def __init__(self, step, n_in, n_out, device="cuda"):
        torch = _lib.require_cuda()
        self.step = step
        self.x = [torch.empty(n_in, dtype=torch.float64, device=device) for _ in range(2)]
        self.y = [torch.empty(n_out, dtype=torch.float64, device=device) for _ in range(2)]
        self.up = torch.cuda.Stream(device=device)
        self.down = torch.cuda.Stream(device=device)
        self.ev_up = [torch.cuda.Event() for _ in range(2)]
        self.ev_done = [torch.cuda.Event() for _ in range(2)]
        self.ev_down = [torch.cuda.Event() for _ in range(2)]
        self.ev_free = [torch.cuda.Event() for _ in range(2)]
        for e in self.ev_down + self.ev_free:
            e.record()

    def run(self, xs_host, ys_host):
        """ys_host[i] = A xs_host[i] for every i (pinned CPU tensors); returns
        when every download is enqueued (synchronise before reading)."""
        torch = _lib.require_cuda()
        comp = torch.cuda.current_stream()
        self.up.wait_stream(comp)  # nothing is uploaded before the call
        for i, (xh, yh) in enumerate(zip(xs_host, ys_host)):
            k = i & 1
            with torch.cuda.stream(self.up):
                self.up.wait_event(self.ev_free[k])   # apply i-2 done with x[k]
                self.x[k].copy_(xh, non_blocking=True)
                self.ev_up[k].record(self.up)
            comp.wait_event(self.ev_up[k])
            comp.wait_event(self.ev_down[k])          # download i-2 done with y[k]
            self.step(self.x[k], self.y[k])
            self.ev_done[k].record(comp)
            self.ev_free[k].record(comp)
            with torch.cuda.stream(self.down):
                self.down.wait_event(self.ev_done[k])
                yh.copy_(self.y[k], non_blocking=True)
                self.ev_down[k].record(self.down)
        comp.wait_stream(self.down)
        return ys_host


del FlopCounter
