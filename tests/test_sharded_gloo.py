"""Multi-rank slab partition of the apply (sharded.py) on CPU with gloo.

Each rank computes its slab with the CPU oracle (the GPU kernel's role on
the box) and exchanges the (p-1)-layer halos through torch.distributed;
the gathered result must equal the single-process apply exactly up to
summation order (≤ 1e-14)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import igs_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, d, p, K, kind, q, split=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1809_05471_b200.sharded import ShardedApply, SlabPartition

    sp = [O.uniform_space(p, K) for _ in range(d)]
    shape = [p * K] * d
    ths = O.first_order_set(d)
    pm = O.plane_map(d, kind)
    n = int(np.prod([s.num_basis for s in sp]))
    layer_n = n // (K + p - 1)
    x = O.recipe_x(n, seed=4)
    part = SlabPartition(K, p, world)
    lo, hi = part.elements(rank)
    layer_x = int(np.prod(shape[:-1]))
    planes = O.synthetic_planes(d, shape, lo * p, hi * p, kind, seed=9)

    def compute(xl, yl):
        # embed the local vector into a full-length x for the oracle's slab apply
        full = np.zeros(n)
        full[lo * layer_n: lo * layer_n + xl.numel()] = xl.numpy()
        yl.copy_(torch.from_numpy(O.apply_slab(sp, p, ths, ths, pm, planes, full, lo, hi)))

    def sub_apply(e0, e1, xv):
        full = np.zeros(n)
        full[e0 * layer_n: e0 * layer_n + xv.numel()] = xv.numpy()
        sub = planes[:, (e0 - lo) * p * layer_x: (e1 - lo) * p * layer_x]
        return torch.from_numpy(O.apply_slab(sp, p, ths, ths, pm, sub, full, e0, e1))

    def interior(xv, yv):
        yv.copy_(sub_apply(lo, hi - p + 1, xv))

    def boundary(xv, yv):
        yv += sub_apply(hi - p + 1, hi, xv)

    sa = ShardedApply(part, rank, layer_n, compute, "cpu", split=(interior, boundary) if split else None)
    olo, ohi = part.own_layers(rank)
    x_own = torch.from_numpy(x[olo * layer_n: ohi * layer_n].copy())
    y_own = sa.apply(x_own).clone()
    del layer_x
    gathered = [None] * world
    dist.all_gather_object(gathered, (olo, y_own.numpy()))
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,d,p,K,kind,split", [(2, 3, 4, 7, 3, False), (3, 3, 3, 9, 2, False),
                                                   (2, 2, 5, 8, 3, False), (3, 3, 3, 12, 3, True),
                                                   (2, 2, 5, 11, 2, True)])
def test_sharded_apply_matches_single_process(world, d, p, K, kind, split):
    """split=True: interior elements are computed while the ghost gather is in
    flight, the last p-1 elements after it lands (SURVEY §8(e) overlap)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, d, p, K, kind, q, split)) for r in range(world)]
    for pr in procs:
        pr.start()
    gathered = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    sp = [O.uniform_space(p, K) for _ in range(d)]
    shape = [p * K] * d
    n = int(np.prod([s.num_basis for s in sp]))
    x = O.recipe_x(n, seed=4)
    planes = O.synthetic_planes(d, shape, 0, shape[-1], kind, seed=9)
    ths = O.first_order_set(d)
    y_ref = O.apply(sp, p, ths, ths, O.plane_map(d, kind), planes, x)
    layer_n = n // (K + p - 1)
    y = np.concatenate([part for _, part in sorted(gathered, key=lambda t: t[0])])
    assert y.size == n
    assert np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref) <= 1e-14
    del layer_n


def _cg_worker(rank, world, port, d, p, K, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1809_05471_b200.sharded import ShardedApply, SlabPartition
    from paper_1809_05471_b200.solvers import cg

    sp = [O.uniform_space(p, K) for _ in range(d)]
    shape = [p * K] * d
    ths = O.first_order_set(d)
    pm = O.plane_map(d, kind)
    n = int(np.prod([s.num_basis for s in sp]))
    layer_n = n // (K + p - 1)
    part = SlabPartition(K, p, world)
    lo, hi = part.elements(rank)
    planes = O.synthetic_planes(d, shape, lo * p, hi * p, kind, seed=9)

    def compute(xl, yl):
        full = np.zeros(n)
        full[lo * layer_n: lo * layer_n + xl.numel()] = xl.numpy()
        yl.copy_(torch.from_numpy(O.apply_slab(sp, p, ths, ths, pm, planes, full, lo, hi)))

    sa = ShardedApply(part, rank, layer_n, compute, "cpu")
    olo, ohi = part.own_layers(rank)
    b = torch.from_numpy(O.recipe_x(n, seed=5)[olo * layer_n: ohi * layer_n].copy())
    x, it, res = cg(lambda v, out: out.copy_(sa.apply(v)), b, tol=1e-12, maxiter=1000, group=dist.group.WORLD)
    gathered = [None] * world
    dist.all_gather_object(gathered, (olo, x.numpy(), it, res))
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,d,p,K,kind", [(2, 2, 3, 8, 3), (3, 2, 4, 9, 3)])
def test_sharded_cg_matches_direct_solve(world, d, p, K, kind):
    """CG on the slab-partitioned apply, the inner products
    all-reduced over the group — the gathered solution equals the direct solve."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cg_worker, args=(r, world, port, d, p, K, kind, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    gathered = q.get(timeout=240)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    its = {g[2] for g in gathered}
    assert len(its) == 1  # every rank saw the same global residuals
    assert all(g[3] <= 1e-12 for g in gathered)
    sp = [O.uniform_space(p, K) for _ in range(d)]
    shape = [p * K] * d
    n = int(np.prod([s.num_basis for s in sp]))
    planes = O.synthetic_planes(d, shape, 0, shape[-1], kind, seed=9)
    ths = O.first_order_set(d)
    pm = O.plane_map(d, kind)
    A = np.stack([O.apply(sp, p, ths, ths, pm, planes, e) for e in np.eye(n)], axis=1)
    b = O.recipe_x(n, seed=5)
    x_ref = np.linalg.solve(A, b)
    x = np.concatenate([g[1] for g in sorted(gathered, key=lambda t: t[0])])
    assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-9
