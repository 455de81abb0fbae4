"""The C-ABI multi-GPU data plane (igs_apply_sharded, NCCL) and the
host-staged multi-process apply.

Only one GPU is available to this build, so:
  * igs_apply_sharded runs at world size 1 (with and without an NCCL
    communicator, with the interior / boundary split forced) and must equal
    the plain apply bit for bit;
  * two processes share cuda:0 with a gloo group: every rank runs the real
    CUDA slab kernels and the halo is staged through host buffers (exactly
    the ShardedApply code the NCCL group runs); the gathered y equals the
    single-process apply;
  * NCCL failures map to IGS_ENCCL -> RuntimeError, argument errors to
    ValueError (CPU).
"""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_errors_map_to_exceptions():
    from paper_1809_05471_b200 import _lib

    lib = _lib.load()
    uid = (ctypes.c_uint8 * 128)()
    h = ctypes.c_void_p()
    with pytest.raises(ValueError):
        _lib.check(lib.igs_nccl_comm_init(uid, 0, 0, ctypes.byref(h)), "init")
    with pytest.raises(ValueError):
        _lib.check(lib.igs_apply_sharded(None, None, None, None, None, 0, None, 0, 2, 0, None, None), "x")
    if not torch.cuda.is_available():
        # no device: NCCL itself fails -> IGS_ENCCL -> RuntimeError
        st = lib.igs_nccl_comm_init(uid, 1, 0, ctypes.byref(h))
        assert st == _lib.IGS_ENCCL
        with pytest.raises(RuntimeError):
            _lib.check(st, "nccl_comm_init")


def _slab_op(d, p, K, kind, part, rank, seed=3):
    from paper_1809_05471_b200 import matfree, workloads
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    bases, quad = workloads.spaces(d, p, K)
    lo, hi = part.elements(rank)
    planes = workloads.synthetic_planes(d, list(quad.shape), kind, seed=seed, z_range=(lo * p, hi * p))
    field = workloads.field_from_planes(d, kind, planes, quad.shape, slab=(lo, hi))
    return matfree.MatrixFreeOperator(AssemblyProblem(bases, bases, quad, field))


@pytest.mark.gpu
@pytest.mark.parametrize("p,K,kind", [(6, 8, 2), (4, 7, 3)])
def test_apply_sharded_capi_world1_equals_apply(cuda, p, K, kind):
    from paper_1809_05471_b200 import workloads
    from paper_1809_05471_b200.sharded import NcclComm, NcclSlabApply, SlabPartition

    d = 3
    full = workloads.make_problem(d, p, K, kind, seed=3)
    from paper_1809_05471_b200 import matfree

    op_full = matfree.MatrixFreeOperator(full)
    n = full.shape[1]
    x = torch.randn(n, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(4))
    y_ref = op_full.apply_device(x)
    part = SlabPartition(K, p, 1)
    op = _slab_op(d, p, K, kind, part, 0)
    comm = NcclComm(0, 1)
    try:
        for c in (None, comm):
            for split in (False, True):
                for overlap in (False, True):
                    sa = NcclSlabApply(op, part, 0, comm=c, overlap=overlap, split_boundary=split)
                    y = torch.empty_like(x)
                    sa.apply(x, y)
                    torch.cuda.synchronize()
                    err = float(torch.linalg.vector_norm(y - y_ref) / torch.linalg.vector_norm(y_ref))
                    assert err <= 1e-12, (c is not None, split, overlap, err)
        comm.check()
    finally:
        comm.close()


def _worker(rank, world, port, p, K, kind, split, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    from paper_1809_05471_b200 import matfree, workloads
    from paper_1809_05471_b200.sharded import ShardedApply, SlabPartition
    from paper_1809_05471_b200.sumfac import AssemblyProblem

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d = 3
    part = SlabPartition(K, p, world)
    op = _slab_op(d, p, K, kind, part, rank)
    bases, quad = workloads.spaces(d, p, K)
    N = int(np.prod([b.num_basis for b in bases]))
    layer = N // (K + p - 1)
    x_full = torch.randn(N, dtype=torch.float64, generator=torch.Generator().manual_seed(9)).cuda()
    olo, ohi = part.own_layers(rank)
    lo, hi = part.elements(rank)
    splitf = None
    if split and rank < world - 1 and hi - lo > p - 1:
        cut = hi - p + 1
        layer_pts = quad.num_points // quad.shape[-1]
        planes = op.problem.coeff_field().planes
        npc = (cut - lo) * p * layer_pts
        kind_ = kind
        op_i = matfree.MatrixFreeOperator(AssemblyProblem(bases, bases, quad, workloads.field_from_planes(
            d, kind_, planes[:, :npc], quad.shape, slab=(lo, cut))))
        op_b = matfree.MatrixFreeOperator(AssemblyProblem(bases, bases, quad, workloads.field_from_planes(
            d, kind_, planes[:, npc:], quad.shape, slab=(cut, hi))))
        splitf = (lambda xv, yv: op_i.apply_device(xv, yv), lambda xv, yv: op_b.apply_device(xv, yv, accumulate=True))
    sa = ShardedApply(part, rank, layer, lambda xl, yl: op.apply_device(xl, yl), "cuda", split=splitf)
    y_own = sa.apply(x_full[olo * layer: ohi * layer].contiguous())
    parts = [None] * world
    dist.all_gather_object(parts, y_own.cpu().numpy())
    if rank == 0:
        np.save(out, np.concatenate(parts))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world,split", [(2, False), (2, True), (3, True)])
def test_host_staged_multiprocess_apply_runs_cuda_kernels(cuda, tmp_path, world, split):
    import torch.multiprocessing as mp

    from paper_1809_05471_b200 import matfree, workloads

    p, K, kind = 4, 9, 3
    out = str(tmp_path / "y.npy")
    mp.spawn(_worker, args=(world, _free_port(), p, K, kind, split, out), nprocs=world, join=True)
    full = workloads.make_problem(3, p, K, kind, seed=3)
    N = full.shape[1]
    x = torch.randn(N, dtype=torch.float64, generator=torch.Generator().manual_seed(9)).cuda()
    y_ref = matfree.MatrixFreeOperator(full).apply_device(x).cpu().numpy()
    y = np.load(out)
    assert np.linalg.norm(y - y_ref) <= 1e-12 * np.linalg.norm(y_ref)
