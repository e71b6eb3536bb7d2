"""Time sharding on world_size 2 and 3 gloo ranks (CPU): shard bounds, and the deep-halo
stack (NEXT-4) whose single exchange (paper_2302_13451_b200.tshard.exchange_halo) reproduces
the unsharded stack rows exactly with the CPU oracle stack injected as the compute.  The
per-layer time-sharded C path is covered by test_dist_host.py (host logic) and
test_gpu_tshard.py (the CUDA kernels under a real multi-process group)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import sa as osa


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_cover_and_align():
    from paper_2302_13451_b200 import tshard
    for T, world, align in ((1750, 8, 128), (180000, 8, 128), (37, 3, 1), (100, 4, 16)):
        b = [tshard.shard_bounds(T, world, r, align) for r in range(world)]
        assert b[0][0] == 0 and b[-1][1] == T
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        assert all(t0 % align == 0 for t0, _ in b)


def _stack_worker(rank, world, port, T, L, R, n, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_13451_b200 import tshard
    from oracle import stack as ostack
    mname = "llsa" if mode == 1 else "sa"
    x = synth.normal(8, "X", (1, 2, T, 4))
    dy = synth.normal(9, "dY", ((R + 1,) if mode == 1 else ()) + (1, 2, T, 4))
    fwd = lambda xe, L_, R_, n_, m_: torch.from_numpy(ostack.stack_forward(xe.numpy(), L_, R_, n_, mname)[0])  # noqa
    bwd = lambda xe, dye, L_, R_, n_, m_: torch.from_numpy(  # noqa: E731
        ostack.stack_backward(xe.numpy(), dye.numpy(), L_, R_, n_, mname))
    t0, t1 = tshard.shard_bounds(T, world, rank, 1)
    xl = torch.from_numpy(x[..., t0:t1, :].copy())
    dyl = torch.from_numpy(dy[..., t0:t1, :].copy())
    y = tshard.stack_forward_tsharded(xl, L, R, n, mode, align=1, stack_fwd=fwd)
    dx = tshard.stack_backward_tsharded(xl, dyl, L, R, n, mode, align=1, stack_bwd=bwd)
    # the smallest shard known from the partition: no agreeing all-reduce, the same halos
    min_T = min(b - a for a, b in (tshard.shard_bounds(T, world, r, 1) for r in range(world)))
    y2 = tshard.stack_forward_tsharded(xl, L, R, n, mode, align=1, stack_fwd=fwd, min_T=min_T)
    dx2 = tshard.stack_backward_tsharded(xl, dyl, L, R, n, mode, align=1, stack_bwd=bwd, min_T=min_T)
    assert torch.equal(y, y2) and torch.equal(dx, dx2)
    Y = ostack.stack_forward(x, L, R, n, mname)[0]
    DX = ostack.stack_backward(x, dy, L, R, n, mname)
    out[rank] = max(float(np.abs(y.numpy() - Y[..., t0:t1, :]).max()),
                    float(np.abs(dx.numpy() - DX[..., t0:t1, :]).max()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T,L,R,n,mode", [(2, 60, 3, 1, 2, 0), (3, 90, 2, 2, 3, 0), (2, 64, 3, 2, 2, 1),
                                                 (3, 96, 2, 1, 2, 1)])
def test_deep_halo_stack_equals_unsharded(world, T, L, R, n, mode):
    # NEXT-4: the n-layer stack (SA and LLSA) on time shards with one deep-halo exchange per
    # stack reproduces the unsharded stack rows, forward and backward (CPU oracle stack injected)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_stack_worker, args=(world, _free_port(), T, L, R, n, mode, out), nprocs=world, join=True)
    assert sorted(out.keys()) == list(range(world))
    assert max(out.values()) < 1e-12, dict(out)
