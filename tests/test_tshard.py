"""Time-sharded SA on world_size 2 and 3 gloo ranks (CPU): the halo exchange of
paper_2302_13451_b200.tshard reproduces the unsharded rows exactly.  The attention
compute is injected (CPU oracle forward; a dense fp64 backward that uses the given
LSE and O, as the CUDA kernels do) - this checks the host-side partition and
exchange logic; the GPU variant is in test_gpu_tshard.py."""
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


def oracle_fwd(q, k, v, L, R):
    o, lse = osa.sa_forward(q.numpy(), k.numpy(), v.numpy(), L, R)
    return torch.from_numpy(o), torch.from_numpy(lse)


def lse_bwd(q, k, v, o, lse, do, L, R):
    """Backward from the given LSE and O (P = exp(z - LSE), delta = dO . O) - dense, fp64."""
    T, D = q.shape[-2:]
    s = 1.0 / D ** 0.5
    i = torch.arange(T)
    mask = (i[None, :] >= i[:, None] - L) & (i[None, :] <= i[:, None] + R)
    z = (q @ k.transpose(-1, -2)) * s
    p = torch.where(mask, torch.exp(z - lse[..., None]), torch.zeros((), dtype=q.dtype))
    delta = (do * o).sum(-1, keepdim=True)
    ds = p * (do @ v.transpose(-1, -2) - delta)
    return ds @ k * s, ds.transpose(-1, -2) @ q * s, p.transpose(-1, -2) @ do


def _worker(rank, world, port, T, L, R, align, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_13451_b200 import tshard
    shape = (2, 2, T, 4)
    q, k, v = (torch.from_numpy(x) for x in synth.qkv(7, shape, "f32"))
    do = torch.from_numpy(synth.grad_out(7, shape, "f32"))
    t0, t1 = tshard.shard_bounds(T, world, rank, align)
    loc = lambda x: x[..., t0:t1, :].contiguous()  # noqa: E731
    o, lse = tshard.sa_forward_tsharded(loc(q), loc(k), loc(v), L, R, align=align, attn_fwd=oracle_fwd)
    g = tshard.sa_backward_tsharded(loc(q), loc(k), loc(v), o, lse, loc(do), L, R, align=align, attn_bwd=lse_bwd)
    O, LSE = osa.sa_forward(q.numpy(), k.numpy(), v.numpy(), L, R)
    G = osa.sa_backward(q.numpy(), k.numpy(), v.numpy(), do.numpy(), L, R)
    errs = [float(np.abs(o.numpy() - O[..., t0:t1, :]).max()), float(np.abs(lse.numpy() - LSE[..., t0:t1]).max())]
    errs += [float(np.abs(a.numpy() - b[..., t0:t1, :]).max()) for a, b in zip(g, G)]
    out[rank] = max(errs)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T,L,R,align", [(2, 40, 3, 2, 1), (2, 64, 5, 0, 8), (3, 50, 2, 6, 1), (3, 96, 4, 4, 16),
                                                (2, 33, 0, 0, 1)])
def test_time_sharded_equals_unsharded(world, T, L, R, align):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), T, L, R, align, out), nprocs=world, join=True)
    assert sorted(out.keys()) == list(range(world))
    assert max(out.values()) < 1e-12, dict(out)


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
