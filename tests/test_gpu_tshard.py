"""Time sharding on the GPU kernels.

1. The library's time-sharded C path (sa_forward_tsharded / sa_backward_tsharded) under a REAL
   multi-process group: 2 and 3 processes share the one leased GPU (NCCL refuses two ranks on one
   device, so the halo moves through the library's callback transport, host-staged over gloo;
   pack / unpack kernels, the interior / edge tile split and the kernels are the production
   path).  Every rank's local rows must be BITWISE equal to the unsharded call on per-head tiles
   (one head per call; shards 128-frame aligned) and match the fp64 oracle on slabs straddling each shard boundary.
2. NCCL transport initialisation (world 1: a communicator of one rank, no neighbours).
3. Virtual ranks on one device: the CUDA path on hand-cut halo slabs == unsharded (bitwise, one
   head per call on both sides: see _per_head).
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _per_head(fn, *xs):
    """fn on each (batch, head) plane separately, outputs concatenated back to [B][H]: every call
    has one head, so the SA kernels tile each head from frame 0 in 128-frame tiles, as a time shard
    does; a multi-head call packs its tiles over the flattened B*H*T axis and rounds in another
    order (equal to the gate, not bitwise)"""
    B, H = xs[0].shape[:2]
    outs = [[fn(*(x[b:b + 1, h:h + 1].clone() for x in xs)) for h in range(H)] for b in range(B)]
    return tuple(torch.cat([torch.cat([o_[i] for o_ in row], dim=1) for row in outs], dim=0)
                 for i in range(len(outs[0][0])))


def _worker(rank, world, port, T, L, R, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import dist as sd
    from paper_2302_13451_b200 import tshard
    import oracle
    from gates import excess
    B, H, D = 1, 3, 64
    g = torch.Generator(device="cuda").manual_seed(21)
    q, k, v, do = (torch.randn(B, H, T, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    # unsharded reference one head per call (_per_head)
    per_head = _per_head
    o, lse = per_head(lambda q_, k_, v_: s.sa_forward(q_, k_, v_, L, R), q, k, v)
    dq, dk, dv = per_head(lambda q_, k_, v_, o_, l_, d_: s.sa_backward(q_, k_, v_, o_, l_, d_, L, R),
                          q, k, v, o, lse, do)
    t0, t1 = tshard.shard_bounds(T, world, rank, 128)
    n = t1 - t0
    d = sd.Dist()
    assert d.transport == "host"
    qm, km, vm, dom = (sd.margined(B, H, n, D) for _ in range(4))
    for m, x in ((qm, q), (km, k), (vm, v), (dom, do)):
        sd.local(m, n).copy_(x[:, :, t0:t1])
    om, lsem = sd.sa_forward_tsharded(qm, km, vm, L, R, t0, T, d)
    gm = sd.sa_backward_tsharded(qm, km, vm, lsem, dom, L, R, t0, T, d)
    res = {}
    res["bitwise_fwd"] = bool(torch.equal(sd.local(om, n), o[:, :, t0:t1]) and
                              torch.equal(sd.local(lsem, n), lse[:, :, t0:t1]))
    res["bitwise_bwd"] = all(bool(torch.equal(sd.local(a, n), b[:, :, t0:t1])) for a, b in zip(gm, (dq, dk, dv)))
    # the stored-band mode on the same shards (W <= 49): bitwise equal to the unsharded calls too
    if L + R + 1 <= 49:
        o_p, lse_p, p_p = per_head(lambda q_, k_, v_: s.sa_forward_p(q_, k_, v_, L, R), q, k, v)
        g_p = per_head(lambda q_, k_, v_, o_, p_, d_: s.sa_backward_p(q_, k_, v_, o_, p_, d_, L, R),
                       q, k, v, o_p, p_p, do)
        dom2 = sd.margined(B, H, n, D)
        sd.local(dom2, n).copy_(do[:, :, t0:t1])
        om2, lsem2, pm2 = sd.sa_forward_p_tsharded(qm, km, vm, L, R, t0, T, d)
        gm2 = sd.sa_backward_p_tsharded(qm, km, vm, pm2, dom2, L, R, t0, T, d)
        res["bitwise_band"] = bool(torch.equal(sd.local(om2, n), o_p[:, :, t0:t1]) and
                                   torch.equal(sd.local(pm2, n), p_p[:, :, t0:t1]) and
                                   all(torch.equal(sd.local(a, n), b[:, :, t0:t1]) for a, b in zip(gm2, g_p)))
    else:
        res["bitwise_band"] = True
    # oracle on a slab around each boundary of this shard: rows whose whole dependency cone
    # (forward +-(L+R), backward +-2(L+R)) lies in the slab
    worst = 0.0
    for c in (t0, t1):
        if c in (0, T):
            continue
        a0, a1 = max(0, c - 200), min(T, c + 200)
        sl = lambda x: x[0, :, a0:a1].double().cpu().numpy()  # noqa: E731
        O, LSE = oracle.sa.sa_forward(sl(q), sl(k), sl(v), L, R)
        G = oracle.sa.sa_backward(sl(q), sl(k), sl(v), sl(do), L, R)
        lo, hi = max(t0, c - 48), min(t1, c + 48)
        if lo >= hi:
            continue
        r = slice(lo - a0, hi - a0)
        loc = lambda m: m[0, :, 128 + lo - t0:128 + hi - t0].double().cpu().numpy()  # noqa: E731
        for name, got, ref in (("O", loc(om), O[:, r]), ("dQ", loc(gm[0]), G[0][:, r]),
                               ("dK", loc(gm[1]), G[1][:, r]), ("dV", loc(gm[2]), G[2][:, r])):
            worst = max(worst, excess(got, ref, "bf16", f"tshard-w{world}-r{rank}-{name}"))
    res["oracle_excess"] = worst
    res["launches"] = s.launch_count()
    out[rank] = res
    d.close()
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("world,T,L,R", [(2, 1000, 32, 8), (3, 1400, 32, 16), (3, 900, 3, 1), (2, 700, 32, 32)])
def test_tsharded_c_path_multiprocess(world, T, L, R):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), T, L, R, out), nprocs=world, join=True)
    assert sorted(out.keys()) == list(range(world))
    for r in range(world):
        res = out[r]
        assert res["bitwise_fwd"] and res["bitwise_bwd"] and res["bitwise_band"], (r, res)
        assert res["oracle_excess"] <= 0, (r, res)


def _llsa_worker(rank, world, port, T, L, R, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as tdist
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import dist as sd
    from paper_2302_13451_b200 import tshard
    import oracle
    from gates import excess
    B, H, D, C = 1, 2, 64, R + 1
    g = torch.Generator(device="cuda").manual_seed(31)
    q, k, v, do = (torch.randn(C, B, H, T, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    o, lse = s.llsa_forward(q, k, v, L, R)
    dq, dk, dv = s.llsa_backward(q, k, v, o, lse, do, L, R)
    t0, t1 = tshard.shard_bounds(T, world, rank, 1)
    n = t1 - t0
    hl, hr = sd.llsa_slab_rows(n, L, R, t0, T)
    d = sd.Dist()
    assert d.transport == "host"
    slab = lambda: torch.zeros(C, B, H, hl + n + hr, D, dtype=torch.bfloat16, device="cuda")  # noqa: E731
    qs, ks, vs, dos = slab(), slab(), slab(), slab()
    for m, x in ((qs, q), (ks, k), (vs, v), (dos, do)):
        m[:, :, :, hl:hl + n].copy_(x[:, :, :, t0:t1])
    os_, lses = sd.llsa_forward_tsharded(qs, ks, vs, n, L, R, t0, T, d)
    gs = sd.llsa_backward_tsharded(qs, ks, vs, os_, lses, dos, n, L, R, t0, T, d)
    loc = lambda m: m[..., hl:hl + n, :] if m.dim() == 5 else m[..., hl:hl + n]  # noqa: E731
    res = {}
    # against the unsharded GPU call (same kernels, different item tiling: the bf16 gate)
    res["vs_unsharded"] = max(
        excess(loc(a).double().cpu().numpy(), b[..., t0:t1, :].double().cpu().numpy(), "bf16", f"llsa-tshard-{nm}")
        for nm, a, b in (("O", os_, o), ("dQ", gs[0], dq), ("dK", gs[1], dk), ("dV", gs[2], dv)))
    res["lse_vs_unsharded"] = float((loc(lses) - lse[..., t0:t1]).abs().max())
    # against the fp64 oracle on a window around each inner boundary: rows whose dependency cones
    # (forward [t-R-L, t+R], backward +-(L+2R)) lie inside the window
    worst = 0.0
    for c in (t0, t1):
        if c in (0, T):
            continue
        a0, a1 = max(0, c - 200), min(T, c + 200)
        sl = lambda x: x[:, 0, :, a0:a1].double().cpu().numpy()  # noqa: E731
        O, _ = oracle.llsa.llsa_forward(sl(q), sl(k), sl(v), L, R)
        G = oracle.llsa.llsa_backward(sl(q), sl(k), sl(v), sl(do), L, R)
        lo, hi = max(t0, c - 48), min(t1, c + 48)
        if lo >= hi:
            continue
        r = slice(lo - a0, hi - a0)
        pick = lambda m: m[:, 0, :, hl + lo - t0:hl + hi - t0].double().cpu().numpy()  # noqa: E731
        for nm, got, ref in (("O", pick(os_), O[:, :, r]), ("dQ", pick(gs[0]), G[0][:, :, r]),
                             ("dK", pick(gs[1]), G[1][:, :, r]), ("dV", pick(gs[2]), G[2][:, :, r])):
            worst = max(worst, excess(got, ref, "bf16", f"llsa-tshard-w{world}-r{rank}-{nm}"))
    res["oracle_excess"] = worst
    out[rank] = res
    d.close()
    tdist.barrier()
    tdist.destroy_process_group()


@pytest.mark.parametrize("world,T,L,R", [(2, 900, 32, 8), (3, 700, 3, 1), (2, 800, 32, 16)])
def test_llsa_tsharded_c_path_multiprocess(world, T, L, R):
    # time-sharded LLSA through the C ABI with the halo exchange live between real
    # processes (callback transport over gloo: the processes share the one GPU): local rows against
    # the unsharded LLSA call and against the fp64 oracle at every shard boundary
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_llsa_worker, args=(world, _free_port(), T, L, R, out), nprocs=world, join=True)
    assert sorted(out.keys()) == list(range(world))
    for r in range(world):
        res = out[r]
        assert res["vs_unsharded"] <= 0 and res["lse_vs_unsharded"] <= 1e-3, (r, res)
        assert res["oracle_excess"] <= 0, (r, res)


def test_llsa_tsharded_nccl_world1_equals_unsharded():
    # world 1 over the NCCL transport: no neighbours, the slab is the whole stream: bitwise equal
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import dist as sd
    C, B, H, T, D, L, R = 9, 1, 2, 600, 64, 32, 8
    g = torch.Generator(device="cuda").manual_seed(6)
    q, k, v, do = (torch.randn(C, B, H, T, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    o, lse = s.llsa_forward(q, k, v, L, R)
    dq, dk, dv = s.llsa_backward(q, k, v, o, lse, do, L, R)
    d = sd.Dist(transport="nccl")
    os_, lses = sd.llsa_forward_tsharded(q.clone(), k.clone(), v.clone(), T, L, R, 0, T, d)
    gs = sd.llsa_backward_tsharded(q, k, v, os_, lses, do.clone(), T, L, R, 0, T, d)
    assert torch.equal(os_, o) and torch.equal(lses, lse)
    for a, b in zip(gs, (dq, dk, dv)):
        assert torch.equal(a, b)
    d.close()


def test_tsharded_nccl_world1_equals_unsharded():
    # the NCCL transport's handle at world 1 (no neighbours, no exchange): the slab is the whole
    # stream and the result must be the unsharded call's, bitwise
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import dist as sd
    B, H, T, D, L, R = 2, 3, 777, 64, 32, 8
    g = torch.Generator(device="cuda").manual_seed(5)
    q, k, v, do = (torch.randn(B, H, T, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    o, lse = _per_head(lambda q_, k_, v_: s.sa_forward(q_, k_, v_, L, R), q, k, v)
    dq, dk, dv = _per_head(lambda q_, k_, v_, o_, l_, d_: s.sa_backward(q_, k_, v_, o_, l_, d_, L, R),
                           q, k, v, o, lse, do)
    d = sd.Dist(transport="nccl")
    qm, km, vm, dom = (sd.margined(B, H, T, D) for _ in range(4))
    for m, x in ((qm, q), (km, k), (vm, v), (dom, do)):
        sd.local(m, T).copy_(x)
    om, lsem = sd.sa_forward_tsharded(qm, km, vm, L, R, 0, T, d)
    gm = sd.sa_backward_tsharded(qm, km, vm, lsem, dom, L, R, 0, T, d)
    assert torch.equal(sd.local(om, T), o) and torch.equal(sd.local(lsem, T), lse)
    for a, b in zip(gm, (dq, dk, dv)):
        assert torch.equal(sd.local(a, T), b)
    d.close()


def _round_up(x, a):
    return -(-x // a) * a


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("L,R", [(32, 8), (32, 16), (3, 1)])
def test_virtual_rank_slabs_bitwise_equal_unsharded(world, L, R):
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import tshard
    B, H, T, D = 1, 3, 3000, 64
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v, do = (torch.randn(B, H, T, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    fwd = lambda q_, k_, v_: s.sa_forward(q_, k_, v_, L, R)  # noqa: E731
    bwd = lambda q_, k_, v_, o_, l_, d_: s.sa_backward(q_, k_, v_, o_, l_, d_, L, R)  # noqa: E731
    o, lse = _per_head(fwd, q, k, v)
    dq, dk, dv = _per_head(bwd, q, k, v, o, lse, do)
    for r in range(world):
        t0, t1 = tshard.shard_bounds(T, world, r, 128)
        hl, hr = _round_up(L, 128), _round_up(R, 128)
        a0, a1 = max(0, t0 - hl), min(T, t1 + hr)
        sl = lambda x: x[:, :, a0:a1].contiguous()  # noqa: E731
        o_r, lse_r = _per_head(fwd, sl(q), sl(k), sl(v))
        n = t1 - t0
        assert torch.equal(o_r[:, :, t0 - a0:t0 - a0 + n], o[:, :, t0:t1])
        assert torch.equal(lse_r[:, :, t0 - a0:t0 - a0 + n], lse[:, :, t0:t1])
        h = _round_up(L + R, 128)
        b0, b1 = max(0, t0 - h), min(T, t1 + h)
        sb = lambda x: x[:, :, b0:b1].contiguous()  # noqa: E731
        gq, gk, gv = _per_head(bwd, sb(q), sb(k), sb(v), sb(o), sb(lse), sb(do))
        for got, ref in ((gq, dq), (gk, dk), (gv, dv)):
            assert torch.equal(got[:, :, t0 - b0:t0 - b0 + n], ref[:, :, t0:t1])


@pytest.mark.parametrize("mode", ["sa", "llsa"])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_deep_halo_stack_slabs_vs_oracle(mode, dt):
    # NEXT-4 deep halo: each virtual rank runs the whole n-layer stack (forward and backward) on its
    # shard extended by the deep halo exchange_halo assembles (forward n(L+R) back for LLSA / nL for
    # SA and nR ahead; backward 2n(L+R) both sides, 128-aligned) and keeps its local rows; those rows
    # are checked against the fp64 oracle stack of the whole stream (composite gate n x gate x mag,
    # reading G24) - not only against the unsharded GPU stack
    import oracle
    import synth
    from gates import excess
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import tshard
    B, H, T, D, L, R, n, world = 1, 2, 1100, 64, 32, 8, 3, 3
    m = s.MODE_SA if mode == "sa" else s.MODE_LLSA
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    x = synth.round_to(synth.normal(12, "X", (B, H, T, D)), dt)
    dyshape = ((R + 1,) if mode == "llsa" else ()) + (B, H, T, D)
    dy = synth.round_to(synth.normal(12, "dY", dyshape), dt)
    Y, _ = oracle.stack.stack_forward(x, L, R, n, mode)
    DX = oracle.stack.stack_backward(x, dy, L, R, n, mode)
    tx = torch.tensor(x, dtype=tdt, device="cuda")
    tdy = torch.tensor(dy, dtype=tdt, device="cuda")
    sy, sdx = n * max(1.0, float(np.abs(Y).max())), n * max(1.0, float(np.abs(DX).max()))
    for r in range(world):
        t0, t1 = tshard.shard_bounds(T, world, r, 128)
        back = n * (L + R) if mode == "llsa" else n * L
        a0, a1 = max(0, t0 - _round_up(back, 128)), min(T, t1 + _round_up(n * R, 128))
        y, _ = s.stack_forward(tx[:, :, a0:a1].contiguous(), L, R, n, m)
        got = y[..., t0 - a0:t1 - a0, :].double().cpu().numpy()
        assert excess(got, Y[..., t0:t1, :], dt, f"deephalo-{mode}-r{r}-Y", scale=sy) <= 0
        h = _round_up(2 * n * (L + R), 128)
        b0, b1 = max(0, t0 - h), min(T, t1 + h)
        xs = tx[:, :, b0:b1].contiguous()
        _, saved = s.stack_forward(xs, L, R, n, m)
        dx = s.stack_backward(xs, saved, tdy[..., b0:b1, :].contiguous(), L, R, n, m)
        got = dx[:, :, t0 - b0:t1 - b0].double().cpu().numpy()
        assert excess(got, DX[:, :, t0:t1], dt, f"deephalo-{mode}-r{r}-dX0", scale=sdx) <= 0
