"""Time sharding on the GPU kernels, emulated on one device (the gloo test covers the
exchange itself): every virtual rank runs the CUDA path on its halo-extended slab —
exactly the slab exchange_halo assembles — and its local rows must be BITWISE equal to
the unsharded call (shards and halos aligned to the 128-frame tile, deterministic kernels)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _round_up(x, a):
    return -(-x // a) * a


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("L,R", [(32, 8), (32, 16), (3, 1)])
def test_tsharded_bitwise_equals_unsharded(world, L, R):
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import tshard
    B, H, T, D = 1, 3, 3000, 64
    g = torch.Generator(device="cuda").manual_seed(11)
    q, k, v, do = (torch.randn(B, H, T, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
    o, lse = s.sa_forward(q, k, v, L, R)
    dq, dk, dv = s.sa_backward(q, k, v, o, lse, do, L, R)
    for r in range(world):
        t0, t1 = tshard.shard_bounds(T, world, r, 128)
        hl, hr = _round_up(L, 128), _round_up(R, 128)
        a0, a1 = max(0, t0 - hl), min(T, t1 + hr)
        sl = lambda x: x[:, :, a0:a1].contiguous()  # noqa: E731
        o_r, lse_r = s.sa_forward(sl(q), sl(k), sl(v), L, R)
        n = t1 - t0
        assert torch.equal(o_r[:, :, t0 - a0:t0 - a0 + n], o[:, :, t0:t1])
        assert torch.equal(lse_r[:, :, t0 - a0:t0 - a0 + n], lse[:, :, t0:t1])
        h = _round_up(max(L, R), 128)
        b0, b1 = max(0, t0 - h), min(T, t1 + h)
        sb = lambda x: x[:, :, b0:b1].contiguous()  # noqa: E731
        gq, gk, gv = s.sa_backward(sb(q), sb(k), sb(v), sb(o), sb(lse), sb(do), L, R)
        for got, ref in ((gq, dq), (gk, dk), (gv, dv)):
            assert torch.equal(got[:, :, t0 - b0:t0 - b0 + n], ref[:, :, t0:t1])


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("world", [2, 3])
def test_deep_halo_stack_bitwise_equals_unsharded(world, mode):
    # NEXT-4 deep halo on the GPU stack driver: each virtual rank runs the n-layer stack (SA or
    # LLSA, bf16) on the slab extended by the deep halo (rounded to the 128-frame tile) exactly
    # as stack_forward_tsharded / stack_backward_tsharded assemble it; its rows must be BITWISE
    # the unsharded stack's
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import tshard
    B, H, T, D, L, R, n = 1, 2, 3000, 64, 32, 8, 3
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(B, H, T, D, device="cuda", generator=g).to(torch.bfloat16)
    dy = torch.randn(((R + 1,) if mode == 1 else ()) + (B, H, T, D), device="cuda", generator=g).to(torch.bfloat16)
    y, saved = s.stack_forward(x, L, R, n, mode)
    dx = s.stack_backward(x, saved, dy, L, R, n, mode)
    back = n * (L + R) if mode == 1 else n * L
    for r in range(world):
        t0, t1 = tshard.shard_bounds(T, world, r, 128)
        a0, a1 = max(0, t0 - _round_up(back, 128)), min(T, t1 + _round_up(n * R, 128))
        ye, _ = s.stack_forward(x[:, :, a0:a1].contiguous(), L, R, n, mode)
        assert torch.equal(ye[..., t0 - a0:t1 - a0, :], y[..., t0:t1, :])
        h = _round_up(2 * n * (L + R), 128)
        b0, b1 = max(0, t0 - h), min(T, t1 + h)
        xe = x[:, :, b0:b1].contiguous()
        _, se = s.stack_forward(xe, L, R, n, mode)
        dxe = s.stack_backward(xe, se, dy[..., b0:b1, :].contiguous(), L, R, n, mode)
        assert torch.equal(dxe[..., t0 - b0:t1 - b0, :], dx[..., t0:t1, :])
