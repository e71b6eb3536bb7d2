"""GPU parity at BASELINE.json's full configuration sizes, in the launch configuration the bench
uses (persistent grids over all tiles), on outputs the oracle can compute: sampled (batch, head)
planes, or — for the hour-long stream, whose T x T oracle is out of reach — slabs around sampled
frames, which are exact by locality (Eq. 4's window: a row depends on frames within L + R of it,
SURVEY §8(c) "time sharding" pins).  Gates as in test_gpu_parity (G27)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

L, R = 32, 8


def _excess(got, ref, name=""):
    from test_gpu_parity import excess
    return excess(got, ref, "bf16", name)


def _rand(shape, seed):
    g = torch.Generator("cuda").manual_seed(seed)
    return torch.randn(*shape, device="cuda", generator=g).to(torch.bfloat16)


def _host(t):
    return t.double().cpu().numpy()


def test_large_config_sampled_heads():
    # configs[3]: wav2vec2-large shape, B=64, H=16, T=1750, D=64 (one GPU's worth is B=8 at 8 GPUs;
    # here the whole batch on one device: 14,336 tiles over the persistent grid)
    import paper_2302_13451_b200 as s
    B, H, T, D = 64, 16, 1750, 64
    q, k, v, do = (_rand((B, H, T, D), 20 + i) for i in range(4))
    o, lse = s.sa_forward(q, k, v, L, R)
    dq, dk, dv = s.sa_backward(q, k, v, o, lse, do, L, R)
    for (b, h) in ((0, 0), (17, 3), (40, 15), (63, 8)):
        Q, K, V, dO = (_host(x[b, h]) for x in (q, k, v, do))
        O, LSE = oracle.sa.sa_forward(Q, K, V, L, R)
        G = oracle.sa.sa_backward(Q, K, V, dO, L, R)
        for name, got, ref in (("O", o[b, h], O), ("LSE", lse[b, h], LSE), ("dQ", dq[b, h], G[0]),
                               ("dK", dk[b, h], G[1]), ("dV", dv[b, h], G[2])):
            assert _excess(got, ref, name) <= 0, (b, h, name)


def test_hour_stream_slabs():
    # configs[4]: one hour-long stream, B=1, H=12, T=180,000.  The oracle runs on slabs of
    # 2 x 160 frames around sampled centres (tile and CTA boundaries, both sequence ends) and
    # only the rows whose whole dependency cone lies inside the slab are compared.
    import paper_2302_13451_b200 as s
    B, H, T, D = 1, 12, 180_000, 64
    q, k, v, do = (_rand((B, H, T, D), 30 + i) for i in range(4))
    o, lse = s.sa_forward(q, k, v, L, R)
    dq, dk, dv = s.sa_backward(q, k, v, o, lse, do, L, R)
    half, chk = 160, 32
    for c in (0, 128, 64_000, 90_047, 121_600, T - 1):
        a, b = max(0, c - half), min(T, c + half)
        sl = lambda x: _host(x[0, :, a:b])  # noqa: E731
        Q, K, V, dO = sl(q), sl(k), sl(v), sl(do)
        O, LSE = oracle.sa.sa_forward(Q, K, V, L, R)
        G = oracle.sa.sa_backward(Q, K, V, dO, L, R)
        lo, hi = max(a, c - chk), min(b, c + chk)
        r = slice(lo - a, hi - a)
        # exactness of the slab: rows lo..hi keep their full window (or the true sequence edge)
        assert (lo - L - R >= a or a == 0) and (hi + L + R <= b or b == T)
        for name, got, ref in (("O", o[0, :, lo:hi], O[:, r]), ("LSE", lse[0, :, lo:hi], LSE[:, r]),
                               ("dQ", dq[0, :, lo:hi], G[0][:, r]), ("dK", dk[0, :, lo:hi], G[1][:, r]),
                               ("dV", dv[0, :, lo:hi], G[2][:, r])):
            assert _excess(got, ref, name) <= 0, (c, name)


def test_llsa_base_config_sampled_heads():
    # configs[2]: LLSA at the base shape, C = R + 1 = 9 channels, B=8, H=12, T=1750 (dense inputs)
    import paper_2302_13451_b200 as s
    B, H, T, D, C = 8, 12, 1750, 64, R + 1
    q, k, v, do = (_rand((C, B, H, T, D), 40 + i) for i in range(4))
    o, lse = s.llsa_forward(q, k, v, L, R)
    dq, dk, dv = s.llsa_backward(q, k, v, o, lse, do, L, R)
    for (b, h) in ((0, 0), (5, 7), (7, 11)):
        Q, K, V, dO = (_host(x[:, b:b + 1, h:h + 1]) for x in (q, k, v, do))
        O, LSE = oracle.llsa.llsa_forward(Q, K, V, L, R)
        G = oracle.llsa.llsa_backward(Q, K, V, dO, L, R)
        for name, got, ref in (("O", o[:, b:b + 1, h:h + 1], O), ("LSE", lse[:, b:b + 1, h:h + 1], LSE),
                               ("dQ", dq[:, b:b + 1, h:h + 1], G[0]), ("dK", dk[:, b:b + 1, h:h + 1], G[1]),
                               ("dV", dv[:, b:b + 1, h:h + 1], G[2])):
            assert _excess(got, ref, name) <= 0, (b, h, name)
