"""GPU parity of the stored-band mode (sa_forward_p / sa_backward_p; NEXT-4, the paper's
N_T x (A+B+1) a_t matrix) against the oracle (oracle.sa.sa_band_probs,
sa_backward_band, sa_forward / sa_backward).  Gates as tests/test_gpu_parity.py."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import TOL, dev, excess, host, maxerr, sattn

pytestmark = pytest.mark.gpu

CASES = [
    ((1, 1, 16, 4), 3, 1, "f32"), ((2, 3, 37, 4), 0, 0, "f32"), ((2, 3, 37, 4), 0, 5, "f32"),
    ((2, 3, 37, 4), 5, 0, "f32"), ((1, 2, 129, 64), 32, 8, "f32"), ((1, 2, 300, 64), 200, 150, "f32"),
    ((1, 1, 1, 8), 3, 2, "f32"), ((1, 2, 65, 2), 1, 1, "f32"), ((1, 1, 200, 32), 0, 63, "f32"),
    ((2, 2, 1750, 64), 32, 8, "bf16"), ((1, 2, 300, 64), 32, 16, "bf16"), ((1, 3, 777, 64), 32, 32, "bf16"),
    ((1, 2, 130, 16), 7, 3, "bf16"), ((1, 2, 129, 64), 0, 0, "bf16"), ((3, 2, 300, 64), 24, 0, "bf16"),
    ((1, 3, 777, 64), 16, 8, "bf16"), ((2, 1, 1000, 64), 40, 23, "bf16"), ((1, 1, 5, 64), 2, 2, "bf16"),
    # wide bands: the backward as 48-column sub-bands of a_t on tensor cores (W = 57, 351, 490)
    ((1, 2, 300, 64), 32, 24, "bf16"), ((1, 2, 600, 64), 200, 150, "bf16"), ((1, 1, 1000, 64), 245, 244, "bf16"),
    # packed tiles over the flattened B*H*T axis (heads shorter than a tile; windows cut by head
    # boundaries inside a tile)
    ((2, 3, 50, 64), 32, 8, "bf16"), ((4, 4, 20, 64), 32, 8, "bf16"), ((3, 5, 100, 64), 8, 8, "bf16"),
    ((5, 40, 1, 64), 32, 8, "bf16"), ((3, 7, 127, 64), 32, 8, "bf16"),
]


def _ld(L, R):
    return (L + R + 1 + 7) // 8 * 8


@pytest.mark.parametrize("impl", ["auto", "ffma"])
@pytest.mark.parametrize("shape,L,R,dt", CASES)
def test_sa_stored_band(shape, L, R, dt, impl):
    # auto: tensor cores for bf16 D=64 (forward W <= 64; backward W <= 49 in one pass, wider bands
    # as 48-column sub-bands), CUDA cores otherwise
    s = sattn()
    if impl == "ffma" and dt == "f32":
        pytest.skip("fp32 runs on the CUDA-core kernels under auto already")
    q, k, v = synth.qkv(11, shape, dt)
    do = synth.grad_out(11, shape, dt)
    tq, tk, tv, tdo = (dev(x, dt) for x in (q, k, v, do))
    W = L + R + 1
    o, lse, p = s.sa_forward_p(tq, tk, tv, L, R, impl=impl)
    assert p.shape == tuple(shape[:-1]) + (_ld(L, R),) and p.dtype == tq.dtype
    O, LSE = oracle.sa.sa_forward(q, k, v, L, R)
    A = oracle.sa.sa_band_probs(q, k, L, R)
    assert excess(o, O, dt, "O") <= 0, ("O", maxerr(o, O))
    assert maxerr(lse, LSE) <= TOL[dt], ("LSE", maxerr(lse, LSE))
    # the band: entries within the gate; exact zeros outside the clipped window and in the padding
    ph = host(p)
    assert maxerr(p[..., :W], A) <= (TOL[dt] if dt == "f32" else 4e-3), ("P", maxerr(p[..., :W], A))
    assert (ph[..., W:] == 0).all()
    t = np.arange(shape[2])[:, None]
    u = t - L + np.arange(W)[None, :]
    assert (ph[..., :W][..., (u < 0) | (u >= shape[2])] == 0).all()
    # backward from the GPU's own band
    dq, dk, dv = s.sa_backward_p(tq, tk, tv, o, p, tdo, L, R, impl=impl)
    G = oracle.sa.sa_backward(q, k, v, do, L, R)
    for name, got, ref in (("dQ", dq, G[0]), ("dK", dk, G[1]), ("dV", dv, G[2])):
        assert excess(got, ref, dt, name) <= 0, (name, maxerr(got, ref))
    # backward from the oracle's band (rounded to the tensor dtype): the band-form oracle
    pa = torch.zeros_like(p)
    pa[..., :W] = dev(A, dt)
    o_ref = dev(O, dt)
    dq2, dk2, dv2 = s.sa_backward_p(tq, tk, tv, o_ref, pa, tdo, L, R, impl=impl)
    Ar = host(pa)[..., :W]
    G2 = oracle.sa.sa_backward_band(Ar, q, k, v, do, L, R)
    for name, got, ref in (("dQ", dq2, G2[0]), ("dK", dk2, G2[1]), ("dV", dv2, G2[2])):
        assert excess(got, ref, dt, name) <= 0, (name, maxerr(got, ref))


def test_sa_stored_band_errors():
    s = sattn()
    q = torch.zeros(1, 1, 16, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(s.SattnError):
        s.sa_forward_p(q.float(), q.float(), q.float(), 3, 1, impl="tc")
    with pytest.raises(s.SattnError):
        s.sa_forward_p(q, q, q, 40, 40, impl="tc")        # W = 81 > 64
    q32 = torch.zeros(1, 1, 16, 32, device="cuda", dtype=torch.bfloat16)
    o, lse, p = s.sa_forward_p(q32, q32, q32, 3, 1)
    with pytest.raises(s.SattnError):
        s.sa_backward_p(q32, q32, q32, o, p, q32, 3, 1, impl="tc")   # D = 32: no tensor-core path
    with pytest.raises(s.SattnError):
        s.sa_forward_p(q.cpu(), q.cpu(), q.cpu(), 3, 1)


def test_sa_stored_band_deterministic():
    s = sattn()
    shape, L, R = (2, 2, 600, 64), 32, 8
    q, k, v = (dev(x, "bf16") for x in synth.qkv(12, shape, "bf16"))
    do = dev(synth.grad_out(12, shape, "bf16"), "bf16")
    o, lse, p = s.sa_forward_p(q, k, v, L, R)
    r1 = s.sa_backward_p(q, k, v, o, p, do, L, R)
    r2 = s.sa_backward_p(q, k, v, o, p, do, L, R)
    for a, b in zip(r1, r2):
        assert torch.equal(a, b)
    o2, _ = s.sa_forward(q, k, v, L, R)
    assert torch.equal(o, o2)   # the band store does not change the forward's arithmetic
    of, _, pf = s.sa_forward_p(q, k, v, L, R, impl="ffma")
    assert torch.equal(of, s.sa_forward(q, k, v, L, R, impl="ffma")[0])
    assert (p.float() - pf.float()).abs().max().item() <= 4e-3   # tensor-core band == CUDA-core band


def test_sa_stored_band_full_base_shape_sampled_heads():
    # BASELINE configs[1] (B=8, H=12, T=1750, D=64, (32,8), bf16) in the launch configuration the
    # bench's headline (stored-band mode) times; 6 sampled heads checked element by element
    s = sattn()
    B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
    W = L + R + 1
    tq, tk, tv = (torch.randn(B, H, T, D, device="cuda", generator=torch.Generator("cuda").manual_seed(i))
                  .to(torch.bfloat16) for i in range(3))
    tdo = torch.randn(B, H, T, D, device="cuda", generator=torch.Generator("cuda").manual_seed(9)).to(torch.bfloat16)
    o, lse, p = s.sa_forward_p(tq, tk, tv, L, R)
    dq, dk, dv = s.sa_backward_p(tq, tk, tv, o, p, tdo, L, R)
    for (b, h) in ((0, 0), (3, 7), (7, 11), (5, 2), (1, 10), (6, 5)):
        q, k, v, do = (host(x[b, h]) for x in (tq, tk, tv, tdo))
        O, LSE = oracle.sa.sa_forward(q, k, v, L, R)
        A = oracle.sa.sa_band_probs(q, k, L, R)
        G = oracle.sa.sa_backward(q, k, v, do, L, R)
        assert maxerr(p[b, h, :, :W], A) <= 4e-3, (b, h, "P")
        for name, got, ref in (("O", o[b, h], O), ("LSE", lse[b, h], LSE), ("dQ", dq[b, h], G[0]),
                               ("dK", dk[b, h], G[1]), ("dV", dv[b, h], G[2])):
            assert excess(got, ref, "bf16", name) <= 0, (b, h, name, maxerr(got, ref))
