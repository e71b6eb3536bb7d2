"""NEXT-3: the encoder layer around the kernels (paper_2302_13451_b200/encoder.py) against the same
layer with masked acausal attention computed by torch (dense scores + band mask): outputs and
every parameter gradient.  fp32 runs the exact CUDA-core attention (1e-4 relative to the
activations' scale); bf16 runs the tensor-core path (bf16 layer, checked at bf16 resolution)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pair(mode, dtype, L, R):
    from paper_2302_13451_b200 import encoder
    torch.manual_seed(0)
    ref = encoder.MaskedEncoderLayer(L=L, R=R).cuda().to(dtype)
    cls = encoder.SAEncoderLayer if mode == "sa" else encoder.LLSAEncoderLayer
    lay = cls(L=L, R=R).cuda().to(dtype)
    lay.load_state_dict(ref.state_dict())
    return ref, lay


@pytest.mark.parametrize("dtype,tol", [(torch.float32, 1e-4), (torch.bfloat16, 6e-2)])
def test_sa_encoder_layer_matches_masked(dtype, tol):
    L, R, B, T = 32, 8, 2, 300
    ref, lay = _pair("sa", dtype, L, R)
    g = torch.Generator("cuda").manual_seed(1)
    x = torch.randn(B, T, 768, device="cuda", generator=g).to(dtype)
    dy = torch.randn(B, T, 768, device="cuda", generator=g).to(dtype)
    xs = [x.clone().requires_grad_(True) for _ in range(2)]
    ys = [m(xx) for m, xx in zip((ref, lay), xs)]
    for y in ys:
        y.backward(dy)
    def rel(a, b):
        return float((a.float() - b.float()).abs().max() / max(1.0, float(b.float().abs().max())))
    assert rel(ys[1], ys[0]) <= tol
    assert rel(xs[1].grad, xs[0].grad) <= tol
    for (n, p0), (_, p1) in zip(ref.named_parameters(), lay.named_parameters()):
        assert rel(p1.grad, p0.grad) <= tol, n


def test_llsa_encoder_layer_channels_and_grad():
    # LLSA layer on [C, B, T, d]: channel R of a duplicated input equals the SA layer with look-back
    # L and look-ahead R (Eq. 14's duplication identity, channel c == SA(L+R-c, c)); and the
    # gradient flows through every channel
    L, R, B, T = 16, 4, 1, 200
    from paper_2302_13451_b200 import encoder
    torch.manual_seed(0)
    ll = encoder.LLSAEncoderLayer(L=L, R=R).cuda()
    g = torch.Generator("cuda").manual_seed(2)
    x = torch.randn(B, T, 768, device="cuda", generator=g)
    xc = x.unsqueeze(0).expand(R + 1, B, T, 768).contiguous().requires_grad_(True)
    y = ll(xc)
    for c in (0, R):
        sa = encoder.SAEncoderLayer(L=L + R - c, R=c).cuda()
        sa.load_state_dict(ll.state_dict())
        ys = sa(x)
        assert float((y[c] - ys).abs().max()) <= 1e-4
    y.sum().backward()
    assert torch.isfinite(xc.grad).all() and float(xc.grad.abs().sum()) > 0
