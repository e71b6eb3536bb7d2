"""NEXT-3: a HuBERT/wav2vec2-base-shaped transformer encoder layer around the
SA / LLSA kernels — the training-step workload the paper's attention module sits in (SHuBERT,
P:L289; the layer is HuBERT's).

    x -> QKV projection -> heads [B, H, T, 64] -> SA (Eq. 4-13) or LLSA (Eq. 14-16) -> output
      projection -> residual -> LayerNorm -> FFN (GELU) -> residual -> LayerNorm   (post-LN,
      as wav2vec2-base / HuBERT-base)

The projections, FFN and LayerNorms are frame-local library ops (cuBLAS GEMMs through
torch); only the attention is this repo's kernels (autograd through SAFunction /
LLSAFunction -> the C ABI).  For LLSA the R+1 channels are folded into the batch for every
frame-local op ("the LLSA channel axis folds into the GEMM M dimension"), so a
layer maps [C, B, T, d] -> [C, B, T, d] and the channel contract of the stack holds.

`MaskedEncoderLayer` is the same layer with masked acausal attention (MAA: dense T x T scores,
band mask, softmax — P:L78-85) computed by torch: the paper's comparison point, used as the
baseline of the bench's `encoder` sub-object and as the reference of the parity test.
"""
from __future__ import annotations

import torch
import torch.nn as nn
import torch.nn.functional as F

from . import LLSAFunction, SAFunction


class _Layer(nn.Module):
    def __init__(self, d_model=768, n_heads=12, d_ff=3072, L=32, R=8):
        super().__init__()
        self.H, self.Dh, self.L, self.R = n_heads, d_model // n_heads, L, R
        self.qkv = nn.Linear(d_model, 3 * d_model)
        self.out = nn.Linear(d_model, d_model)
        self.ln1 = nn.LayerNorm(d_model)
        self.ff1 = nn.Linear(d_model, d_ff)
        self.ff2 = nn.Linear(d_ff, d_model)
        self.ln2 = nn.LayerNorm(d_model)

    def _heads(self, x):
        # [N, T, 3d] -> three [N, H, T, Dh] contiguous
        N, T, _ = x.shape
        q, k, v = x.view(N, T, 3, self.H, self.Dh).permute(2, 0, 3, 1, 4).unbind(0)
        return q.contiguous(), k.contiguous(), v.contiguous()

    def attention(self, q, k, v):
        raise NotImplementedError

    def forward(self, x):
        lead = x.shape[:-2]
        T, d = x.shape[-2:]
        xf = x.reshape(-1, T, d)
        q, k, v = self._heads(self.qkv(xf))
        o = self.attention(q.view(*lead, self.H, T, self.Dh), k.view(*lead, self.H, T, self.Dh),
                           v.view(*lead, self.H, T, self.Dh))
        o = o.reshape(-1, self.H, T, self.Dh).transpose(1, 2).reshape(-1, T, d)
        h = self.ln1(xf + self.out(o))
        y = self.ln2(h + self.ff2(F.gelu(self.ff1(h))))
        return y.view(*lead, T, d)


class SAEncoderLayer(_Layer):
    """Encoder layer with streaming attention (the repo's kernels).  x [B, T, d]."""

    def attention(self, q, k, v):
        return SAFunction.apply(q, k, v, self.L, self.R)


class LLSAEncoderLayer(_Layer):
    """Encoder layer with low-latency streaming attention.  x [C = R+1, B, T, d] (channel-major;
    the first layer's input is the frame sequence duplicated into every channel)."""

    def attention(self, q, k, v):
        return LLSAFunction.apply(q, k, v, self.L, self.R)


class MaskedEncoderLayer(_Layer):
    """The same layer with masked acausal attention (dense scores + band mask), torch ops."""

    def attention(self, q, k, v):
        T = q.shape[-2]
        i = torch.arange(T, device=q.device)
        band = (i[None, :] >= i[:, None] - self.L) & (i[None, :] <= i[:, None] + self.R)
        return F.scaled_dot_product_attention(q, k, v, attn_mask=band)
