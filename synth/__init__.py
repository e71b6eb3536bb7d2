"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no scores, softmax, windows or
gradients).  It only draws numbers: a counter-based generator so that every
value is a pure function of (seed, tensor id, flat index), independent of
platform, call order and tensor shape.

Generator (documented so it can be re-implemented anywhere):
    x = SplitMix64(seed * 0x9E3779B97F4A7C15 + tensor_id * 0xD1B54A32D192ED03
                   + 2*i) and the same with 2*i+1, i = flat element index
    u1 = ((x1 >> 11) + 0.5) / 2**53,  u2 = ((x2 >> 11) + 0.5) / 2**53
    z  = sqrt(-2 ln u1) * cos(2 pi u2)                 (Box-Muller, fp64)
Values are then rounded (round-to-nearest-even) to the kernel dtype; both the
GPU path and the oracle consume those rounded values.

Workload recipe: Q, K, V, dO iid N(0,1) at the
wav2vec2/HuBERT-base attention shape (50 Hz frames, head dim 64); the latency
witness input of SURVEY.md §8(c) is provided by :func:`witness`.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)
_TID = np.uint64(0xD1B54A32D192ED03)

# tensor ids used across tests/bench so the same (seed, name) is the same data
TENSOR_IDS = {"Q": 1, "K": 2, "V": 3, "dO": 4, "X": 5, "dY": 6, "perturb": 7}


def _splitmix64(x: np.ndarray) -> np.ndarray:
    x = x + _GOLD
    z = x
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def uniform_bits(seed: int, tensor_id: int, n: int, offset: int = 0) -> np.ndarray:
    """2n raw 64-bit draws for flat indices [offset, offset+n)."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed) * _GOLD + np.uint64(tensor_id) * _TID
        idx = np.arange(offset, offset + n, dtype=np.uint64) * np.uint64(2)
        x1 = _splitmix64(base + idx)
        x2 = _splitmix64(base + idx + np.uint64(1))
    return x1, x2


def normal(seed: int, tensor_id: int | str, shape, offset: int = 0) -> np.ndarray:
    """iid N(0,1) fp64 array of `shape`, element i = f(seed, tensor_id, offset + i)."""
    if isinstance(tensor_id, str):
        tensor_id = TENSOR_IDS[tensor_id]
    n = int(np.prod(shape)) if len(shape) else 1
    x1, x2 = uniform_bits(seed, tensor_id, n, offset)
    inv = 1.0 / 9007199254740992.0  # 2**-53
    u1 = ((x1 >> np.uint64(11)).astype(np.float64) + 0.5) * inv
    u2 = ((x2 >> np.uint64(11)).astype(np.float64) + 0.5) * inv
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return z.reshape(shape)


def round_to(x: np.ndarray, dtype: str) -> np.ndarray:
    """Round fp64 values to the kernel dtype ('f32' | 'bf16'), returned as fp64.

    bf16 is round-to-nearest-even of the fp32 value (the conversion torch and
    the CUDA intrinsics perform).  Pure bit manipulation, no method arithmetic.
    """
    f = np.asarray(x, dtype=np.float32)
    if dtype == "f32":
        return f.astype(np.float64)
    if dtype == "bf16":
        b = f.view(np.uint32).astype(np.uint64)
        lsb = (b >> np.uint64(16)) & np.uint64(1)
        r = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)) << np.uint64(16)
        r = r.astype(np.uint32)
        nan = np.isnan(f)
        out = r.view(np.float32).astype(np.float64)
        out[nan] = np.nan
        return out
    raise ValueError(f"unknown dtype {dtype!r}")


def qkv(seed: int, shape, dtype: str = "f32", q_scale: float = 1.0):
    """Q, K, V iid N(0,1) (Q optionally scaled: the stress distribution), rounded."""
    q = round_to(q_scale * normal(seed, "Q", shape), dtype)
    k = round_to(normal(seed, "K", shape), dtype)
    v = round_to(normal(seed, "V", shape), dtype)
    return q, k, v


def grad_out(seed: int, shape, dtype: str = "f32"):
    return round_to(normal(seed, "dO", shape), dtype)


def witness(seed: int, B: int, H: int, T: int, D: int, kappa: float = 20.0, dtype: str = "f64"):
    """Latency-witness input of SURVEY.md §8(c) O7(ii):
    x_u = 0.1*N(0,1) + [kappa*u/T, 1, 0, ...]  (scores grow with u, so each layer
    attends hardest to its furthest look-ahead key and the depth*R chain survives
    rounding).  Returned shape [B,H,T,D]."""
    x = 0.1 * normal(seed, "X", (B, H, T, D))
    u = np.arange(T, dtype=np.float64)
    x[..., 0] += kappa * u / T
    if D > 1:
        x[..., 1] += 1.0
    return x if dtype == "f64" else round_to(x, dtype)
