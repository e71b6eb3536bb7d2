"""Oracle: n-layer attention stack (the layer-stack driver of SURVEY.md §8(a) a11).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy fp64.

The paper stacks SA / LLSA layers inside HuBERT transformer blocks
but the hot path has no projections or FFN, so the block is read as (G12):
    Q = K = V = X_l   (tied, per head and per channel)
    Y_l = SA(X_l) or LLSA(X_l)
    X_{l+1} = (X_l + Y_l) / 2          frame-local and channel-wise
LLSA channelizes once at layer 1 (G11); its designated output is
channel R (G10).  The backward chains
    dO_l = dX_{l+1} / 2,   dX_l = dX_{l+1} / 2 + dQ_l + dK_l + dV_l
and, for LLSA, dX_0 = sum_c dX_0[c] (adjoint of the duplication).
"""
from __future__ import annotations

import numpy as np

from .sa import sa_forward, sa_backward
from .llsa import llsa_forward, llsa_backward, channelize


def stack_forward(X0, L: int, R: int, n_layers: int, mode: str, scale=None):
    """Returns (X_n, xs) with xs = [X_0 .. X_{n-1}] as fed to each layer.
    mode 'sa': X [.., T, D].  mode 'llsa': X_n [C, .., T, D] (X_0 channelized)."""
    X = np.asarray(X0, dtype=np.float64)
    if mode == "llsa":
        X = channelize(X, R)
    xs = []
    for _ in range(n_layers):
        xs.append(X)
        if mode == "sa":
            Y, _ = sa_forward(X, X, X, L, R, scale)
        elif mode == "llsa":
            Y, _ = llsa_forward(X, X, X, L, R, scale)
        else:
            raise ValueError(mode)
        X = 0.5 * (X + Y)
    return X, xs


def stack_backward(X0, dXn, L: int, R: int, n_layers: int, mode: str, scale=None):
    """Gradient of <dXn, X_n> with respect to X_0 (the stack input)."""
    _, xs = stack_forward(X0, L, R, n_layers, mode, scale)
    dX = np.asarray(dXn, dtype=np.float64)
    for X in reversed(xs):
        dO = 0.5 * dX
        if mode == "sa":
            dq, dk, dv = sa_backward(X, X, X, dO, L, R, scale)
        else:
            dq, dk, dv = llsa_backward(X, X, X, dO, L, R, scale)
        dX = 0.5 * dX + dq + dk + dv
    if mode == "llsa":
        dX = dX.sum(axis=0)
    return dX
