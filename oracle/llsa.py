"""Oracle: low-latency streaming attention (LLSA), Eq. 14-16, Fig. 3(c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy fp64.

Tensors are channel-major: X[c, ..., t, :] is "the version of frame t computed
with c frames of look-ahead", c in [0, R], C = R + 1.

Reading of Eq. 14 (G6): the paper's key subscripts follow Fig. 3(c)
but its output index runs the other way.  With c_eq = R - c (c = number of
look-ahead frames output (t, c) uses, the figure's convention) and the
anchor s = t - c_eq, Eq. 14 reads

    z_{t,c} = [k_{s-L,R}, ..., k_{s,R}, k_{s+1,R-1}, ..., k_{s+R,0}]^T q_{t,c} / sqrt(d_k)

i.e. L+1 look-back keys from channel R and then frame s+j from channel R-j,
j = 1..R.  Eq. 15 sums the values of the same slots with a_{t,c} = softmax(z_{t,c}).
The query is q_{t,c} of the same channel (G7).  Slots outside [0, T-1] are
dropped (G2).  The primary functions below transcribe this gather form; the
flattened-mask functions are an independent second formulation (the "horizon
form": output (t,c) attends slots (u, min(R, t+c-u)) for u in [t+c-R-L, t+c]).
"""
from __future__ import annotations

import numpy as np

from .sa import attention_fwd, attention_bwd


def window_slots(t: int, c: int, T: int, L: int, R: int):
    """The slots (frame, channel) of Eq. 14 for output (t, c), in Eq. 14's order."""
    s = t - (R - c)
    slots = [(s - L + i, R) for i in range(L + 1)] + [(s + j, R - j) for j in range(1, R + 1)]
    return [(u, ch) for (u, ch) in slots if 0 <= u < T]


def _gather_index(T: int, L: int, R: int, c: int):
    """Vectorised window_slots for every t at fixed c: frames [T, W], channels [W], valid [T, W]."""
    W = L + R + 1
    t = np.arange(T)[:, None]
    s = t - (R - c)
    i = np.arange(W)[None, :]
    frames = np.where(i <= L, s - L + i, s + (i - L))
    chans = np.where(np.arange(W) <= L, R, R - (np.arange(W) - L))
    valid = (frames >= 0) & (frames < T)
    return np.clip(frames, 0, T - 1), chans, valid


def channelize(X, R: int):
    """Layer-1 channel construction: every channel is a copy of X ("simply
    duplicated"; reading G11).  [..., T, D] -> [R+1, ..., T, D]."""
    X = np.asarray(X, dtype=np.float64)
    return np.stack([X] * (R + 1), axis=0)


def _scale(D, scale):
    return 1.0 / np.sqrt(D) if not scale else float(scale)


def llsa_forward(Q, K, V, L: int, R: int, scale: float | None = None):
    """Eq. 14-15: (O [C, ..., T, D], LSE [C, ..., T]) from channel-major Q, K, V."""
    Q, K, V = (np.asarray(x, dtype=np.float64) for x in (Q, K, V))
    C = R + 1
    assert Q.shape[0] == C, "channel axis must be R+1"
    T, D = Q.shape[-2:]
    s = _scale(D, scale)
    O = np.empty_like(Q)
    LSE = np.empty(Q.shape[:-1])
    for idx in np.ndindex(*Q.shape[1:-2]):
        for c in range(C):
            f, ch, valid = _gather_index(T, L, R, c)
            Kw = K[(ch[None, :],) + idx + (f,)]          # [T, W, D]: k_{slot} of Eq. 14
            Vw = V[(ch[None, :],) + idx + (f,)]          # [T, W, D]: v_{slot} of Eq. 15
            q = Q[(c,) + idx]                             # q_{t,c}
            z = np.einsum("td,twd->tw", q, Kw) * s        # Eq. 14
            z = np.where(valid, z, -np.inf)
            m = z.max(axis=1, keepdims=True)
            e = np.exp(z - m)
            l = e.sum(axis=1, keepdims=True)
            a = e / l                                     # a_{t,c} = softmax(z_{t,c})
            O[(c,) + idx] = np.einsum("tw,twd->td", a, Vw)  # Eq. 15
            LSE[(c,) + idx] = m[:, 0] + np.log(l[:, 0])
    return O, LSE


def llsa_backward(Q, K, V, dO, L: int, R: int, scale: float | None = None):
    """Exact gradient of llsa_forward (G8/G9): the chain rule over the same slots.

    dv_{slot} += a_{t,c,slot} dy_{t,c}   -- Eq. 16's double sum over (n, c1)
    dz_{t,c}  = J^T (V_win dy_{t,c})      -- as Eq. 9 for SA
    dq_{t,c}  = dz K_win / sqrt d          -- as Eq. 10
    dk_{slot} += dz_{t,c,slot} q_{t,c} / sqrt d   -- as Eq. 11-13
    """
    Q, K, V, dO = (np.asarray(x, dtype=np.float64) for x in (Q, K, V, dO))
    C = R + 1
    T, D = Q.shape[-2:]
    s = _scale(D, scale)
    dQ = np.zeros_like(Q)
    dK = np.zeros_like(K)
    dV = np.zeros_like(V)
    for idx in np.ndindex(*Q.shape[1:-2]):
        for c in range(C):
            f, ch, valid = _gather_index(T, L, R, c)
            chb = np.broadcast_to(ch[None, :], f.shape)
            Kw = K[(chb,) + idx + (f,)]
            Vw = V[(chb,) + idx + (f,)]
            q = Q[(c,) + idx]
            dy = dO[(c,) + idx]
            z = np.where(valid, np.einsum("td,twd->tw", q, Kw) * s, -np.inf)
            e = np.exp(z - z.max(axis=1, keepdims=True))
            a = e / e.sum(axis=1, keepdims=True)
            da = np.einsum("td,twd->tw", dy, Vw)
            dz = a * (da - (a * da).sum(axis=1, keepdims=True))
            dQ[(c,) + idx] = np.einsum("tw,twd->td", dz, Kw) * s
            tgt_v = dV[(slice(None),) + idx]
            tgt_k = dK[(slice(None),) + idx]
            np.add.at(tgt_v, (chb[valid], f[valid]), (a[..., None] * dy[:, None, :])[valid])
            np.add.at(tgt_k, (chb[valid], f[valid]), (dz[..., None] * q[:, None, :] * s)[valid])
    return dQ, dK, dV


# ---------------------------------------------------------------------------
# Independent second formulation: flatten slots (t, c) -> i = t*C + c and run
# the dense masked attention of oracle.sa over the flattened sequence with the
# horizon mask.  O((T*C)^2): tiny inputs only.
# ---------------------------------------------------------------------------

def horizon_mask(T: int, L: int, R: int) -> np.ndarray:
    """M[(t,c),(u,c')] = [t+c-R-L <= u <= t+c] and [c' == min(R, t+c-u)], flattened t-major."""
    C = R + 1
    t = np.repeat(np.arange(T), C)
    c = np.tile(np.arange(C), T)
    h = (t + c)[:, None]
    u = t[None, :]
    cp = c[None, :]
    return (u >= h - R - L) & (u <= h) & (cp == np.minimum(R, h - u))


def _flat(X):
    # [C, ..., T, D] -> [..., T*C, D] with i = t*C + c
    X = np.moveaxis(X, 0, -2)
    return X.reshape(X.shape[:-3] + (X.shape[-3] * X.shape[-2], X.shape[-1]))


def _unflat(Xf, C):
    T = Xf.shape[-2] // C
    X = Xf.reshape(Xf.shape[:-2] + (T, C, Xf.shape[-1]))
    return np.moveaxis(X, -2, 0)


def llsa_forward_flat(Q, K, V, L: int, R: int, scale: float | None = None):
    C = R + 1
    T, D = np.shape(Q)[-2:]
    s = _scale(D, scale)
    Qf, Kf, Vf = (_flat(np.asarray(x, dtype=np.float64)) for x in (Q, K, V))
    M = horizon_mask(T, L, R)
    Of = np.empty_like(Qf)
    for idx in np.ndindex(*Qf.shape[:-2]):
        Of[idx], _, _ = attention_fwd(Qf[idx], Kf[idx], Vf[idx], M, s)
    return _unflat(Of, C)


def llsa_backward_flat(Q, K, V, dO, L: int, R: int, scale: float | None = None):
    C = R + 1
    T, D = np.shape(Q)[-2:]
    s = _scale(D, scale)
    Qf, Kf, Vf, dOf = (_flat(np.asarray(x, dtype=np.float64)) for x in (Q, K, V, dO))
    M = horizon_mask(T, L, R)
    g = [np.empty_like(Qf) for _ in range(3)]
    for idx in np.ndindex(*Qf.shape[:-2]):
        r = attention_bwd(Qf[idx], Kf[idx], Vf[idx], M, s, dOf[idx])
        for j in range(3):
            g[j][idx] = r[j]
    return tuple(_unflat(x, C) for x in g)
