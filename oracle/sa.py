"""Oracle: acausal (AA), masked acausal (MAA) and streaming attention (SA).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy fp64.

SA is defined by Eq. 4-6: each query t uses keys/values
t-B .. t+A (paper letters; this build: L = look-back B, R = look-ahead A, G1).
The method reaches exactly the band-masked dense attention of Eq. 3
-- SA only skips computing the z's MAA would discard -- so the
oracle is that plain definition written out: all T x T scores (Eq. 1), the
band mask applied before the softmax (Eq. 3, "replaced by a large negative
value", read as -inf, G14), softmax, value sum (Eq. 2).  Sequence edges clip
the band to [0, T-1] and the softmax runs over the valid keys only (G2).
"""
from __future__ import annotations

import numpy as np


def band_mask(T: int, L: int, R: int) -> np.ndarray:
    """m_t of Eq. 3 for SA's receptive field (Eq. 4):
    row t is True exactly on u in [t-L, t+R] (clipped to [0, T-1])."""
    t = np.arange(T)[:, None]
    u = np.arange(T)[None, :]
    return (u >= t - L) & (u <= t + R)


def attention_fwd(q, k, v, mask, scale):
    """One head of masked SDPA.  q [Tq,D], k/v [Tk,D], mask [Tq,Tk] bool.

    z_t = K^T q_t / sqrt(d_k)        Eq. 1
    z_t[~m_t] = -inf                 Eq. 3
    a_t = softmax(z_t)
    y_t = V^T a_t                    Eq. 2
    LSE_t = log sum_u exp(z_tu)      (the forward's saved statistic)
    """
    z = (q @ k.T) * scale
    z = np.where(mask, z, -np.inf)
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    l = e.sum(axis=1, keepdims=True)
    a = e / l
    y = a @ v
    lse = m[:, 0] + np.log(l[:, 0])
    return y, lse, a


def attention_bwd(q, k, v, mask, scale, dy):
    """Exact gradient of attention_fwd composed with <dy, y>.

    dv_t = sum_n a_{n,t} dy_n                        Eq. 7-8 (bounds per G3)
    dl/da_n = V^T-window dy_n ; dl/dz_n = J^T dl/da_n with the softmax Jacobian
      J = diag(a_n) - a_n a_n^T (Bishop 5.3.4)      Eq. 9
    dq_n = (1/sqrt d) dl/dz_n K                      Eq. 10
    dk_t = sum_n dl/dz_{n,t} q_n / sqrt d  (M_n has one nonzero row q_n^T/sqrt d)
                                                     Eq. 11-13
    """
    _, _, a = attention_fwd(q, k, v, mask, scale)
    dv = a.T @ dy
    da = dy @ v.T
    dz = a * (da - (a * da).sum(axis=1, keepdims=True))
    dq = (dz @ k) * scale
    dk = (dz.T @ q) * scale
    return dq, dk, dv


def _scale(D, scale):
    return 1.0 / np.sqrt(D) if not scale else float(scale)


def _heads(x):
    """Iterate over all leading (batch, head, ...) indices of a [..., T, D] array."""
    return np.ndindex(*x.shape[:-2])


def sa_forward(Q, K, V, L: int, R: int, scale: float | None = None):
    """SA forward over [..., T, D] arrays -> (O [..., T, D], LSE [..., T]).
    Eq. 4-6 via its plain definition (band-masked dense, see module doc)."""
    Q, K, V = (np.asarray(x, dtype=np.float64) for x in (Q, K, V))
    T, D = Q.shape[-2:]
    s = _scale(D, scale)
    mask = band_mask(T, L, R)
    O = np.empty_like(Q)
    LSE = np.empty(Q.shape[:-1])
    for idx in _heads(Q):
        O[idx], LSE[idx], _ = attention_fwd(Q[idx], K[idx], V[idx], mask, s)
    return O, LSE


def sa_backward(Q, K, V, dO, L: int, R: int, scale: float | None = None):
    """SA backward -> (dQ, dK, dV), Eq. 7-13 as the dense chain rule
    over the band-masked definition (masked entries have a = 0, hence dz = 0)."""
    Q, K, V, dO = (np.asarray(x, dtype=np.float64) for x in (Q, K, V, dO))
    T, D = Q.shape[-2:]
    s = _scale(D, scale)
    mask = band_mask(T, L, R)
    dQ, dK, dV = np.empty_like(Q), np.empty_like(K), np.empty_like(V)
    for idx in _heads(Q):
        dQ[idx], dK[idx], dV[idx] = attention_bwd(Q[idx], K[idx], V[idx], mask, s, dO[idx])
    return dQ, dK, dV


def aa_forward(Q, K, V, scale: float | None = None):
    """Acausal attention, Eq. 1-2: every key for every query."""
    Q = np.asarray(Q, dtype=np.float64)
    T, D = Q.shape[-2:]
    O = np.empty_like(Q)
    full = np.ones((T, T), dtype=bool)
    for idx in _heads(Q):
        O[idx], _, _ = attention_fwd(Q[idx], np.asarray(K)[idx], np.asarray(V)[idx], full, _scale(D, scale))
    return O


# ---------------------------------------------------------------------------
# The paper's stored band (NEXT-4).  The paper keeps z_t and a_t
# as N_T x (A+B+1) matrices; the build's stored-band mode keeps a_t.
# ---------------------------------------------------------------------------

def sa_band_probs(Q, K, L: int, R: int, scale: float | None = None):
    """a_t of Eq. 5 stored in the band layout: A[..., t, j] = a_{t, t-L+j},
    j in [0, W), W = L+R+1; 0 where t-L+j is outside [0, T-1] (G2).  Taken from the dense
    definition (attention_fwd's a), entry by entry."""
    Q, K = (np.asarray(x, dtype=np.float64) for x in (Q, K))
    T, D = Q.shape[-2:]
    W = L + R + 1
    s = _scale(D, scale)
    mask = band_mask(T, L, R)
    A = np.zeros(Q.shape[:-1] + (W,))
    for idx in _heads(Q):
        _, _, a = attention_fwd(Q[idx], K[idx], K[idx], mask, s)
        for t in range(T):
            for j in range(W):
                u = t - L + j
                if 0 <= u < T:
                    A[idx + (t, j)] = a[t, u]
    return A


def sa_backward_band(A, Q, K, V, dO, L: int, R: int, scale: float | None = None):
    """SA gradients from a stored band A (layout of sa_band_probs), Eq. 7-13 written in
    the band index j (key u = n - L + j), one shifted slice per j:
      dv_u  = sum_n a_{n,u-n+L} dy_n                  Eq. 7-8 (index condition per G3)
      da_nj = dy_n . v_{n-L+j}                        Eq. 9's dl/da
      dz_nj = a_nj (da_nj - sum_j' a_nj' da_nj')      softmax Jacobian (Eq. 9)
      dq_n  = s sum_j dz_nj k_{n-L+j}                 Eq. 10
      dk_u  = s sum_n dz_{n,u-n+L} q_n                Eq. 11-13
    """
    A, Q, K, V, dO = (np.asarray(x, dtype=np.float64) for x in (A, Q, K, V, dO))
    T, D = Q.shape[-2:]
    W = L + R + 1
    s = _scale(D, scale)
    A = A[..., :W]
    da = np.zeros(A.shape)
    for j in range(W):                      # key u = n - L + j, valid rows n
        n0, n1 = max(0, L - j), min(T, T + L - j)
        if n0 < n1:
            da[..., n0:n1, j] = np.einsum("...nd,...nd->...n", dO[..., n0:n1, :], V[..., n0 - L + j:n1 - L + j, :])
    dz = A * (da - (A * da).sum(axis=-1, keepdims=True))
    dQ, dK, dV = np.zeros_like(Q), np.zeros_like(K), np.zeros_like(V)
    for j in range(W):
        n0, n1 = max(0, L - j), min(T, T + L - j)
        if n0 >= n1:
            continue
        u0, u1 = n0 - L + j, n1 - L + j
        dQ[..., n0:n1, :] += s * dz[..., n0:n1, j, None] * K[..., u0:u1, :]
        dK[..., u0:u1, :] += s * dz[..., n0:n1, j, None] * Q[..., n0:n1, :]
        dV[..., u0:u1, :] += A[..., n0:n1, j, None] * dO[..., n0:n1, :]
    return dQ, dK, dV
