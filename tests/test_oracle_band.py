"""Pins for the stored-band oracle functions (oracle.sa.sa_band_probs / sa_backward_band,
the paper's N_T x (A+B+1) a_t matrix; NEXT-4) against things other than
themselves: closed forms (identical keys -> uniform weights over the clipped window; the
clipped count of SURVEY App. A), the row-sum invariant, brute-force softmax loops, the dense
chain rule (oracle.sa.sa_backward, a different computation), torch autograd and finite
differences."""
import numpy as np
import pytest
import torch

import synth
from oracle import counts, sa as osa


def _inputs(seed, B, H, T, D):
    return synth.qkv(seed, (B, H, T, D), "f32")


@pytest.mark.parametrize("T,L,R", [(13, 3, 2), (9, 0, 0), (7, 6, 6), (20, 5, 0), (6, 0, 9)])
def test_band_rows_are_softmax_rows(T, L, R):
    q, k, _ = _inputs(1, 1, 2, T, 4)
    A = osa.sa_band_probs(q, k, L, R)
    W = L + R + 1
    assert A.shape == (1, 2, T, W)
    np.testing.assert_allclose(A.sum(-1), 1.0, atol=1e-13)
    assert (A >= 0).all()
    # zero exactly where the key t-L+j is clipped away (G2)
    t = np.arange(T)[:, None]
    u = t - L + np.arange(W)[None, :]
    assert (A[..., (u < 0) | (u >= T)] == 0).all()
    # nonzero count = the clipped score count (closed form, oracle.counts / SURVEY App. A)
    assert int((A[0, 0] > 0).sum()) == counts.sa_score_elements(T, L, R)


def test_band_identical_keys_uniform():
    # k_u all equal -> every in-window score equal -> a_tj = 1 / |clipped window|
    T, L, R = 11, 3, 2
    q, k, _ = _inputs(2, 1, 1, T, 8)
    k[:] = k[..., :1, :]
    A = osa.sa_band_probs(q, k, L, R)
    for t in range(T):
        n = min(T - 1, t + R) - max(0, t - L) + 1
        row = A[0, 0, t]
        np.testing.assert_allclose(row[row > 0], 1.0 / n, rtol=1e-14)


def test_band_brute_force_loops():
    T, L, R, D = 10, 2, 3, 3
    q, k, _ = _inputs(3, 1, 1, T, D)
    A = osa.sa_band_probs(q, k, L, R)
    s = 1 / np.sqrt(D)
    for t in range(T):
        keys = [u for u in range(t - L, t + R + 1) if 0 <= u < T]
        z = [s * float(np.dot(q[0, 0, t], k[0, 0, u])) for u in keys]
        e = [np.exp(x - max(z)) for x in z]
        for u, x in zip(keys, e):
            assert abs(A[0, 0, t, u - t + L] - x / sum(e)) < 1e-14


@pytest.mark.parametrize("T,L,R", [(17, 4, 2), (9, 0, 0), (8, 7, 7), (12, 0, 3), (30, 6, 1)])
def test_band_backward_equals_dense_chain_rule(T, L, R):
    q, k, v = _inputs(4, 2, 1, T, 6)
    do = synth.qkv(5, (2, 1, T, 6), "f32")[0]
    A = osa.sa_band_probs(q, k, L, R)
    got = osa.sa_backward_band(A, q, k, v, do, L, R)
    want = osa.sa_backward(q, k, v, do, L, R)
    for g, w in zip(got, want):
        np.testing.assert_allclose(g, w, atol=1e-12, rtol=0)


def test_band_backward_matches_autograd():
    T, L, R, D = 15, 3, 2, 4
    q, k, v = (torch.from_numpy(x).requires_grad_() for x in _inputs(6, 1, 2, T, D))
    do = torch.from_numpy(synth.qkv(7, (1, 2, T, D), "f32")[0])
    i = torch.arange(T)
    band = (i[None, :] >= i[:, None] - L) & (i[None, :] <= i[:, None] + R)
    y = torch.nn.functional.scaled_dot_product_attention(q, k, v, attn_mask=band)
    (y * do).sum().backward()
    A = osa.sa_band_probs(q.detach().numpy(), k.detach().numpy(), L, R)
    got = osa.sa_backward_band(A, q.detach().numpy(), k.detach().numpy(), v.detach().numpy(), do.numpy(), L, R)
    for g, w in zip(got, (q.grad, k.grad, v.grad)):
        np.testing.assert_allclose(g, w.numpy(), atol=1e-12, rtol=0)


def test_band_backward_dv_is_linear_in_band():
    # dv depends on A only: scaling the band by 2 doubles dv (a dropped or doubled term fails)
    T, L, R = 12, 2, 2
    q, k, v = _inputs(8, 1, 1, T, 4)
    do = synth.qkv(9, (1, 1, T, 4), "f32")[0]
    A = osa.sa_band_probs(q, k, L, R)
    _, _, dv1 = osa.sa_backward_band(A, q, k, v, do, L, R)
    _, _, dv2 = osa.sa_backward_band(2 * A, q, k, v, do, L, R)
    np.testing.assert_allclose(dv2, 2 * dv1, atol=1e-13)
