"""Pins for oracle.sa (SA / MAA / AA, Eq. 1-13) against things other than itself:
library SDPA (torch fp64), brute-force loops of Eq. 4-6, closed-form special
cases, finite differences, torch autograd and invariants."""
import itertools

import numpy as np
import pytest
import torch

import synth
from oracle import sa as osa


def _inputs(seed, B, H, T, D):
    return synth.qkv(seed, (B, H, T, D), "f32")


def _torch_sdpa(q, k, v, causal=False):
    t = [torch.from_numpy(x) for x in (q, k, v)]
    return torch.nn.functional.scaled_dot_product_attention(*t, is_causal=causal).numpy()


def test_band_covering_everything_is_acausal_attention():
    # SA with L, R >= T-1 equals AA (Eq. 1-2) -- library SDPA, fp64, no mask.
    q, k, v = _inputs(0, 2, 3, 11, 5)
    O, _ = osa.sa_forward(q, k, v, 10, 10)
    np.testing.assert_allclose(O, _torch_sdpa(q, k, v), atol=1e-12, rtol=0)
    np.testing.assert_allclose(osa.aa_forward(q, k, v), O, atol=1e-12, rtol=0)


def test_zero_lookahead_full_lookback_is_causal_attention():
    q, k, v = _inputs(1, 1, 2, 13, 4)
    O, _ = osa.sa_forward(q, k, v, 12, 0)
    np.testing.assert_allclose(O, _torch_sdpa(q, k, v, causal=True), atol=1e-12, rtol=0)


def test_window_of_one_returns_values_exactly():
    q, k, v = _inputs(2, 1, 1, 9, 3)
    O, LSE = osa.sa_forward(q, k, v, 0, 0)
    assert np.array_equal(O, v)
    dq, dk, dv = osa.sa_backward(q, k, v, synth.grad_out(2, v.shape), 0, 0)
    assert np.all(dq == 0) and np.all(dk == 0)
    np.testing.assert_array_equal(dv, synth.grad_out(2, v.shape))
    # LSE of a single score is the score itself
    np.testing.assert_allclose(LSE, (q * k).sum(-1) / np.sqrt(3), atol=1e-14)


def test_single_frame_returns_value():
    q, k, v = _inputs(3, 1, 1, 1, 4)
    O, _ = osa.sa_forward(q, k, v, 5, 7)
    assert np.array_equal(O, v)


def test_identical_keys_give_window_mean_of_values():
    T, L, R = 12, 3, 2
    q, k, v = _inputs(4, 1, 1, T, 4)
    k[...] = k[..., :1, :]
    O, _ = osa.sa_forward(q, k, v, L, R)
    for t in range(T):
        lo, hi = max(0, t - L), min(T - 1, t + R)
        np.testing.assert_allclose(O[0, 0, t], v[0, 0, lo:hi + 1].mean(0), atol=1e-13)


def _brute_force(q, k, v, L, R):
    """Eq. 4-6 written as scalar loops over j = -B..A (paper letters), clipped."""
    T, D = q.shape
    y = np.zeros((T, D))
    lse = np.zeros(T)
    for t in range(T):
        js = [j for j in range(-L, R + 1) if 0 <= t + j < T]
        z = [sum(k[t + j][d] * q[t][d] for d in range(D)) / np.sqrt(D) for j in js]
        m = max(z)
        e = [np.exp(x - m) for x in z]
        s = sum(e)
        a = [x / s for x in e]
        for i, j in enumerate(js):
            for d in range(D):
                y[t][d] += v[t + j][d] * a[i]
        lse[t] = m + np.log(s)
    return y, lse


@pytest.mark.parametrize("T,L,R", [(16, 3, 1), (9, 0, 4), (9, 4, 0), (7, 8, 8), (10, 2, 2)])
def test_forward_matches_brute_force_loops(T, L, R):
    q, k, v = _inputs(5, 1, 1, T, 4)
    O, LSE = osa.sa_forward(q, k, v, L, R)
    y, lse = _brute_force(q[0, 0], k[0, 0], v[0, 0], L, R)
    np.testing.assert_allclose(O[0, 0], y, atol=1e-12, rtol=0)
    np.testing.assert_allclose(LSE[0, 0], lse, atol=1e-12, rtol=0)


def test_forward_locality_exact_zero():
    # perturbing key/value frame s changes O_t iff t-L <= s <= t+R
    T, L, R = 20, 3, 2
    q, k, v = _inputs(6, 1, 1, T, 4)
    O, _ = osa.sa_forward(q, k, v, L, R)
    for s in (0, 7, 19):
        k2, v2 = k.copy(), v.copy()
        k2[0, 0, s] += 0.3
        v2[0, 0, s] -= 0.7
        O2, _ = osa.sa_forward(q, k2, v2, L, R)
        changed = np.abs(O2 - O)[0, 0].max(-1) > 0
        expect = np.array([t - L <= s <= t + R for t in range(T)])
        assert np.array_equal(changed, expect), s


def test_convex_hull():
    T, L, R = 25, 4, 3
    q, k, v = _inputs(7, 1, 2, T, 3)
    O, _ = osa.sa_forward(q, k, v, L, R)
    for h in range(2):
        for t in range(T):
            w = v[0, h, max(0, t - L):min(T, t + R + 1)]
            assert np.all(O[0, h, t] >= w.min(0) - 1e-9) and np.all(O[0, h, t] <= w.max(0) + 1e-9)


def _torch_masked_loss_grads(q, k, v, dO, L, R):
    """torch autograd (fp64) on the dense masked form with masked_fill(-inf)."""
    T, D = q.shape[-2:]
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    idx = torch.arange(T)
    mask = (idx[None, :] >= idx[:, None] - L) & (idx[None, :] <= idx[:, None] + R)
    z = (tq @ tk.transpose(-1, -2)) / D ** 0.5
    a = torch.softmax(z.masked_fill(~mask, float("-inf")), dim=-1)
    y = a @ tv
    (y * torch.from_numpy(dO)).sum().backward()
    return tq.grad.numpy(), tk.grad.numpy(), tv.grad.numpy()


@pytest.mark.parametrize("T,L,R", [(16, 3, 1), (8, 1, 2), (12, 0, 3), (10, 9, 9)])
def test_backward_matches_torch_autograd(T, L, R):
    q, k, v = _inputs(8, 2, 2, T, 4)
    dO = synth.grad_out(8, q.shape)
    got = osa.sa_backward(q, k, v, dO, L, R)
    ref = _torch_masked_loss_grads(q, k, v, dO, L, R)
    for g, r in zip(got, ref):
        np.testing.assert_allclose(g, r, atol=1e-12, rtol=0)


def test_backward_matches_central_differences():
    T, L, R, D = 8, 2, 1, 3
    q, k, v = _inputs(9, 1, 1, T, D)
    dO = synth.grad_out(9, q.shape)
    dq, dk, dv = osa.sa_backward(q, k, v, dO, L, R)

    def loss(q_, k_, v_):
        return float((osa.sa_forward(q_, k_, v_, L, R)[0] * dO).sum())

    h = 1e-6
    for which, g in ((0, dq), (1, dk), (2, dv)):
        for i in itertools.product(range(T), range(D)):
            xs = [q.copy(), k.copy(), v.copy()]
            xs[which][(0, 0) + i] += h
            lp = loss(*xs)
            xs[which][(0, 0) + i] -= 2 * h
            lm = loss(*xs)
            fd = (lp - lm) / (2 * h)
            assert abs(fd - g[(0, 0) + i]) <= 1e-5 * max(1.0, abs(fd)), (which, i, fd, g[(0, 0) + i])


def test_backward_invariants():
    # sum_u dK_u = 0 (shift all keys); sum dV = sum dO (shift all values);
    # sum <dQ,Q> = sum <dK,K> (Q -> aQ, K -> K/a)
    q, k, v = _inputs(10, 2, 3, 40, 6)
    dO = synth.grad_out(10, q.shape)
    dq, dk, dv = osa.sa_backward(q, k, v, dO, 5, 3)
    assert np.abs(dk.sum(axis=-2)).max() < 1e-12
    assert np.abs(dv.sum(axis=-2) - dO.sum(axis=-2)).max() < 1e-12
    assert np.abs((dq * q).sum(axis=(-1, -2)) - (dk * k).sum(axis=(-1, -2))).max() < 1e-11


def test_backward_dv_locality_eq7_condition():
    # dV_u is fed only by dO_n with n in [u-R, u+L] (Eq. 7's condition, reading G3)
    T, L, R = 18, 3, 1
    q, k, v = _inputs(11, 1, 1, T, 3)
    dO = synth.grad_out(11, q.shape)
    _, _, dv = osa.sa_backward(q, k, v, dO, L, R)
    n = 9
    dO2 = dO.copy()
    dO2[0, 0, n] += 1.0
    _, _, dv2 = osa.sa_backward(q, k, v, dO2, L, R)
    changed = np.abs(dv2 - dv)[0, 0].max(-1) > 0
    expect = np.array([u - R <= n <= u + L for u in range(T)])
    assert np.array_equal(changed, expect)
    # Eq. 8's printed bounds (n in [u-L, u+R]) would differ here since L != R
    assert not np.array_equal(expect, np.array([u - L <= n <= u + R for u in range(T)]))
