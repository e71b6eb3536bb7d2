"""Pins for oracle.llsa (Eq. 14-16, Fig. 3(c)): reduction to SA, the duplication
identity (ties LLSA to the dense SA definition), the paper's Fig. 3(c) window,
an independent flattened-mask formulation, finite differences, invariants and
the support of Eq. 16."""
import itertools
import json
import os

import numpy as np
import pytest

import synth
from oracle import llsa as oll
from oracle import sa as osa

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def _chan_inputs(seed, C, B, H, T, D):
    return synth.qkv(seed, (C, B, H, T, D), "f32")


def test_zero_lookahead_reduces_to_sa():
    q, k, v = _chan_inputs(0, 1, 1, 2, 15, 4)
    O, LSE = oll.llsa_forward(q, k, v, 4, 0)
    Os, LSEs = osa.sa_forward(q[0], k[0], v[0], 4, 0)
    np.testing.assert_allclose(O[0], Os, atol=1e-12)
    np.testing.assert_allclose(LSE[0], LSEs, atol=1e-12)


@pytest.mark.parametrize("T,L,R", [(14, 2, 3), (16, 3, 1), (20, 4, 4), (9, 0, 2), (6, 5, 3)])
def test_duplication_identity_forward(T, L, R):
    # layer-1 (duplicated) channels: channel c == SA with band (L+R-c, c)
    x, _, _ = synth.qkv(1, (1, 2, T, 3), "f32")
    X = oll.channelize(x, R)
    O, _ = oll.llsa_forward(X, X, X, L, R)
    for c in range(R + 1):
        Os, _ = osa.sa_forward(x, x, x, L + R - c, c)
        np.testing.assert_allclose(O[c], Os, atol=1e-12, rtol=0)


def test_duplication_identity_backward():
    T, L, R = 13, 2, 2
    q, k, v = synth.qkv(2, (1, 1, T, 3), "f32")
    Q, K, V = (oll.channelize(x, R) for x in (q, k, v))
    dO = synth.grad_out(2, Q.shape)
    dQ, dK, dV = oll.llsa_backward(Q, K, V, dO, L, R)
    sk = np.zeros_like(k)
    sv = np.zeros_like(v)
    for c in range(R + 1):
        dq, dk, dv = osa.sa_backward(q, k, v, dO[c], L + R - c, c)
        np.testing.assert_allclose(dQ[c], dq, atol=1e-12)
        sk += dk
        sv += dv
    # the duplicated keys' gradients summed over channels equal the per-band sums
    np.testing.assert_allclose(dK.sum(0), sk, atol=1e-12)
    np.testing.assert_allclose(dV.sum(0), sv, atol=1e-12)


def test_fig3c_window_structure():
    g = GOLD["llsa_fig3c_window"]
    L, R, T, t = g["B"], g["A"], 20, 10
    slots = oll.window_slots(t, g["query_c"], T, L, R)
    assert [u - t for u, _ in slots] == g["slots_rel_frame"]
    assert [ch for _, ch in slots] == g["slots_channel"]
    wins = [sorted(oll.window_slots(t + dt, c, T, L, R)) for dt, c in g["same_window_outputs_rel"]]
    assert all(w == wins[0] for w in wins)


@pytest.mark.parametrize("T,L,R", [(12, 2, 2), (10, 3, 1), (9, 1, 3), (7, 0, 2)])
def test_gather_form_equals_flattened_horizon_mask(T, L, R):
    C = R + 1
    q, k, v = _chan_inputs(3, C, 1, 2, T, 3)
    dO = synth.grad_out(3, q.shape)
    O, _ = oll.llsa_forward(q, k, v, L, R)
    np.testing.assert_allclose(O, oll.llsa_forward_flat(q, k, v, L, R), atol=1e-12)
    for a, b in zip(oll.llsa_backward(q, k, v, dO, L, R), oll.llsa_backward_flat(q, k, v, dO, L, R)):
        np.testing.assert_allclose(a, b, atol=1e-12)


def test_backward_matches_central_differences():
    T, L, R, D = 6, 1, 2, 3
    C = R + 1
    q, k, v = _chan_inputs(4, C, 1, 1, T, D)
    dO = synth.grad_out(4, q.shape)
    g = oll.llsa_backward(q, k, v, dO, L, R)

    def loss(*xs):
        return float((oll.llsa_forward(*xs, L, R)[0] * dO).sum())

    h = 1e-6
    worst = 0.0
    for which in range(3):
        for i in itertools.product(range(C), range(T), range(D)):
            xs = [q.copy(), k.copy(), v.copy()]
            ix = (i[0], 0, 0, i[1], i[2])
            xs[which][ix] += h
            lp = loss(*xs)
            xs[which][ix] -= 2 * h
            fd = (lp - loss(*xs)) / (2 * h)
            worst = max(worst, abs(fd - g[which][ix]) / max(1.0, abs(fd)))
    assert worst < 1e-5, worst


def test_backward_invariants():
    T, L, R = 30, 4, 3
    q, k, v = _chan_inputs(5, R + 1, 1, 2, T, 4)
    dO = synth.grad_out(5, q.shape)
    dq, dk, dv = oll.llsa_backward(q, k, v, dO, L, R)
    ax = (0, -2)  # all slots (channels x frames)
    assert np.abs(dk.sum(axis=ax)).max() < 1e-12
    assert np.abs(dv.sum(axis=ax) - dO.sum(axis=ax)).max() < 1e-12
    assert abs((dq * q).sum() - (dk * k).sum()) < 1e-11


def test_eq16_support():
    # dV_{t,c2} receives dy_{n,c1} only for n in [t-A+c2, t+B+c2] (Eq. 16, P:L274-277;
    # paper letters A = R look-ahead, B = L look-back); tight for c2 = R (reading G8)
    T, L, R = 16, 3, 2
    C = R + 1
    q, k, v = _chan_inputs(6, C, 1, 1, T, 3)
    dO = synth.grad_out(6, q.shape)
    _, _, dv = oll.llsa_backward(q, k, v, dO, L, R)
    for n, c1 in itertools.product((6, 9), range(C)):
        dO2 = dO.copy()
        dO2[c1, 0, 0, n] += 1.0
        _, _, dv2 = oll.llsa_backward(q, k, v, dO2, L, R)
        changed = np.abs(dv2 - dv)[:, 0, 0].max(-1) > 0      # [C, T]
        for c2, t in itertools.product(range(C), range(T)):
            if changed[c2, t]:
                assert t - R + c2 <= n <= t + L + c2, (n, c1, c2, t)
    # tightness for c2 = R: every n in the range feeds dV_{t,R} through some c1
    t = 8
    feeds = set()
    for n, c1 in itertools.product(range(T), range(C)):
        dO2 = dO.copy()
        dO2[c1, 0, 0, n] += 1.0
        _, _, dv2 = oll.llsa_backward(q, k, v, dO2, L, R)
        if np.abs(dv2 - dv)[R, 0, 0, t].max() > 0:
            feeds.add(n)
    assert feeds == set(range(t - R + R, t + L + R + 1))


def test_per_output_causality_contract_one_layer():
    # output (t, c) depends on input frames <= t + c only (c = look-ahead used)
    T, L, R = 14, 2, 3
    x, _, _ = synth.qkv(7, (1, 1, T, 3), "f32")
    X = oll.channelize(x, R)
    O, _ = oll.llsa_forward(X, X, X, L, R)
    for s in range(T):
        x2 = x.copy()
        x2[0, 0, s] += 0.5
        X2 = oll.channelize(x2, R)
        O2, _ = oll.llsa_forward(X2, X2, X2, L, R)
        ch = np.abs(O2 - O)[:, 0, 0].max(-1) > 0
        for c, t in zip(*np.nonzero(ch)):
            assert s <= t + c
