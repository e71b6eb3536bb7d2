"""Pins for oracle.stack, oracle.stream, oracle.latency and oracle.counts:
finite differences through the stack, the paper's latency figures (Fig. 3(b),
Table 3), structural and numeric (witness) latency, online == offline
streaming, and the P:L87 worked example."""
import itertools
import json
import os

import numpy as np
import pytest

import synth
from oracle import counts, latency, stack, stream
from oracle import llsa as oll

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


@pytest.mark.parametrize("mode", ["sa", "llsa"])
def test_stack_backward_central_differences(mode):
    T, L, R, D, n = 7, 2, 1, 3, 2
    x = synth.normal(0, "X", (1, 1, T, D))
    shape = ((R + 1,) if mode == "llsa" else ()) + x.shape
    dY = synth.normal(0, "dY", shape)
    g = stack.stack_backward(x, dY, L, R, n, mode)

    def loss(x_):
        return float((stack.stack_forward(x_, L, R, n, mode)[0] * dY).sum())

    h = 1e-6
    for i in itertools.product(range(T), range(D)):
        xp = x.copy()
        xp[(0, 0) + i] += h
        xm = x.copy()
        xm[(0, 0) + i] -= h
        fd = (loss(xp) - loss(xm)) / (2 * h)
        assert abs(fd - g[(0, 0) + i]) <= 1e-6 * max(1.0, abs(fd))


def test_fig3b_two_sa_layers_latency_four():
    g = GOLD["sa_stack_latency_fig3b"]
    T = 30
    assert latency.structural_lookahead("sa", T, g["B"], g["A"], g["layers"]) == g["latency_frames"]
    assert latency.latency_frames("sa", g["A"], g["layers"]) == g["latency_frames"]


@pytest.mark.parametrize("L,R,n", [(2, 2, 2), (3, 1, 4), (1, 2, 3)])
def test_structural_latency_llsa_channel_c_is_c_at_any_depth(L, R, n):
    T = 3 * (L + R) * n + 4
    assert latency.structural_lookahead("llsa", T, L, R, n) == list(range(R + 1))
    assert latency.structural_lookahead("sa", T, L, R, n) == n * R


def test_table3_latency_column():
    g = GOLD["table3_latency"]
    for row in g["rows"]:
        mode = "sa" if row["infer"] == "infer_sa" else "llsa"
        got = latency.latency_seconds(mode, row["R"], g["layers"], g["frame_seconds"])
        assert abs(got - row["latency_s"]) < 1e-12, row


@pytest.mark.slow
@pytest.mark.parametrize("R", [8, 16])
def test_witness_probe_12_layers(R):
    # numeric probe, fp64: SA (masked-acausal) stack latency 12R, LLSA designated latency R
    L, n, T, D, tau = 32, 12, 300, 8, 250
    x = synth.witness(0, 1, 1, T, D)
    x2 = x.copy()
    x2[0, 0, tau] += 0.5
    ysa = stack.stack_forward(x, L, R, n, "sa")[0]
    ysa2 = stack.stack_forward(x2, L, R, n, "sa")[0]
    assert tau - latency.earliest_changed(ysa, ysa2) == n * R
    yl = stack.stack_forward(x, L, R, n, "llsa")[0][R]
    yl2 = stack.stack_forward(x2, L, R, n, "llsa")[0][R]
    assert tau - latency.earliest_changed(yl, yl2) == R


def test_witness_probe_small():
    L, R, n, T, D, tau = 3, 2, 4, 60, 4, 45
    x = synth.witness(1, 1, 1, T, D)
    x2 = x.copy()
    x2[0, 0, tau] += 0.5
    ysa = stack.stack_forward(x, L, R, n, "sa")[0]
    assert tau - latency.earliest_changed(ysa, stack.stack_forward(x2, L, R, n, "sa")[0]) == n * R
    yl = stack.stack_forward(x, L, R, n, "llsa")[0]
    yl2 = stack.stack_forward(x2, L, R, n, "llsa")[0]
    for c in range(R + 1):
        assert tau - latency.earliest_changed(yl[c], yl2[c]) == c


@pytest.mark.parametrize("L,R,n,T", [(3, 2, 3, 25), (2, 1, 2, 16), (4, 3, 2, 11), (3, 0, 2, 9), (5, 4, 3, 6)])
def test_stream_online_equals_offline(L, R, n, T):
    x = synth.normal(2, "X", (2, 3, T, 4))
    y_off = stack.stack_forward(x, L, R, n, "llsa")[0][R]
    y_on, emitted_at = stream.stream_all(x, L, R, n)
    np.testing.assert_allclose(y_on, y_off, atol=1e-12, rtol=0)
    # frame t is emitted at push t+R (first emission after R+1 pushes), the tail at flush
    np.testing.assert_array_equal(emitted_at, np.minimum(np.arange(T) + R, T))


def test_stream_state_is_bounded():
    L, R, n, T = 4, 2, 3, 80
    st = stream.LLSAStream(L, R, n)
    peak = 0
    for h in range(T):
        st.push(synth.normal(3, "X", (1, 1, 4), offset=4 * h))
        peak = max(peak, st.state_frames())
    assert peak <= (R + 1) + n * L


def test_maa_worked_example_counts():
    g = GOLD["maa_worked_example"]
    T, W = g["N_T"], g["window"]
    # 120 ones / 5880 zeros per interior mask row (e.g. look-back 111, look-ahead 8)
    L, R = 111, 8
    assert L + R + 1 == g["ones_per_row"] and T - (L + R + 1) == g["zeros_per_row"]
    assert counts.sa_score_elements_unclipped(T, L, R) == g["used"]
    assert counts.maa_score_elements(T) == g["computed"]
    assert counts.maa_score_elements(T) - counts.sa_score_elements_unclipped(T, L, R) == g["dummy_replacements"]


@pytest.mark.parametrize("T,L,R,expect", [(6000, 111, 8, 713748), (1750, 32, 8, 71186), (16, 3, 1, 73)])
def test_clipped_count_closed_form(T, L, R, expect):
    assert counts.sa_score_elements(T, L, R) == expect
    assert expect == T * (L + R + 1) - L * (L + 1) // 2 - R * (R + 1) // 2


def test_llsa_extra_compute_ratio():
    # P:L417 "extra A times more computations": (R+1) windows of W slots per frame
    T, L, R = 200, 32, 8
    n_llsa = counts.llsa_score_elements(T, L, R)
    assert n_llsa <= (R + 1) * counts.sa_score_elements_unclipped(T, L, R)
    # interior frames: exactly (R+1) * W
    interior = sum(len(oll.window_slots(t, c, T, L, R)) for t in range(50, 150) for c in range(R + 1))
    assert interior == 100 * (R + 1) * (L + R + 1)


# ---- infer_sa (NEXT-2): the SA stack run incrementally; latency n_layers x R (Table 3)
@pytest.mark.parametrize("L,R,n,T", [(3, 1, 2, 16), (4, 2, 3, 40), (0, 3, 2, 25), (5, 0, 3, 20), (6, 2, 1, 9),
                                     (5, 4, 3, 7), (2, 3, 4, 5)])  # T < n R: every output from the flush
def test_sa_stream_online_equals_offline(L, R, n, T):
    x = synth.normal(4, "X", (2, 3, T, 4))
    y_off = stack.stack_forward(x, L, R, n, "sa")[0]
    y_on, emitted_at = stream.sa_stream_all(x, L, R, n)
    np.testing.assert_allclose(y_on, y_off, atol=1e-12, rtol=0)
    # frame t is emitted at push t + n R (latency builds up with depth), the tail at flush
    np.testing.assert_array_equal(emitted_at, np.minimum(np.arange(T) + n * R, T))


def test_sa_stream_state_is_bounded():
    L, R, n, T = 4, 2, 3, 80
    st = stream.SAStream(L, R, n)
    peak = 0
    for h in range(T):
        st.push(synth.normal(5, "X", (1, 1, 4), offset=4 * h))
        peak = max(peak, st.state_frames())
    assert peak <= n * (L + R + 1)
