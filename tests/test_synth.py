"""The seeded generator is deterministic, counter-based (shape-independent) and
its bf16 rounding agrees with torch's round-to-nearest-even."""
import numpy as np
import torch

import synth


def test_deterministic_and_counter_based():
    a = synth.normal(3, "Q", (4, 5, 6))
    b = synth.normal(3, "Q", (120,))
    assert np.array_equal(a.ravel(), b)
    c = synth.normal(3, "Q", (20,), offset=100)
    assert np.array_equal(b[100:], c)
    assert not np.array_equal(synth.normal(4, "Q", (120,)), b)
    assert not np.array_equal(synth.normal(3, "K", (120,)), b)


def test_normal_moments():
    z = synth.normal(0, 1, (200000,))
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1) < 0.01


def test_bf16_rounding_matches_torch():
    z = synth.normal(1, 2, (10000,)) * 7.3
    ours = synth.round_to(z, "bf16")
    theirs = torch.from_numpy(z.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(ours, theirs)
