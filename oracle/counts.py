"""Oracle: score-element counts (P:L85-87 MAA example; P:L337 / P:L342 SA bounds).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Counts are obtained by
counting mask entries / window slots, not by a closed form (the closed forms
live in the tests as pins).
"""
from __future__ import annotations

import numpy as np

from .sa import band_mask
from .llsa import window_slots


def maa_score_elements(T: int) -> int:
    """MAA computes all N_T^2 scores ("O(d_k N_T^2)")."""
    return T * T


def sa_score_elements(T: int, L: int, R: int) -> int:
    """Scores SA actually computes: the True entries of the clipped band (Eq. 4)."""
    return int(band_mask(T, L, R).sum())


def sa_score_elements_unclipped(T: int, L: int, R: int) -> int:
    """N_T x (A+B+1), the size of SA's z_t / a_t store."""
    return T * (L + R + 1)


def llsa_score_elements(T: int, L: int, R: int) -> int:
    """sum over outputs (t, c) of |window(t, c)| (Eq. 14, clipped)."""
    return sum(len(window_slots(t, c, T, L, R)) for t in range(T) for c in range(R + 1))
