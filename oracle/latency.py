"""Oracle: latency of stacked SA / masked-acausal vs LLSA layers (Table 3).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* latency_frames / latency_seconds: the Table 3 arithmetic.  SA (and MAA, which
  has the same receptive field) adds R frames per layer: "2 layers x 2 frames =
  four frames".  LLSA keeps R frames at any depth.  Frame
  period 20 ms and 12 layers are the reading G13 (1.92 s / (8 * 20 ms) = 12).
* structural_lookahead: exact receptive-field propagation, dep_{l+1}(slot) =
  union of dep_l over the slot's window (Eq. 4 / Eq. 14 windows), starting from
  dep_0(t, c) = {t} (layer-1 duplication).  Returns, per output channel,
  the largest (input frame - output frame) any output depends on.
"""
from __future__ import annotations

import numpy as np

from .sa import band_mask
from .llsa import window_slots

FRAME_SECONDS = 0.020   # 50 Hz frames (G13)


def latency_frames(mode: str, R: int, n_layers: int) -> int:
    if mode in ("sa", "maa"):
        return n_layers * R
    if mode == "llsa":
        return R
    raise ValueError(mode)


def latency_seconds(mode: str, R: int, n_layers: int, frame_s: float = FRAME_SECONDS) -> float:
    return latency_frames(mode, R, n_layers) * frame_s


def structural_lookahead(mode: str, T: int, L: int, R: int, n_layers: int):
    """SA: int.  LLSA: list over output channels c = 0..R."""
    if mode == "sa":
        W = band_mask(T, L, R).astype(np.int64)
        dep = np.eye(T, dtype=np.int64)
        for _ in range(n_layers):
            dep = ((W @ dep) > 0).astype(np.int64)
        u = np.arange(T)
        last = np.where(dep.any(axis=1), (dep * u[None, :]).max(axis=1), -1)
        return int((last - np.arange(T)).max())
    if mode == "llsa":
        C = R + 1
        n = T * C
        W = np.zeros((n, n), dtype=np.int64)
        for t in range(T):
            for c in range(C):
                for (u, ch) in window_slots(t, c, T, L, R):
                    W[t * C + c, u * C + ch] = 1
        dep = np.zeros((n, T), dtype=np.int64)        # dep_0(t, c) = {t}
        for t in range(T):
            dep[t * C:(t + 1) * C, t] = 1
        for _ in range(n_layers):
            dep = ((W @ dep) > 0).astype(np.int64)
        u = np.arange(T)
        last = (dep * u[None, :]).max(axis=1)
        t_of = np.repeat(np.arange(T), C)
        ahead = last - t_of
        return [int(ahead[c::C].max()) for c in range(C)]
    raise ValueError(mode)


def earliest_changed(Y0, Y1, atol: float = 0.0):
    """Smallest frame index t whose output row differs (|diff| > atol) between two
    [..., T, D] outputs; -1 if none.  Used by the numeric witness probe."""
    d = np.abs(np.asarray(Y1, dtype=np.float64) - np.asarray(Y0, dtype=np.float64))
    d = d.reshape(-1, d.shape[-2], d.shape[-1]).max(axis=(0, 2))
    idx = np.nonzero(d > atol)[0]
    return int(idx[0]) if idx.size else -1
