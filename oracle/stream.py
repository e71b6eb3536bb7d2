"""Oracle: per-frame incremental LLSA inference (infer_llsa).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  numpy fp64.

Written as its own recurrence (no call into oracle.llsa / oracle.stack), so the
online == offline equality is a real cross-check.  At step h (frame x_h
arrives), every layer computes the R+1 outputs of horizon h, (h-c, c) for
c = 0..R.  Per Eq. 14 read as in oracle.llsa (G6) those all share one window:
channel-R slots (u, R), u in [h-R-L, h-R], and the diagonal (h-c', c'),
c' = 0..R-1 ("the same keys and values of the red vector are used").
Everything but the diagonal was produced at earlier steps, so each layer keeps
a ring of its input's channel-R frames for the last L frames; this is why the
latency does not build up.  The stack block is the tied-QKV
X_{l+1} = (X_l + Y_l)/2 rule of oracle.stack (G12); layer 1 sees every channel
equal to x.  The designated output is channel R of the last layer, so
frame h-R is emitted at step h (latency R frames).  flush() runs the R
remaining horizons with windows clipped at the last frame.
"""
from __future__ import annotations

import numpy as np


class LLSAStream:
    def __init__(self, L: int, R: int, n_layers: int, scale: float | None = None):
        self.L, self.R, self.n_layers = L, R, n_layers
        self.scale = scale
        self.raw = {}                                    # x_u, last R+1 frames
        self.hist = [dict() for _ in range(n_layers)]    # hist[l][u] = X_l(u, R), last L frames
        self.h = 0                                       # next horizon to run
        self.n_in = 0                                    # frames pushed
        self.closed = False

    def state_frames(self):
        """Retained frames (bounded by R+1 + n_layers*L, independent of stream length)."""
        return len(self.raw) + sum(len(d) for d in self.hist)

    def _horizon(self, h: int, last: int):
        L, R = self.L, self.R
        diag = {cp: self.raw[h - cp] for cp in range(R + 1) if 0 <= h - cp <= last}
        for l in range(self.n_layers):
            hist = self.hist[l]
            out = {}
            for c in range(R + 1):
                t = h - c
                if t < 0 or t > last:
                    continue
                q = diag[c]
                kv = []
                for i in range(L + R + 1):
                    u = h - R - L + i
                    if u < 0 or u > last:
                        continue
                    if i <= L:
                        kv.append(hist[u] if u < h - R else diag[R])   # slot (u, R)
                    else:
                        kv.append(diag[L + R - i])                     # slot (u, L+R-i)
                kw = np.stack(kv, axis=-2)                              # [..., n, D]
                D = q.shape[-1]
                s = 1.0 / np.sqrt(D) if not self.scale else self.scale
                z = np.einsum("...d,...nd->...n", q, kw) * s
                a = np.exp(z - z.max(axis=-1, keepdims=True))
                a = a / a.sum(axis=-1, keepdims=True)
                y = np.einsum("...n,...nd->...d", a, kw)
                out[c] = 0.5 * (q + y)
            if R in diag:                       # X_l(h-R, R) joins the ring
                hist[h - R] = diag[R]
            for u in [u for u in hist if u < h + 1 - R - L]:
                del hist[u]
            diag = out
        return diag.get(R)                      # X_n(h-R, R) or None

    def push(self, x):
        """Ingest frame x [..., D]; returns (frame index, designated output) or None."""
        assert not self.closed
        h = self.n_in
        self.raw[h] = np.asarray(x, dtype=np.float64)
        self.n_in += 1
        for u in [u for u in self.raw if u < h - self.R]:
            del self.raw[u]
        y = self._horizon(h, last=h)
        self.h = h + 1
        return None if y is None else (h - self.R, y)

    def flush(self):
        """Run the remaining horizons h = T .. T+R-1 (T = frames pushed); returns [(frame, y)]."""
        self.closed = True
        T = self.n_in
        outs = []
        for h in range(T, T + self.R):
            y = self._horizon(h, last=T - 1)
            if y is not None:
                outs.append((h - self.R, y))
        return outs


def stream_all(X, L: int, R: int, n_layers: int, scale=None):
    """Push every frame of X [..., T, D] then flush; returns the designated output [..., T, D]
    and the push index at which each frame was emitted."""
    X = np.asarray(X, dtype=np.float64)
    T = X.shape[-2]
    st = LLSAStream(L, R, n_layers, scale)
    Y = np.full(X.shape, np.nan)
    emitted_at = np.full(T, -1)
    for h in range(T):
        r = st.push(X[..., h, :])
        if r is not None:
            Y[..., r[0], :] = r[1]
            emitted_at[r[0]] = h
    for t, y in st.flush():
        Y[..., t, :] = y
        emitted_at[t] = T
    return Y, emitted_at


class SAStream:
    """Incremental SA inference (infer_sa) — its own recurrence.

    Layer l (0-based) of an SA stack can emit frame t only once its input holds frame t + R
    (Eq. 4's look-ahead), and its input frame t + R is itself layer l-1's output at that frame.
    So after frame h arrives, layer l computes t_l = h - (l+1) R from the window
    [t_l - L, t_l + R] of its input, and the stack emits X_n(h - n R): the latency builds up to
    n_layers x R frames (Table 3's infer_sa).  Each layer keeps the last L + R + 1
    frames of its input; the block rule is oracle.stack's tied-QKV X_{l+1} = (X_l + Y_l)/2 (G12).
    flush() runs h = T .. T - 1 + n R with every window clipped at the last frame."""

    def __init__(self, L: int, R: int, n_layers: int, scale: float | None = None):
        self.L, self.R, self.n_layers = L, R, n_layers
        self.scale = scale
        self.X = [dict() for _ in range(n_layers + 1)]   # X[l][u] = input frame u of layer l (X[n]: output)
        self.n_in = 0
        self.closed = False

    def state_frames(self):
        """Retained frames (bounded by n_layers (L + R + 1), independent of the stream length)."""
        return sum(len(d) for d in self.X[:-1])

    def _step(self, h: int, last: int):
        L, R = self.L, self.R
        for l in range(self.n_layers):
            t = h - (l + 1) * R
            if t < 0 or t > last:
                continue
            X = self.X[l]
            us = [u for u in range(t - L, t + R + 1) if 0 <= u <= last]
            kw = np.stack([X[u] for u in us], axis=-2)
            q = X[t]
            D = q.shape[-1]
            s = 1.0 / np.sqrt(D) if not self.scale else self.scale
            z = np.einsum("...d,...nd->...n", q, kw) * s
            a = np.exp(z - z.max(axis=-1, keepdims=True))
            a = a / a.sum(axis=-1, keepdims=True)
            y = np.einsum("...n,...nd->...d", a, kw)
            self.X[l + 1][t] = 0.5 * (q + y)
            for u in [u for u in X if u < t + 1 - L]:    # frame t - L leaves every later window
                del X[u]
        t = h - self.n_layers * R
        out = self.X[self.n_layers].pop(t, None) if 0 <= t <= last else None
        return out

    def push(self, x):
        """Ingest frame x [..., D]; returns (frame index, stack output) or None."""
        assert not self.closed
        h = self.n_in
        self.X[0][h] = np.asarray(x, dtype=np.float64)
        self.n_in += 1
        y = self._step(h, last=h)
        return None if y is None else (h - self.n_layers * self.R, y)

    def flush(self):
        """Run h = T .. T - 1 + n_layers R (T = frames pushed); returns [(frame, y)]."""
        self.closed = True
        T = self.n_in
        outs = []
        for h in range(T, T + self.n_layers * self.R):
            y = self._step(h, last=T - 1)
            if y is not None:
                outs.append((h - self.n_layers * self.R, y))
        return outs


def sa_stream_all(X, L: int, R: int, n_layers: int, scale=None):
    """Push every frame of X [..., T, D] through SAStream, then flush; returns the stack output
    [..., T, D] and the push index at which each frame was emitted."""
    X = np.asarray(X, dtype=np.float64)
    T = X.shape[-2]
    st = SAStream(L, R, n_layers, scale)
    Y = np.full(X.shape, np.nan)
    emitted_at = np.full(T, -1)
    for h in range(T):
        r = st.push(X[..., h, :])
        if r is not None:
            Y[..., r[0], :] = r[1]
            emitted_at[r[0]] = h
    for t, y in st.flush():
        Y[..., t, :] = y
        emitted_at[t] = T
    return Y, emitted_at
