"""paper_2302_13451_b200 — SA / LLSA (arXiv 2302.13451) on B200: thin Python binding of libsattn.so.

Every step of the hot path runs in the CUDA kernels behind the C ABI declared in
include/sattn.h; this module only marshals arguments (torch CUDA tensors ->
device pointers, the current CUDA stream) and raises on a non-zero status.
PyTorch is used for device memory and streams only.  There is no CPU fallback:
if libsattn.so is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "SattnError", "lib", "sa_forward", "sa_backward", "sa_forward_p", "sa_backward_p", "llsa_forward", "llsa_backward",
    "stack_forward", "stack_backward", "stack_saved_views", "LLSAStream", "SAFunction", "LLSAFunction", "launch_count",
    "MODE_SA", "MODE_LLSA", "IMPL_AUTO", "IMPL_FFMA", "IMPL_TC",
]

LIB_PATH = os.environ.get("SATTN_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libsattn.so")
F32, BF16 = 0, 1
MODE_SA, MODE_LLSA = 0, 1
IMPL_AUTO, IMPL_FFMA, IMPL_TC = 0, 1, 2
_IMPL = {"auto": IMPL_AUTO, "ffma": IMPL_FFMA, "tc": IMPL_TC}


class SattnError(RuntimeError):
    pass


class Desc(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("H", ctypes.c_int64), ("T", ctypes.c_int64), ("D", ctypes.c_int64),
                ("L", ctypes.c_int32), ("R", ctypes.c_int32), ("dtype", ctypes.c_int32), ("scale", ctypes.c_float),
                ("in_broadcast", ctypes.c_int32), ("impl", ctypes.c_int32)]


_lib = None
_P = ctypes.c_void_p
_SZ = ctypes.c_size_t
_I = ctypes.c_int
_PD = ctypes.POINTER(Desc)

EXPORTS = {
    "sa_forward": (_I, [_PD, _P, _P, _P, _P, _P, _P]),
    "sa_backward_workspace": (_SZ, [_PD]),
    "sa_forward_workspace": (_SZ, [_PD]),
    "sa_forward_ws": (_I, [_PD, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_backward": (_I, [_PD, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_p_ld": (ctypes.c_int64, [_PD]),
    "sa_forward_p": (_I, [_PD, _P, _P, _P, _P, _P, _P, _P]),
    "sa_backward_p_workspace": (_SZ, [_PD]),
    "sa_backward_p": (_I, [_PD, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "llsa_forward": (_I, [_PD, _P, _P, _P, _P, _P, _P]),
    "llsa_backward_workspace": (_SZ, [_PD]),
    "llsa_backward": (_I, [_PD, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "sattn_stack_saved_bytes": (_SZ, [_PD, _I, _I]),
    "sattn_stack_saved_offsets": (_I, [_PD, _I, _I, _I, ctypes.POINTER(ctypes.c_int64)]),
    "sattn_stack_forward": (_I, [_PD, _I, _I, _P, _P, _SZ, _P, _P]),
    "sattn_stack_workspace": (_SZ, [_PD, _I, _I]),
    "sattn_stack_backward": (_I, [_PD, _I, _I, _P, _P, _P, _P, _SZ, _P]),
    "llsa_stream_create": (_I, [_PD, _I, ctypes.POINTER(_P)]),
    "llsa_stream_step": (_I, [_P, _P, _P, ctypes.POINTER(ctypes.c_int64), _P]),
    "llsa_stream_flush": (_I, [_P, _P, ctypes.POINTER(ctypes.c_int32), _P]),
    "llsa_stream_reset": (_I, [_P]),
    "llsa_stream_destroy": (None, [_P]),
    "sa_stream_create": (_I, [_PD, _I, ctypes.POINTER(_P)]),
    "sa_stream_step": (_I, [_P, _P, _P, ctypes.POINTER(ctypes.c_int64), _P]),
    "sa_stream_flush": (_I, [_P, _P, ctypes.POINTER(ctypes.c_int32), _P]),
    "sa_stream_reset": (_I, [_P]),
    "sa_stream_destroy": (None, [_P]),
    "sattn_last_error": (ctypes.c_char_p, []),
    "sattn_version": (ctypes.c_char_p, []),
    "sattn_launch_count": (ctypes.c_int64, []),
}


def lib():
    """Load libsattn.so (built in-tree by __graft_entry__.build()); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SattnError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int, what: str):
    if status != 0:
        raise SattnError(f"{what} failed (status {status}): {lib().sattn_last_error().decode()}")


def launch_count() -> int:
    return int(lib().sattn_launch_count())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return F32
    if t.dtype == torch.bfloat16:
        return BF16
    raise SattnError(f"unsupported dtype {t.dtype} (float32 or bfloat16)")


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise SattnError("tensors must be CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise SattnError("tensors must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def make_desc(B, H, T, D, L, R, dtype, scale=None, in_broadcast=False, impl="auto") -> Desc:
    return Desc(B, H, T, D, L, R, dtype, float(scale or 0.0), int(bool(in_broadcast)), _IMPL[impl])


def _desc_from(q: torch.Tensor, L, R, scale, impl, llsa=False, broadcast=False):
    if llsa and not broadcast:
        C, B, H, T, D = q.shape
        if C != R + 1:
            raise SattnError(f"LLSA tensors need R+1={R + 1} channels, got {C}")
    else:
        B, H, T, D = q.shape
    return make_desc(B, H, T, D, L, R, _dtype_code(q), scale, broadcast, impl)


def _same(ref, *ts):
    for t in ts:
        if t.shape != ref.shape or t.dtype != ref.dtype or t.device != ref.device:
            raise SattnError("Q, K, V (and dO) must share shape, dtype and device")


def _expect(t, shape, dtype, device, name):
    """Shape / dtype / device check of a tensor the kernels index directly (no device-side checks)."""
    if t is None:
        raise SattnError(f"{name} is None")
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != device:
        raise SattnError(f"{name}: expected {tuple(shape)} {dtype} on {device}, got {tuple(t.shape)} {t.dtype} on "
                         f"{t.device}")


# --------------------------------------------------------------------------- SA

def sa_forward(q, k, v, L: int, R: int, scale=None, impl="auto"):
    """SA forward (Eq. 4-6): q, k, v [B, H, T, D] -> (o [B,H,T,D], lse [B,H,T] fp32)."""
    _same(q, k, v)
    d = _desc_from(q, L, R, scale, impl)
    o = torch.empty_like(q)
    lse = torch.empty(q.shape[:-1], device=q.device, dtype=torch.float32)
    nws = lib().sa_forward_workspace(ctypes.byref(d))
    if nws:   # wide bands on tensor cores (sub-bands merged by log-sum-exp)
        ws = torch.empty(nws, device=q.device, dtype=torch.uint8)
        _check(lib().sa_forward_ws(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(ws), nws,
                                   _stream()), "sa_forward_ws")
        return o, lse
    _check(lib().sa_forward(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _stream()), "sa_forward")
    return o, lse


def sa_backward(q, k, v, o, lse, do, L: int, R: int, scale=None, impl="auto", ws=None):
    """SA backward (Eq. 7-13) -> (dq, dk, dv)."""
    _same(q, k, v, o, do)
    _expect(lse, q.shape[:-1], torch.float32, q.device, "lse")
    d = _desc_from(q, L, R, scale, impl)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    nws = lib().sa_backward_workspace(ctypes.byref(d))
    if ws is None or ws.numel() < nws:
        ws = torch.empty(nws, device=q.device, dtype=torch.uint8)
    _check(lib().sa_backward(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(do),
                             _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), nws, _stream()), "sa_backward")
    return dq, dk, dv


def sa_forward_p(q, k, v, L: int, R: int, scale=None, impl="auto"):
    """SA forward that also stores the band of probabilities (the paper's a_t):
    -> (o, lse, p) with p [B, H, T, ld] in q's dtype, p[..., t, j] = a_{t, t-L+j} for
    j < W = L+R+1, zero outside the clipped window and in the padding j >= W."""
    _same(q, k, v)
    d = _desc_from(q, L, R, scale, impl)
    o = torch.empty_like(q)
    lse = torch.empty(q.shape[:-1], device=q.device, dtype=torch.float32)
    ld = int(lib().sa_p_ld(ctypes.byref(d)))
    p = torch.empty(tuple(q.shape[:-1]) + (ld,), device=q.device, dtype=q.dtype)
    _check(lib().sa_forward_p(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(p), _stream()),
           "sa_forward_p")
    return o, lse, p


def sa_backward_p(q, k, v, o, p, do, L: int, R: int, scale=None, impl="auto", ws=None):
    """SA backward from the stored band p of sa_forward_p (no score recompute) -> (dq, dk, dv)."""
    _same(q, k, v, o, do)
    d = _desc_from(q, L, R, scale, impl)
    ld = int(lib().sa_p_ld(ctypes.byref(d)))
    _expect(p, tuple(q.shape[:-1]) + (ld,), q.dtype, q.device, "p (the band of sa_forward_p with the same L, R)")
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    nws = lib().sa_backward_p_workspace(ctypes.byref(d))
    if ws is None or ws.numel() < nws:
        ws = torch.empty(nws, device=q.device, dtype=torch.uint8)
    _check(lib().sa_backward_p(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(p), _ptr(do),
                               _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), nws, _stream()), "sa_backward_p")
    return dq, dk, dv


# ------------------------------------------------------------------------- LLSA

def llsa_forward(q, k, v, L: int, R: int, scale=None, impl="auto", broadcast=False):
    """LLSA forward (Eq. 14-15).  q, k, v: [C=R+1, B, H, T, D] channel-major, or with
    broadcast=True one [B, H, T, D] tensor used as every channel (layer-1 duplication).
    Returns (o [C,B,H,T,D], lse [C,B,H,T])."""
    _same(q, k, v)
    d = _desc_from(q, L, R, scale, impl, llsa=True, broadcast=broadcast)
    C = R + 1
    shp = (C,) + tuple(q.shape[-4:])
    o = torch.empty(shp, device=q.device, dtype=q.dtype)
    lse = torch.empty(shp[:-1], device=q.device, dtype=torch.float32)
    _check(lib().llsa_forward(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _stream()),
           "llsa_forward")
    return o, lse


def llsa_backward(q, k, v, o, lse, do, L: int, R: int, scale=None, impl="auto", broadcast=False, ws=None):
    """LLSA backward (exact gradient; Eq. 16 for dv) -> dense (dq, dk, dv) [C,B,H,T,D]."""
    _same(q, k, v)
    d = _desc_from(q, L, R, scale, impl, llsa=True, broadcast=broadcast)
    shp = (R + 1,) + tuple(q.shape[-4:])
    _expect(o, shp, q.dtype, q.device, "o")
    _expect(do, shp, q.dtype, q.device, "do")
    _expect(lse, shp[:-1], torch.float32, q.device, "lse")
    dq = torch.empty_like(o)
    dk = torch.empty_like(o)
    dv = torch.empty_like(o)
    nws = lib().llsa_backward_workspace(ctypes.byref(d))
    if ws is None or ws.numel() < nws:
        ws = torch.empty(nws, device=q.device, dtype=torch.uint8)
    _check(lib().llsa_backward(ctypes.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(do),
                               _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), nws, _stream()), "llsa_backward")
    return dq, dk, dv


# ------------------------------------------------------------------------ stack

def stack_forward(x0, L: int, R: int, n_layers: int, mode: int = MODE_SA, scale=None, impl="auto"):
    """n-layer tied-QKV stack, X_{l+1} = (X_l + ATT(X_l))/2.  Returns (y, saved):
    y [B,H,T,D] (SA) or [C,B,H,T,D] (LLSA); saved = opaque buffer for stack_backward."""
    d = _desc_from(x0, L, R, scale, impl)
    nb = lib().sattn_stack_saved_bytes(ctypes.byref(d), mode, n_layers)
    if nb == 0:
        raise SattnError(lib().sattn_last_error().decode() or "invalid stack configuration")
    saved = torch.empty(nb, device=x0.device, dtype=torch.uint8)
    shp = ((R + 1,) if mode == MODE_LLSA else ()) + tuple(x0.shape)
    y = torch.empty(shp, device=x0.device, dtype=x0.dtype)
    _check(lib().sattn_stack_forward(ctypes.byref(d), mode, n_layers, _ptr(x0), _ptr(saved), nb, _ptr(y), _stream()),
           "sattn_stack_forward")
    return y, saved


def stack_saved_views(x0_like, saved, L: int, R: int, n_layers: int, mode: int = MODE_SA, scale=None, impl="auto"):
    """Per-layer views into stack_forward's `saved` buffer: [(X_l, O_l, LSE_l)] for l < n_layers."""
    d = _desc_from(x0_like, L, R, scale, impl)
    B, H, T, D = x0_like.shape
    C = R + 1 if mode == MODE_LLSA else 1
    es = x0_like.element_size()
    out = []
    for layer in range(n_layers):
        off = (ctypes.c_int64 * 3)()
        _check(lib().sattn_stack_saved_offsets(ctypes.byref(d), mode, n_layers, layer, off), "sattn_stack_saved_offsets")
        xs = (B, H, T, D) if (layer == 0 or C == 1) else (C, B, H, T, D)
        os_ = (C, B, H, T, D) if C > 1 else (B, H, T, D)
        view = lambda o, shp, dt, e: saved[o:o + e * int(torch.tensor(shp).prod())].view(dt).view(shp)  # noqa: E731
        out.append((view(off[0], xs, x0_like.dtype, es), view(off[1], os_, x0_like.dtype, es),
                    view(off[2], os_[:-1], torch.float32, 4)))
    return out


def stack_backward(x0_like, saved, dy, L: int, R: int, n_layers: int, mode: int = MODE_SA, scale=None, impl="auto",
                   ws=None):
    """Gradient of <dy, y> w.r.t. x0 (shape/dtype of x0_like)."""
    d = _desc_from(x0_like, L, R, scale, impl)
    nws = lib().sattn_stack_workspace(ctypes.byref(d), mode, n_layers)
    if ws is None or ws.numel() < nws:
        ws = torch.empty(nws, device=dy.device, dtype=torch.uint8)
    dx0 = torch.empty_like(x0_like)
    _check(lib().sattn_stack_backward(ctypes.byref(d), mode, n_layers, _ptr(saved), _ptr(dy), _ptr(dx0), _ptr(ws),
                                      nws, _stream()), "sattn_stack_backward")
    return dx0


# ----------------------------------------------------------------------- stream

class LLSAStream:
    """Incremental LLSA inference (one kernel launch per frame for all layers)."""

    def __init__(self, B, H, D, L, R, n_layers, dtype=torch.float32, scale=None, device="cuda"):
        self.B, self.H, self.D, self.L, self.R = B, H, D, L, R
        self.dtype, self.device = dtype, torch.device(device)
        code = F32 if dtype == torch.float32 else BF16
        d = make_desc(B, H, 1, D, L, R, code, scale)
        h = ctypes.c_void_p()
        _check(lib().llsa_stream_create(ctypes.byref(d), n_layers, ctypes.byref(h)), "llsa_stream_create")
        self._h = h
        self._y = torch.empty((B, H, D), device=self.device, dtype=dtype)

    def _check_x(self, x):
        _expect(x, (self.B, self.H, self.D), self.dtype, self.device if self.device.index is not None else x.device, "x")

    def step(self, x):
        """x [B,H,D] -> (frame index, y [B,H,D]) or None while h < R (y is a fresh tensor)."""
        self._check_x(x)
        fr = ctypes.c_int64(-1)
        y = torch.empty((self.B, self.H, self.D), device=self.device, dtype=self.dtype)
        _check(lib().llsa_stream_step(self._h, _ptr(x), _ptr(y), ctypes.byref(fr), _stream()), "llsa_stream_step")
        return None if fr.value < 0 else (fr.value, y)

    def step_into(self, x, y):
        """Graph-capturable variant: writes into y, returns the emitted frame index (-1 if none)."""
        self._check_x(x)
        self._check_x(y)
        fr = ctypes.c_int64(-1)
        _check(lib().llsa_stream_step(self._h, _ptr(x), _ptr(y), ctypes.byref(fr), _stream()), "llsa_stream_step")
        return fr.value

    def flush(self):
        tail = torch.empty((max(self.R, 1), self.B, self.H, self.D), device=self.device, dtype=self.dtype)
        n = ctypes.c_int32(0)
        _check(lib().llsa_stream_flush(self._h, _ptr(tail), ctypes.byref(n), _stream()), "llsa_stream_flush")
        return tail[: n.value]

    def reset(self):
        _check(lib().llsa_stream_reset(self._h), "llsa_stream_reset")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.llsa_stream_destroy(h)
            self._h = None


class SAStream:
    """Incremental SA inference (infer_sa): the SA stack frame by frame, latency n_layers x R
    (one kernel launch per frame for all layers)."""

    def __init__(self, B, H, D, L, R, n_layers, dtype=torch.float32, scale=None, device="cuda"):
        self.B, self.H, self.D, self.L, self.R, self.n_layers = B, H, D, L, R, n_layers
        self.dtype, self.device = dtype, torch.device(device)
        code = F32 if dtype == torch.float32 else BF16
        d = make_desc(B, H, 1, D, L, R, code, scale)
        h = ctypes.c_void_p()
        _check(lib().sa_stream_create(ctypes.byref(d), n_layers, ctypes.byref(h)), "sa_stream_create")
        self._h = h

    _check_x = LLSAStream._check_x

    def step(self, x):
        """x [B,H,D] -> (frame index, y [B,H,D]) or None while h < n_layers R."""
        self._check_x(x)
        fr = ctypes.c_int64(-1)
        y = torch.empty((self.B, self.H, self.D), device=self.device, dtype=self.dtype)
        _check(lib().sa_stream_step(self._h, _ptr(x), _ptr(y), ctypes.byref(fr), _stream()), "sa_stream_step")
        return None if fr.value < 0 else (fr.value, y)

    def step_into(self, x, y):
        self._check_x(x)
        self._check_x(y)
        fr = ctypes.c_int64(-1)
        _check(lib().sa_stream_step(self._h, _ptr(x), _ptr(y), ctypes.byref(fr), _stream()), "sa_stream_step")
        return fr.value

    def flush(self):
        n_tail = max(self.n_layers * self.R, 1)
        tail = torch.empty((n_tail, self.B, self.H, self.D), device=self.device, dtype=self.dtype)
        n = ctypes.c_int32(0)
        _check(lib().sa_stream_flush(self._h, _ptr(tail), ctypes.byref(n), _stream()), "sa_stream_flush")
        return tail[: n.value]

    def reset(self):
        _check(lib().sa_stream_reset(self._h), "sa_stream_reset")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.sa_stream_destroy(h)
            self._h = None


# --------------------------------------------------------------------- autograd

class SAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, L, R, scale=None, impl="auto"):
        o, lse = sa_forward(q, k, v, L, R, scale, impl)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.cfg = (L, R, scale, impl)
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        L, R, scale, impl = ctx.cfg
        dq, dk, dv = sa_backward(q, k, v, o, lse, do.contiguous(), L, R, scale, impl)
        return dq, dk, dv, None, None, None, None


class LLSAFunction(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, L, R, scale=None, impl="auto"):
        o, lse = llsa_forward(q, k, v, L, R, scale, impl)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.cfg = (L, R, scale, impl)
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        L, R, scale, impl = ctx.cfg
        dq, dk, dv = llsa_backward(q, k, v, o, lse, do.contiguous(), L, R, scale, impl)
        return dq, dk, dv, None, None, None, None
