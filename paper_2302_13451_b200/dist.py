"""Time-sharded SA and LLSA over ranks through the C ABI (include/sattn.h "time sharding"): thin binding.

The library does the work — halo pack/unpack kernels, the exchange (NCCL point-to-point on a
library stream, or a caller callback), the interior/edge tile split that overlaps it, and the
tensor-core SA kernels on the halo-extended slab.  This module only marshals arguments and
provides the two transports' plumbing:

* ``Dist(group)`` on an NCCL process group: rank 0 draws the NCCL unique id
  (``sattn_dist_unique_id``), it is broadcast over the torch group, every rank calls
  ``sattn_dist_init`` — the library owns its communicator and stream.
* ``Dist(group)`` on a gloo group (CPU tests, or several processes sharing one GPU, where NCCL
  refuses duplicate devices): ``sattn_dist_init_external`` with a host-staged callback (device
  -> host copy, gloo send/recv with rank +- 1, host -> device copy).

Tensors are MARGINED ([B, H, M + T_loc + M, D], M = ``MARGIN``; LSE [B, H, M + T_loc + M]),
local frames at rows [M, M + T_loc): ``margined()`` allocates (zero-filled, as the ABI asks),
``local()`` views the local rows.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as tdist

from . import Desc, SattnError, _check, _dtype_code, _ptr, _stream, lib, make_desc

MARGIN = 128


class TShardDesc(ctypes.Structure):
    _fields_ = [("local", Desc), ("t0", ctypes.c_int64), ("T_global", ctypes.c_int64)]


EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p,
                               ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                               ctypes.c_void_p)
_P, _SZ, _I = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
_PT = ctypes.POINTER(TShardDesc)
EXPORTS = {
    "sattn_tshard_margin": (ctypes.c_int64, []),
    "sattn_dist_unique_id": (_I, [_P]),
    "sattn_dist_init": (_I, [_I, _I, _P, ctypes.POINTER(_P)]),
    "sattn_dist_init_external": (_I, [_I, _I, EXCHANGE_FN, _P, ctypes.POINTER(_P)]),
    "sattn_dist_destroy": (None, [_P]),
    "sa_tsharded_workspace": (_SZ, [_PT, _P]),
    "sa_forward_tsharded": (_I, [_PT, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_backward_tsharded": (_I, [_PT, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "sattn_tshard_geometry": (_I, [_PT, _I, _I, ctypes.POINTER(ctypes.c_int64)]),
    "sa_forward_p_tsharded": (_I, [_PT, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_backward_p_tsharded": (_I, [_PT, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "llsa_tshard_margin": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32]),
    "llsa_tsharded_workspace": (_SZ, [_PT, _P]),
    "llsa_forward_tsharded": (_I, [_PT, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
    "llsa_backward_tsharded": (_I, [_PT, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _SZ, _P]),
}
_bound = False


def _lib():
    global _bound
    L = lib()
    if not _bound:
        for name, (res, args) in EXPORTS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _bound = True
    return L


def _cudart():
    import glob
    import os
    for cand in ("libcudart.so.12", "libcudart.so"):
        try:
            return ctypes.CDLL(cand)
        except OSError:
            pass
    for p in glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                    "libcudart.so*")):
        return ctypes.CDLL(p)
    raise SattnError("libcudart not found for the host-staged exchange")


def tdesc(B, H, T_loc, D, L, R, t0, T_global, dtype=torch.bfloat16, scale=None) -> TShardDesc:
    code = 1 if dtype == torch.bfloat16 else 0
    return TShardDesc(make_desc(B, H, T_loc, D, L, R, code, scale), t0, T_global)


def geometry(B, H, T_loc, D, L, R, t0, T_global, rank, world):
    """(hl, hr, slab frames, query tiles, first interior tile, first right-edge tile) — host only."""
    out = (ctypes.c_int64 * 6)()
    d = tdesc(B, H, T_loc, D, L, R, t0, T_global)
    _check(_lib().sattn_tshard_geometry(ctypes.byref(d), rank, world, out), "sattn_tshard_geometry")
    return tuple(int(x) for x in out)


def margined(B, H, T_loc, D=None, dtype=torch.bfloat16, device="cuda"):
    """Zero-filled margined buffer: [B, H, M + T_loc + M, D] (D=None: LSE-shaped [B, H, M + T_loc + M])."""
    shp = (B, H, T_loc + 2 * MARGIN) + ((D,) if D else ())
    return torch.zeros(shp, dtype=dtype, device=device)


def local(x, T_loc):
    """The local rows of a margined tensor (a view)."""
    return x[:, :, MARGIN:MARGIN + T_loc]


class Dist:
    """Library-owned time-sharding handle for this rank of `group` (see module doc)."""

    def __init__(self, group=None, transport: str = "auto"):
        self.group = group
        self.rank = tdist.get_rank(group) if tdist.is_initialized() else 0
        self.world = tdist.get_world_size(group) if tdist.is_initialized() else 1
        backend = tdist.get_backend(group) if tdist.is_initialized() else "none"
        if transport == "auto":
            transport = "nccl" if backend == "nccl" or self.world == 1 else "host"
        self.transport = transport
        h = ctypes.c_void_p()
        L = _lib()
        if transport == "nccl":
            uid = (ctypes.c_uint8 * 128)()
            if self.world > 1:
                if self.rank == 0:
                    _check(L.sattn_dist_unique_id(uid), "sattn_dist_unique_id")
                t = torch.tensor(bytearray(uid), dtype=torch.uint8)
                if backend == "nccl":
                    t = t.cuda()
                tdist.broadcast(t, src=tdist.get_global_rank(group, 0) if group is not None else 0, group=group)
                uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
            _check(L.sattn_dist_init(self.rank, self.world, uid, ctypes.byref(h)), "sattn_dist_init")
        elif transport == "host":
            self._cb = EXCHANGE_FN(self._exchange)
            self._rt = _cudart()
            _check(L.sattn_dist_init_external(self.rank, self.world, self._cb, None, ctypes.byref(h)),
                   "sattn_dist_init_external")
        else:
            raise SattnError(f"unknown transport {transport}")
        self._h = h
        self._ws = None

    # host-staged exchange (gloo): called by the library with device pointers
    def _exchange(self, user, sl, nsl, rl, nrl, sr, nsr, rr, nrr, stream):
        try:
            rt = self._rt
            if rt.cudaStreamSynchronize(ctypes.c_void_p(stream)) != 0:
                return 1

            def d2h(p, n):
                a = np.empty(n, dtype=np.uint8)
                if n and rt.cudaMemcpy(a.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(p), ctypes.c_size_t(n), 2):
                    raise RuntimeError("cudaMemcpy D2H")
                return torch.from_numpy(a)

            got_l, got_r = host_swap(self.group, self.rank, self.world,
                                     d2h(sl, nsl) if sl else None, nrl if rl else 0,
                                     d2h(sr, nsr) if sr else None, nrr if rr else 0)
            for p, buf in ((rl, got_l), (rr, got_r)):
                if buf is not None and buf.numel():
                    a = buf.numpy()
                    if rt.cudaMemcpy(ctypes.c_void_p(p), a.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(a.size), 1):
                        return 1
            return 0
        except Exception:  # no exception may cross the C boundary
            import traceback
            traceback.print_exc()
            return 1

    def _workspace(self, d, device, query="sa_tsharded_workspace"):
        n = int(getattr(_lib(), query)(ctypes.byref(d), self._h))
        if n == 0:
            raise SattnError(_lib().sattn_last_error().decode() or "invalid time-shard configuration")
        if self._ws is None or self._ws.numel() < n or self._ws.device != device:
            self._ws = torch.empty(n, dtype=torch.uint8, device=device)
        return self._ws

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib().sattn_dist_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_swap(group, rank, world, send_l, n_recv_l, send_r, n_recv_r):
    """One halo swap with rank -+ 1 over torch.distributed point-to-point on host byte tensors:
    send_l goes to rank-1 (which receives it as its recv_r), send_r to rank+1; returns
    (recv_l from rank-1, recv_r from rank+1), None where there is no neighbour or nothing to receive."""
    peer = (lambda r: tdist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    ops, recv_l, recv_r = [], None, None
    if rank > 0:
        if send_l is not None and send_l.numel():
            ops.append(tdist.P2POp(tdist.isend, send_l, peer(rank - 1), group))
        if n_recv_l:
            recv_l = torch.empty(n_recv_l, dtype=torch.uint8)
            ops.append(tdist.P2POp(tdist.irecv, recv_l, peer(rank - 1), group))
    if rank < world - 1:
        if send_r is not None and send_r.numel():
            ops.append(tdist.P2POp(tdist.isend, send_r, peer(rank + 1), group))
        if n_recv_r:
            recv_r = torch.empty(n_recv_r, dtype=torch.uint8)
            ops.append(tdist.P2POp(tdist.irecv, recv_r, peer(rank + 1), group))
    if ops:
        for w in tdist.batch_isend_irecv(ops):
            w.wait()
    return recv_l, recv_r


def _tdesc_from(qm, L, R, t0, T_global, scale):
    B, H, Tm, D = qm.shape
    T_loc = Tm - 2 * MARGIN
    if T_loc <= 0:
        raise SattnError("margined tensors need more than 2 x MARGIN frames")
    return TShardDesc(make_desc(B, H, T_loc, D, L, R, _dtype_code(qm), scale), t0, T_global)


def sa_forward_tsharded(qm, km, vm, L: int, R: int, t0: int, T_global: int, d: Dist, scale=None):
    """Margined q, k, v [B, H, M + T_loc + M, D] of this rank (frames [t0, t0 + T_loc)) ->
    margined (o, lse); local rows = the unsharded sa_forward's rows [t0, t0 + T_loc).  Fills
    the K, V, Q margins (kept for sa_backward_tsharded)."""
    td = _tdesc_from(qm, L, R, t0, T_global, scale)
    for t in (km, vm):
        if t.shape != qm.shape or t.dtype != qm.dtype:
            raise SattnError("q, k, v must share shape and dtype")
    om = torch.zeros_like(qm)
    lsem = torch.zeros(qm.shape[:-1], dtype=torch.float32, device=qm.device)
    ws = d._workspace(td, qm.device)
    _check(_lib().sa_forward_tsharded(ctypes.byref(td), d._h, _ptr(qm), _ptr(km), _ptr(vm), _ptr(om), _ptr(lsem),
                                      _ptr(ws), ws.numel(), _stream()), "sa_forward_tsharded")
    return om, lsem


def sa_backward_tsharded(qm, km, vm, lsem, dom, L: int, R: int, t0: int, T_global: int, d: Dist, scale=None):
    """Margined dq, dk, dv (local rows = the unsharded sa_backward's).  q, k, v, lse: the
    forward's margined buffers; dom: margined dO (its margins are filled here)."""
    td = _tdesc_from(qm, L, R, t0, T_global, scale)
    if dom.shape != qm.shape or lsem.shape != qm.shape[:-1] or lsem.dtype != torch.float32:
        raise SattnError("dO must be shaped like q and lse [B, H, M + T_loc + M] fp32")
    dq, dk, dv = torch.zeros_like(qm), torch.zeros_like(qm), torch.zeros_like(qm)
    ws = d._workspace(td, qm.device)
    _check(_lib().sa_backward_tsharded(ctypes.byref(td), d._h, _ptr(qm), _ptr(km), _ptr(vm), _ptr(lsem), _ptr(dom),
                                       _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(), _stream()),
           "sa_backward_tsharded")
    return dq, dk, dv


def sa_forward_p_tsharded(qm, km, vm, L: int, R: int, t0: int, T_global: int, d: Dist, scale=None):
    """The stored-band forward on margined shards -> margined (o, lse, p); p [B, H, M + T_loc + M, ld]
    (ld = W rounded to 8), its local rows = the unsharded sa_forward_p's band rows."""
    td = _tdesc_from(qm, L, R, t0, T_global, scale)
    for t in (km, vm):
        if t.shape != qm.shape or t.dtype != qm.dtype:
            raise SattnError("q, k, v must share shape and dtype")
    ld = (L + R + 1 + 7) // 8 * 8
    om = torch.zeros_like(qm)
    lsem = torch.zeros(qm.shape[:-1], dtype=torch.float32, device=qm.device)
    pm = torch.zeros(qm.shape[:-1] + (ld,), dtype=qm.dtype, device=qm.device)
    ws = d._workspace(td, qm.device)
    _check(_lib().sa_forward_p_tsharded(ctypes.byref(td), d._h, _ptr(qm), _ptr(km), _ptr(vm), _ptr(om), _ptr(lsem),
                                        _ptr(pm), _ptr(ws), ws.numel(), _stream()), "sa_forward_p_tsharded")
    return om, lsem, pm


def sa_backward_p_tsharded(qm, km, vm, pm, dom, L: int, R: int, t0: int, T_global: int, d: Dist, scale=None):
    """Margined dq, dk, dv from the stored band (local rows = the unsharded sa_backward_p's).  q, k, v,
    p: the forward's margined buffers; dom: margined dO (its margins are filled here)."""
    td = _tdesc_from(qm, L, R, t0, T_global, scale)
    ld = (L + R + 1 + 7) // 8 * 8
    if dom.shape != qm.shape or pm.shape != qm.shape[:-1] + (ld,) or pm.dtype != qm.dtype:
        raise SattnError("dO must be shaped like q and p [B, H, M + T_loc + M, ld] in q's dtype")
    dq, dk, dv = torch.zeros_like(qm), torch.zeros_like(qm), torch.zeros_like(qm)
    ws = d._workspace(td, qm.device)
    _check(_lib().sa_backward_p_tsharded(ctypes.byref(td), d._h, _ptr(qm), _ptr(km), _ptr(vm), _ptr(pm), _ptr(dom),
                                         _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(), _stream()),
           "sa_backward_p_tsharded")
    return dq, dk, dv

# ------------------------------------------------------------------ time-sharded LLSA (slab layout)

def llsa_margin(L: int, R: int) -> int:
    """Frames of a time-sharded LLSA slab's margin on a side with a neighbour (L + 2R)."""
    return int(_lib().llsa_tshard_margin(L, R))


def llsa_slab_rows(T_loc: int, L: int, R: int, t0: int, T_global: int):
    """(hl, hr): margin frames before / after this rank's local rows in its LLSA slab."""
    m = llsa_margin(L, R)
    return (m if t0 > 0 else 0), (m if t0 + T_loc < T_global else 0)


def _ltdesc(x, T_loc, L, R, t0, T_global, scale):
    C, B, H, Ts, D = x.shape
    if C != R + 1:
        raise SattnError(f"LLSA slab has {C} channels, expected R + 1 = {R + 1}")
    hl, hr = llsa_slab_rows(T_loc, L, R, t0, T_global)
    if Ts != hl + T_loc + hr:
        raise SattnError(f"slab frames {Ts} != {hl} + {T_loc} + {hr}")
    return TShardDesc(make_desc(B, H, T_loc, D, L, R, _dtype_code(x), scale), t0, T_global)


def llsa_forward_tsharded(q, k, v, T_loc: int, L: int, R: int, t0: int, T_global: int, d: Dist, scale=None):
    """Slabs q, k, v [C, B, H, hl + T_loc + hr, D] (local frames [t0, t0 + T_loc) at rows
    [hl, hl + T_loc)) -> slabs (o, lse); fills the q, k, v margins (kept for the backward)."""
    td = _ltdesc(q, T_loc, L, R, t0, T_global, scale)
    for t in (k, v):
        if t.shape != q.shape or t.dtype != q.dtype:
            raise SattnError("q, k, v must share shape and dtype")
    o = torch.zeros_like(q)
    lse = torch.zeros(q.shape[:-1], dtype=torch.float32, device=q.device)
    ws = d._workspace(td, q.device, "llsa_tsharded_workspace")
    _check(_lib().llsa_forward_tsharded(ctypes.byref(td), d._h, _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                        _ptr(ws), ws.numel(), _stream()), "llsa_forward_tsharded")
    return o, lse


def llsa_backward_tsharded(q, k, v, o, lse, do, T_loc: int, L: int, R: int, t0: int, T_global: int, d: Dist,
                           scale=None):
    """Slabs dq, dk, dv (local rows exact).  q, k, v, o, lse: the forward's slabs; do: this
    rank's dO slab (local rows set; its halo rows are filled here)."""
    td = _ltdesc(q, T_loc, L, R, t0, T_global, scale)
    if do.shape != q.shape or o.shape != q.shape or lse.shape != q.shape[:-1] or lse.dtype != torch.float32:
        raise SattnError("o, do must be shaped like q and lse [C, B, H, Ts] fp32")
    dq, dk, dv = torch.zeros_like(q), torch.zeros_like(q), torch.zeros_like(q)
    ws = d._workspace(td, q.device, "llsa_tsharded_workspace")
    _check(_lib().llsa_backward_tsharded(ctypes.byref(td), d._h, _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                         _ptr(do), _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(), _stream()),
           "llsa_backward_tsharded")
    return dq, dk, dv
