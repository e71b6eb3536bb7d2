"""Time sharding over ranks: partition helpers and the deep-halo stack.

The per-layer time-sharded SA call is in the C ABI (``sa_forward_tsharded`` /
``sa_backward_tsharded``, include/sattn.h; Python binding ``paper_2302_13451_b200.dist``):
the library packs, exchanges (NCCL or a callback) and unpacks the halo rows and overlaps
the exchange with the interior tiles.  This module keeps

* ``shard_bounds``: rank r's frames [t0, t1), 128-frame aligned so that every local frame
  keeps its tile offset (the sharded rows are then bitwise equal to the unsharded call's);
* the deep-halo variant (NEXT-4): a whole n-layer stack on a time shard with ONE exchange
  of n x (L + R) frames (``exchange_halo`` over torch.distributed point-to-point), traded
  against recomputing the halo frames in every layer.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(T: int, world: int, rank: int, align: int = 1):
    """[t0, t1) of `rank`: `align`-frame units split as evenly as possible."""
    units = -(-T // align)
    u0 = units * rank // world
    u1 = units * (rank + 1) // world
    return min(T, u0 * align), min(T, u1 * align)


def _round_up(x: int, a: int) -> int:
    return -(-x // a) * a


def _peer(group, r):
    return dist.get_global_rank(group, r) if group is not None else r


def exchange_halo(x: torch.Tensor, left: int, right: int, group=None):
    """Extend the local slab x[..., T_loc, D] with `left` frames from rank-1 and `right`
    frames from rank+1 (none at the global edges).  Every rank must pass the same
    (left, right) and hold at least max(left, right) frames.
    Returns (x_ext, number of frames prepended)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    T_loc = x.shape[-2]
    ops, recv_l, recv_r = [], None, None
    if rank > 0 and (left or right):
        if left:
            recv_l = torch.empty(x.shape[:-2] + (left, x.shape[-1]), dtype=x.dtype, device=x.device)
            ops.append(dist.P2POp(dist.irecv, recv_l, _peer(group, rank - 1), group))
        if right:
            ops.append(dist.P2POp(dist.isend, x[..., :right, :].contiguous(), _peer(group, rank - 1), group))
    if rank < world - 1 and (left or right):
        if left:
            ops.append(dist.P2POp(dist.isend, x[..., T_loc - left:, :].contiguous(), _peer(group, rank + 1), group))
        if right:
            recv_r = torch.empty(x.shape[:-2] + (right, x.shape[-1]), dtype=x.dtype, device=x.device)
            ops.append(dist.P2POp(dist.irecv, recv_r, _peer(group, rank + 1), group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    parts = [p for p in (recv_l, x, recv_r) if p is not None]
    return torch.cat(parts, dim=-2), (left if recv_l is not None else 0)


def _halo(width: int, align: int, T_loc: int, group, min_T: int | None = None) -> int:
    """`width` rounded up to `align` if every shard can supply it (agreed across ranks).  `min_T`,
    the smallest shard's frames, when the caller knows it (e.g. from shard_bounds): then no
    collective and no host synchronisation; else a MIN all-reduce of T_loc."""
    if min_T is None:
        t = torch.tensor([T_loc], dtype=torch.int64)
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        min_T = int(t.item())
    if width > min_T:
        raise ValueError(f"shards of {min_T} frames cannot supply a {width}-frame halo: use fewer ranks")
    r = _round_up(width, align) if width else 0
    return r if r <= min_T else width


# ------------------------------------------------------------------ deep halo (NEXT-4)
# A whole n-layer stack on a time shard with ONE exchange instead of one per layer: an output
# frame t of the stack depends on input frames [t - n (L + R), t + n R] (each SA layer reaches
# L back and R ahead; an LLSA layer's band reaches L + R back, reading G6), so a
# slab extended by that deep halo reproduces the local rows exactly; the backward's dX_0(u)
# reaches dY over [u - n R, u + n L] and the activations around them, so twice the forward
# halo on both sides (SURVEY §8(c) time-sharding pins: per-layer margins L + R forward and
# 2 (L + R) backward, times n_layers).  The trade: recompute of the halo frames in every layer
# against n - 1 fewer exchanges (for the hour-long stream at 8 ranks: 480 of 22,500 frames).

def _stack_fwd_default(x, L, R, n, mode):
    import paper_2302_13451_b200 as s
    return s.stack_forward(x, L, R, n, mode)[0]


def _stack_bwd_default(x, dy, L, R, n, mode):
    import paper_2302_13451_b200 as s
    _, saved = s.stack_forward(x, L, R, n, mode)
    return s.stack_backward(x, saved, dy, L, R, n, mode)


def stack_forward_tsharded(x, L: int, R: int, n_layers: int, mode: int = 0, group=None, align: int = 128,
                           stack_fwd=None, min_T: int | None = None):
    """x: this rank's slab [B, H, T_loc, D].  Returns this rank's rows of the n-layer stack
    output (SA: [B, H, T_loc, D]; LLSA mode 1: [C, B, H, T_loc, D])."""
    stack_fwd = stack_fwd or _stack_fwd_default
    T_loc = x.shape[-2]
    back = n_layers * (L + R) if mode == 1 else n_layers * L
    hl, hr = _halo(back, align, T_loc, group, min_T), _halo(n_layers * R, align, T_loc, group, min_T)
    x_e, nl = exchange_halo(x, hl, hr, group)
    y = stack_fwd(x_e, L, R, n_layers, mode)
    return y[..., nl:nl + T_loc, :].contiguous()


def stack_backward_tsharded(x, dy, L: int, R: int, n_layers: int, mode: int = 0, group=None, align: int = 128,
                            stack_bwd=None, min_T: int | None = None):
    """x: this rank's input slab [B, H, T_loc, D]; dy: its rows of dL/dY (SA [B, H, T_loc, D],
    LLSA [C, B, H, T_loc, D]).  Returns this rank's rows of dL/dX_0."""
    stack_bwd = stack_bwd or _stack_bwd_default
    T_loc = x.shape[-2]
    h = _halo(2 * n_layers * (L + R), align, T_loc, group, min_T)
    x_e, nl = exchange_halo(x, h, h, group)
    dy_e, _ = exchange_halo(dy, h, h, group)
    dx = stack_bwd(x_e, dy_e, L, R, n_layers, mode)
    return dx[..., nl:nl + T_loc, :].contiguous()
