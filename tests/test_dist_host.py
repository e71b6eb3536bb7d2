"""Host-side logic of the time-sharded C path (no GPU): the slab / tile-split geometry the
library computes (sattn_tshard_geometry) against a brute-force reading of which tiles touch
a margin, and the host-staged halo swap of paper_2302_13451_b200.dist over gloo (world 2, 3)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

M = 128


def _nk(L, R):
    # rows of the K/V box one 128-query tile loads (the kernels' NK: 16-rounded 96 + CW,
    # CW = the first of 32, 48, 64, 72, 80, 96 >= W + 31)
    need = L + R + 1 + 31
    cw = next(c for c in (32, 48, 64, 72, 80, 96) if c >= need)
    return (96 + cw + 15) // 16 * 16


def _brute(T_loc, L, R, left, right):
    hl, hr = (M if left else 0), (M if right else 0)
    Ts = hl + T_loc + hr
    ntq = -(-Ts // 128)
    nk = _nk(L, R)
    edge = []
    for kt in range(ntq):
        rows = set(range(128 * kt, min(Ts, 128 * kt + 128)))
        rows |= set(range(max(0, 128 * kt - L), min(Ts, 128 * kt - L + nk)))
        touches = any((r < hl) or (r >= hl + T_loc) for r in rows)
        edge.append(touches)
    return hl, hr, Ts, ntq, edge


@pytest.mark.parametrize("T_loc,L,R", [(22528, 32, 8), (22528, 32, 16), (1750, 32, 32), (300, 3, 1), (128, 0, 0),
                                       (200, 60, 4), (130, 5, 2)])
@pytest.mark.parametrize("pos", ["first", "middle", "last"])
def test_tshard_geometry_matches_brute_force(T_loc, L, R, pos):
    from paper_2302_13451_b200 import dist as sd
    world = 3
    rank = {"first": 0, "middle": 1, "last": 2}[pos]
    t0 = rank * 100000
    T_global = 3 * 100000 if pos != "last" else t0 + T_loc
    if pos == "last":
        T_global = t0 + T_loc
    hl, hr, Ts, ntq, e0, e1 = sd.geometry(1, 2, T_loc, 64, L, R, t0, T_global, rank, world)
    bhl, bhr, bTs, bntq, edge = _brute(T_loc, L, R, rank > 0, rank < world - 1)
    assert (hl, hr, Ts, ntq) == (bhl, bhr, bTs, bntq)
    # the library's split: edge = [0, e0) + [e1, ntq); it may only call a tile interior if it is
    assert all(not edge[kt] for kt in range(e0, e1))
    assert all(edge[kt] for kt in list(range(e0)) + list(range(e1, ntq))) or not (rank > 0 or rank < world - 1)


def test_tshard_geometry_rejects_bad_configs():
    from paper_2302_13451_b200 import SattnError
    from paper_2302_13451_b200 import dist as sd
    with pytest.raises(SattnError):     # shard position inconsistent with the rank
        sd.geometry(1, 1, 256, 64, 32, 8, 0, 1024, 1, 2)
    with pytest.raises(SattnError):     # L + R beyond the margin
        sd.geometry(1, 1, 256, 64, 100, 40, 256, 1024, 1, 4)
    with pytest.raises(SattnError):     # shard shorter than the halo its neighbours need
        sd.geometry(1, 1, 30, 64, 32, 8, 256, 1024, 1, 4)
    with pytest.raises(SattnError):     # not the tensor-core path (D = 32)
        sd.geometry(1, 1, 256, 32, 32, 8, 256, 1024, 1, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _swap_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2302_13451_b200.dist import host_swap
    # rank r sends (r, 'L') * 3 + r bytes to the left and (r, 'R') * 5 bytes to the right
    sl = torch.full((3 + rank,), 10 + rank, dtype=torch.uint8)
    sr = torch.full((5,), 100 + rank, dtype=torch.uint8)
    nrl = 5 if rank > 0 else 0                 # the left neighbour's send_r
    nrr = 3 + rank + 1 if rank < world - 1 else 0  # the right neighbour's send_l
    rl, rr = host_swap(None, rank, world, sl, nrl, sr, nrr)
    out[rank] = (None if rl is None else rl.tolist(), None if rr is None else rr.tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_swap_gloo(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_swap_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        rl, rr = out[r]
        assert rl == (None if r == 0 else [100 + r - 1] * 5)
        assert rr == (None if r == world - 1 else [10 + r + 1] * (3 + r + 1))


def _noop_exchange(*args):
    return 0


def test_llsa_tshard_margin_and_workspace_validation():
    # the time-sharded LLSA slab: margin L + 2R on a side with a neighbour (the halo outputs'
    # windows); the workspace query rejects what the calls would reject
    import ctypes
    from paper_2302_13451_b200 import dist as sd
    assert sd.llsa_margin(32, 8) == 48 and sd.llsa_margin(32, 16) == 64 and sd.llsa_margin(3, 1) == 5
    assert sd.llsa_slab_rows(1000, 32, 8, 0, 3000) == (0, 48)
    assert sd.llsa_slab_rows(1000, 32, 8, 1000, 3000) == (48, 48)
    assert sd.llsa_slab_rows(1000, 32, 8, 2000, 3000) == (48, 0)
    L = sd._lib()
    cb = sd.EXCHANGE_FN(_noop_exchange)
    for rank, t0, T_global in ((0, 0, 2000), (1, 1000, 2000)):
        h = ctypes.c_void_p()
        assert L.sattn_dist_init_external(rank, 2, cb, None, ctypes.byref(h)) == 0
        td = sd.tdesc(2, 3, 1000, 64, 32, 8, t0, T_global)
        n = L.llsa_tsharded_workspace(ctypes.byref(td), h)
        # at least the forward's messages: 3 tensors x (R+1) channels x B*H x (L+2R) rows x 128 B, sent and received
        assert n >= 2 * 3 * 9 * 6 * 48 * 128
        bad = sd.tdesc(2, 3, 40, 64, 32, 8, t0, T_global)        # shard shorter than L + 2R
        assert L.llsa_tsharded_workspace(ctypes.byref(bad), h) == 0
        bad = sd.tdesc(2, 3, 1000, 64, 32, 8, 500 if rank == 0 else 0, T_global)   # position vs rank
        assert L.llsa_tsharded_workspace(ctypes.byref(bad), h) == 0
        td.local.in_broadcast = 1                                 # dense inputs only
        assert L.llsa_tsharded_workspace(ctypes.byref(td), h) == 0
        L.sattn_dist_destroy(h)
