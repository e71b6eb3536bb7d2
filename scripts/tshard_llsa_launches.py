"""Diagnostic: launch counts of the time-sharded LLSA calls on a 2-process group sharing the GPU
(gloo + the callback transport).  The overlapped path launches the interior and edge items
separately: forward = exchange copies + 2 item launches, backward = exchange copies + 2 fused
launches + the kv pass (4 / 5 here; 3 / 4 before the interior/edge split)."""
import os, sys, socket
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import torch
def port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p
def w(rank, world, p):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(p)
    import torch.distributed as tdist
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2302_13451_b200 as s
    from paper_2302_13451_b200 import dist as sd
    from paper_2302_13451_b200 import tshard
    L, R, T = 32, 8, 900
    C, B, H, D = R + 1, 1, 2, 64
    t0, t1 = tshard.shard_bounds(T, world, rank, 1)
    n = t1 - t0
    hl, hr = sd.llsa_slab_rows(n, L, R, t0, T)
    d = sd.Dist()
    slab = lambda: torch.randn(C, B, H, hl + n + hr, D, device="cuda").to(torch.bfloat16)
    qs, ks, vs, dos = slab(), slab(), slab(), slab()
    c0 = s.launch_count()
    os_, lses = sd.llsa_forward_tsharded(qs, ks, vs, n, L, R, t0, T, d)
    torch.cuda.synchronize(); c1 = s.launch_count()
    gs = sd.llsa_backward_tsharded(qs, ks, vs, os_, lses, dos, n, L, R, t0, T, d)
    torch.cuda.synchronize(); c2 = s.launch_count()
    print(f"rank {rank}: fwd launches {c1 - c0}, bwd launches {c2 - c1}", flush=True)
    d.close(); tdist.barrier(); tdist.destroy_process_group()
if __name__ == "__main__":
    import torch.multiprocessing as mp
    mp.spawn(w, args=(2, port()), nprocs=2, join=True)
