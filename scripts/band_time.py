"""Time the stored-band mode (sa_forward_p + sa_backward_p) against the LSE-recompute path
at the bench shape (one layer, CUDA events, median of 20)."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2302_13451_b200 as s

B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
if len(sys.argv) > 2:
    L, R = int(sys.argv[1]), int(sys.argv[2])
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v, do = (torch.randn(B, H, T, D, device="cuda", generator=g).bfloat16() for _ in range(4))


def t(fn, n=20):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return sorted(ts)[n // 2]


o, lse, p = s.sa_forward_p(q, k, v, L, R)
res = {}
for impl in ("auto", "ffma"):
    o2, l2 = s.sa_forward(q, k, v, L, R, impl=impl)
    res[f"fwd_{impl}"] = t(lambda: s.sa_forward(q, k, v, L, R, impl=impl))
    res[f"bwd_{impl}"] = t(lambda: s.sa_backward(q, k, v, o2, l2, do, L, R, impl=impl))
res["fwd_p"] = t(lambda: s.sa_forward_p(q, k, v, L, R))
res["bwd_p"] = t(lambda: s.sa_backward_p(q, k, v, o, p, do, L, R))
print({k_: round(v_, 1) for k_, v_ in res.items()}, "us; band bytes", p.numel() * 2)
