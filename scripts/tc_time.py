"""Time the SA kernels (CUDA events) at the bench shape: debug aid."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
N = 12
qs = [[torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4)] for _ in range(N)]
for impl in ("tc",):
    outs = [s.sa_forward(q, k, v, L, R, impl=impl) for q, k, v, _ in qs]
    for _ in range(3):
        for (q, k, v, do), (o, lse) in zip(qs, outs):
            s.sa_forward(q, k, v, L, R, impl=impl); s.sa_backward(q, k, v, o, lse, do, L, R, impl=impl)
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record()
    for (q, k, v, do) in qs:
        s.sa_forward(q, k, v, L, R, impl=impl)
    e[1].record()
    for (q, k, v, do), (o, lse) in zip(qs, outs):
        s.sa_backward(q, k, v, o, lse, do, L, R, impl=impl)
    e[2].record()
    torch.cuda.synchronize()
    f = e[0].elapsed_time(e[1]) / N * 1e3
    b = e[1].elapsed_time(e[2]) / N * 1e3
    unit = B * H * T
    print(f"{impl}: fwd {f:.1f} us ({516*unit/f/1e3:.0f} GB/s)  bwd {b:.1f} us ({1028*unit/b/1e3:.0f} GB/s)")
