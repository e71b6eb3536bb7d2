import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
for R in (5, 6, 7, 8):
    L, B, H, T = 16, 1, 1, 96
    C = R + 1
    q, k, v, do = (torch.randn(C, B, H, T, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
    o, lse = s.llsa_forward(q, k, v, L, R, impl="ffma")
    g1 = s.llsa_backward(q, k, v, o, lse, do, L, R, impl="tc")
    g2 = s.llsa_backward(q, k, v, o, lse, do, L, R, impl="ffma")
    print(R, [[round(float(x), 3) for x in (a.float() - b.float()).abs().amax(dim=(1, 2, 3, 4))] for a, b in zip(g1, g2)], flush=True)
