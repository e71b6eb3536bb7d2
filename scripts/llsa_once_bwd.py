import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
C = R + 1
q, k, v, do = (torch.randn(C, B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = s.llsa_forward(q, k, v, L, R)
for _ in range(2):
    s.llsa_backward(q, k, v, o, lse, do, L, R)
torch.cuda.synchronize()
