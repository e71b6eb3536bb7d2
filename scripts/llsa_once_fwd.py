"""One LLSA forward at the bench shape (ncu target: llsa_fwd_item_tc)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
C = R + 1
q, k, v = (torch.randn(C, B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(3))
for _ in range(2):
    o, lse = s.llsa_forward(q, k, v, L, R)
torch.cuda.synchronize()
