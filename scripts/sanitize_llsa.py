"""Small LLSA calls (tensor-core and CUDA-core, dense and broadcast inputs) + one stream step loop,
for compute-sanitizer."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2302_13451_b200 as s

g = torch.Generator(device="cuda").manual_seed(0)
for (B, H, T, L, R) in ((1, 2, 300, 32, 8), (1, 1, 130, 16, 4)):
    C = R + 1
    for bc in (False, True):
        shp = (B, H, T, 64) if bc else (C, B, H, T, 64)
        q, k, v = (torch.randn(*shp, device="cuda", generator=g).bfloat16() for _ in range(3))
        do = torch.randn(C, B, H, T, 64, device="cuda", generator=g).bfloat16()
        o, lse = s.llsa_forward(q, k, v, L, R, broadcast=bc)
        s.llsa_backward(q, k, v, o, lse, do, L, R, broadcast=bc)
torch.cuda.synchronize()
print("done")
