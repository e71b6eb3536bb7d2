"""Small stored-band and LSE-mode SA calls for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2302_13451_b200 as s

g = torch.Generator(device="cuda").manual_seed(0)
for (B, H, T, L, R) in ((1, 2, 300, 32, 8), (1, 1, 200, 32, 16), (1, 1, 129, 0, 0)):
    q, k, v, do = (torch.randn(B, H, T, 64, device="cuda", generator=g).bfloat16() for _ in range(4))
    o, lse, p = s.sa_forward_p(q, k, v, L, R)
    s.sa_backward_p(q, k, v, o, p, do, L, R)
    o, lse = s.sa_forward(q, k, v, L, R)
    s.sa_backward(q, k, v, o, lse, do, L, R)
    qf, kf, vf, dof = (x.float() for x in (q, k, v, do))
    o, lse, p = s.sa_forward_p(qf, kf, vf, L, R)
    s.sa_backward_p(qf, kf, vf, o, p, dof, L, R)
torch.cuda.synchronize()
print("done")
