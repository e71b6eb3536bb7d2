import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
L, R, T, H = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
q, k, v, do = (torch.randn(1, H, T, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = s.sa_forward(q, k, v, L, R, impl="tc"); torch.cuda.synchronize()
o2, lse2 = s.sa_forward(q, k, v, L, R, impl="ffma")
print(L, R, "fwd ok", float((o.float()-o2.float()).abs().max()), flush=True)
g = s.sa_backward(q, k, v, o, lse, do, L, R, impl="auto"); torch.cuda.synchronize()
g2 = s.sa_backward(q, k, v, o, lse, do, L, R, impl="ffma")
print(L, R, "bwd ok", [float((a.float()-b.float()).abs().max()) for a, b in zip(g, g2)], flush=True)
