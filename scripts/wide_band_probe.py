"""Probe the stored-band path over the Fig. 5 widths (debug aid): sync after every call."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
T, D, B, H = 1000, 64, 8, 8
g = torch.Generator(device="cuda").manual_seed(5)
q, k, v, do = (torch.randn(B, H, T, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(4))
for W in [int(x) for x in sys.argv[1:]] or range(10, 491, 10):
    L = W // 2; R = W - 1 - L
    o, lse, pb = s.sa_forward_p(q, k, v, L, R); torch.cuda.synchronize()
    print("fwd ok", W, flush=True)
    s.sa_backward_p(q, k, v, o, pb, do, L, R); torch.cuda.synchronize()
    print("bwd ok", W, flush=True)
