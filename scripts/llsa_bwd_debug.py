"""LLSA backward: tensor-core path vs FFMA kernels (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
for (B, H, T, L, R, bc) in [(1, 1, 200, 32, 8, False), (1, 2, 300, 32, 8, False), (2, 3, 1750, 32, 8, False),
                            (1, 2, 300, 32, 8, True), (1, 2, 200, 16, 4, False), (1, 1, 100, 3, 5, False),
                            (1, 1, 130, 5, 1, False)]:
    C = R + 1
    shp = (B, H, T, 64) if bc else (C, B, H, T, 64)
    q, k, v = (torch.randn(*shp, device="cuda").to(torch.bfloat16) for _ in range(3))
    do = torch.randn(C, B, H, T, 64, device="cuda").to(torch.bfloat16)
    o, lse = s.llsa_forward(q, k, v, L, R, impl="ffma", broadcast=bc)
    try:
        g1 = s.llsa_backward(q, k, v, o, lse, do, L, R, impl="tc", broadcast=bc)
        torch.cuda.synchronize()
    except Exception as e:
        print((B, H, T, L, R, bc), "TC ERR", e, flush=True); continue
    g2 = s.llsa_backward(q, k, v, o, lse, do, L, R, impl="ffma", broadcast=bc)
    errs = [float((a.float() - b.float()).abs().max()) for a, b in zip(g1, g2)]
    print((B, H, T, L, R, bc), "dQ dK dV", errs, flush=True)
    if max(errs) > 0.05:
        for name, a, b in zip("QKV", g1, g2):
            d = (a.float() - b.float()).abs().amax(dim=(1, 2, 3, 4))
            print("   d" + name, "per channel:", [round(float(x), 3) for x in d])
