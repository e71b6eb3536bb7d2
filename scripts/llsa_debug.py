"""LLSA forward: tensor-core vs FFMA kernel (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
for (B, H, T, L, R, bc) in [(1, 1, 64, 32, 8, False), (1, 2, 300, 32, 8, False), (2, 3, 1750, 32, 8, False),
                            (1, 2, 300, 32, 8, True), (1, 2, 200, 16, 4, False), (1, 1, 100, 3, 5, False)]:
    C = R + 1
    shp = (B, H, T, 64) if bc else (C, B, H, T, 64)
    q, k, v = (torch.randn(*shp, device="cuda").to(torch.bfloat16) for _ in range(3))
    try:
        o1, l1 = s.llsa_forward(q, k, v, L, R, impl="tc", broadcast=bc)
        torch.cuda.synchronize()
    except Exception as e:
        print((B, H, T, L, R, bc), "TC ERR", e); continue
    o2, l2 = s.llsa_forward(q, k, v, L, R, impl="ffma", broadcast=bc)
    d = (o1.float() - o2.float()).abs()
    print((B, H, T, L, R, bc), "O", float(d.max()), "LSE", float((l1 - l2).abs().max()), flush=True)
    if float(d.max()) > 0.05:
        print("  per channel max:", [round(float(d[c].max()), 3) for c in range(C)])
        dc = d.amax(dim=(1, 2, 4))
        print("  bad rows ch0:", torch.nonzero(dc[0] > 0.05).flatten()[:10].tolist(), " ch8:", torch.nonzero(dc[-1] > 0.05).flatten()[:10].tolist())
