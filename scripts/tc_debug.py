"""Quick tensor-core vs FFMA comparison on GPU (debug aid, not a test)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s

torch.manual_seed(0)
for (B, H, T, L, R) in [(1, 1, 128, 32, 8), (1, 2, 300, 32, 8), (2, 3, 1750, 32, 8), (1, 2, 500, 32, 16), (1, 1, 200, 0, 0)]:
    q, k, v, do = (torch.randn(B, H, T, 64, device="cuda").to(torch.bfloat16) for _ in range(4))
    res = {}
    for impl in ("ffma", "tc"):
        try:
            o, lse = s.sa_forward(q, k, v, L, R, impl=impl)
            g = s.sa_backward(q, k, v, o, lse, do, L, R, impl=impl)
            torch.cuda.synchronize()
            res[impl] = (o, lse) + g
        except Exception as e:
            print(impl, "ERR", e)
    if len(res) == 2:
        names = ["O", "LSE", "dQ", "dK", "dV"]
        errs = {n: float((a.float() - b.float()).abs().max()) for n, a, b in zip(names, res["ffma"], res["tc"])}
        print((B, H, T, L, R), errs, flush=True)
        if errs["O"] > 0.05:
            d = (res["ffma"][0].float() - res["tc"][0].float()).abs()[0, 0]
            print("  O row err:", d.max(-1).values[:16].tolist())
            print("  O col err row0:", d[0, :16].tolist())
