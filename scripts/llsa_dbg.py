import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2302_13451_b200 as s
for shape, L, R in (((2, 2, 1750, 64), 32, 8), ((1, 2, 200, 64), 16, 4)):
    C = R + 1
    q, k, v = synth.qkv(2, (C,) + shape, "bf16")
    do = synth.grad_out(2, (C,) + shape, "bf16")
    dev = lambda x: torch.tensor(np.asarray(x), dtype=torch.bfloat16, device="cuda")
    tq, tk, tv, tdo = (dev(x) for x in (q, k, v, do))
    o, lse = s.llsa_forward(tq, tk, tv, L, R)
    dq, dk, dv = s.llsa_backward(tq, tk, tv, o, lse, tdo, L, R)
    G = oracle.llsa.llsa_backward(q, k, v, do, L, R)
    for name, got, ref in (("dQ", dq, G[0]), ("dK", dk, G[1]), ("dV", dv, G[2])):
        e = np.abs(got.double().cpu().numpy() - ref)
        print(shape, L, R, name, "per-channel max err", [round(float(e[c].max()), 4) for c in range(C)])
        if e.max() > 0.05:
            idx = np.argwhere(e > 0.05)
            print("   bad (c,b,h,t,d) first:", idx[:6].tolist(), "count", len(idx), "t values", sorted(set(idx[:, 3].tolist()))[:20])
