"""Where does LLSA TC dK (channel R) error concentrate? broadcast and dense inputs."""
import numpy as np, torch, sys
sys.path.insert(0, ".")
import oracle, synth
import paper_2302_13451_b200 as s
dt = "bf16"; shape = (2, 2, 1750, 64); L, R = 32, 8; C = R + 1
dev = lambda x: torch.tensor(np.asarray(x), dtype=torch.bfloat16, device="cuda")
for bc in (True, False):
    q, k, v = synth.qkv(2, ((1,) if bc else (C,)) + shape, dt); do = synth.grad_out(2, (C,) + shape, dt)
    if bc:
        q, k, v = (x[0] for x in (q, k, v))
    tq, tk, tv, tdo = map(dev, (q, k, v, do))
    Q, K, V = (oracle.llsa.channelize(x, R) if bc else x for x in (q, k, v))
    G = oracle.llsa.llsa_backward(Q, K, V, do, L, R)
    res = {}
    for impl in ("tc", "ffma"):
        o, lse = s.llsa_forward(tq, tk, tv, L, R, broadcast=bc, impl=impl)
        g = s.llsa_backward(tq, tk, tv, o, lse, tdo, L, R, broadcast=bc, impl=impl)
        res[impl] = [x.double().cpu().numpy() for x in g]
    for j, name in enumerate(("dQ", "dK", "dV")):
        ref = G[j]
        for impl in ("tc", "ffma"):
            e = np.abs(res[impl][j] - ref)[R]          # channel R, [B,H,T,D]
            et = e.max(axis=(0, 1, 3))
            top = np.argsort(et)[::-1][:8]
            print(bc, impl, name, "chR max", e.max(), "mean", e.mean(), "top t", list(zip(top.tolist(), np.round(et[top], 4).tolist())))
        d = np.abs(res["tc"][j] - res["ffma"][j])[R]
        print(bc, name, "tc-ffma chR max", d.max(), "mean", d.mean())
