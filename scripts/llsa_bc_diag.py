"""Diagnose LLSA broadcast dK error: TC vs FFMA vs oracle, error in bf16 ulps of the reference."""
import numpy as np, torch, sys
sys.path.insert(0, ".")
import oracle, synth
import paper_2302_13451_b200 as s
dt = "bf16"; shape = (2, 2, 1750, 64); L, R = 32, 8; C = R + 1
q, k, v = synth.qkv(2, (1,) + shape, dt); do = synth.grad_out(2, (C,) + shape, dt)
q, k, v = (x[0] for x in (q, k, v))
dev = lambda x: torch.tensor(np.asarray(x), dtype=torch.bfloat16, device="cuda")
tq, tk, tv, tdo = map(dev, (q, k, v, do))
Q, K, V = (oracle.llsa.channelize(x, R) for x in (q, k, v))
G = oracle.llsa.llsa_backward(Q, K, V, do, L, R)
for impl in ("tc", "ffma"):
    o, lse = s.llsa_forward(tq, tk, tv, L, R, broadcast=True, impl=impl)
    g = s.llsa_backward(tq, tk, tv, o, lse, tdo, L, R, broadcast=True, impl=impl)
    for name, a, ref in zip(("dQ", "dK", "dV"), g, G):
        a = a.double().cpu().numpy(); e = np.abs(a - ref); i = np.unravel_index(e.argmax(), e.shape)
        ulp = 2.0 ** (np.floor(np.log2(np.abs(ref[i]) + 1e-30)) - 7)
        per_ch = [float(e[c].max()) for c in range(C)]
        print(impl, name, "max", e.max(), "at", i, "ref", ref[i], "got", a[i], "ulps", e.max() / ulp,
              "maxref", np.abs(ref).max(), "per-ch", np.round(per_ch, 4))
