"""LLSA parity diagnostics for one case: per-output, per-channel max error, location, ulps.
usage: python scripts/llsa_case_diag.py B H T D L R broadcast(0/1) [impl]"""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle, synth
import paper_2302_13451_b200 as s
B, H, T, D, L, R, bc = map(int, sys.argv[1:8]); impl = sys.argv[8] if len(sys.argv) > 8 else "auto"
dt = "bf16"; shape = (B, H, T, D); C = R + 1
q, k, v = synth.qkv(2, ((1,) if bc else (C,)) + shape, dt); do = synth.grad_out(2, (C,) + shape, dt)
if bc:
    q, k, v = (x[0] for x in (q, k, v))
dev = lambda x: torch.tensor(np.asarray(x), dtype=torch.bfloat16, device="cuda")
tq, tk, tv, tdo = map(dev, (q, k, v, do))
Q, K, V = (oracle.llsa.channelize(x, R) if bc else x for x in (q, k, v))
O, LSE = oracle.llsa.llsa_forward(Q, K, V, L, R)
G = oracle.llsa.llsa_backward(Q, K, V, do, L, R)
o, lse = s.llsa_forward(tq, tk, tv, L, R, broadcast=bool(bc), impl=impl)
g = s.llsa_backward(tq, tk, tv, o, lse, tdo, L, R, broadcast=bool(bc), impl=impl)
for name, a, ref in zip(("O", "LSE", "dQ", "dK", "dV"), (o, lse) + tuple(g), (O, LSE) + tuple(G)):
    a = a.double().cpu().numpy(); e = np.abs(a - ref); i = np.unravel_index(e.argmax(), e.shape)
    ulp = 2.0 ** (np.floor(np.log2(np.abs(ref[i]) + 1e-30)) - 7)
    print(name, "max %.4g at %s ref %.5g got %.5g ulps %.2f" % (e.max(), tuple(int(x) for x in i), ref[i], a[i], e.max() / ulp),
          "per-ch", np.round([float(e[c].max()) for c in range(C)], 4) if name != "LSE" else "")
