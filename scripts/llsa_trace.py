"""Debug: phase timeline of the fused LLSA backward's CTA 0 (clock64 stamps per item)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
C = R + 1
q, k, v, do = (torch.randn(C, B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = s.llsa_forward(q, k, v, L, R)
tr = torch.zeros(16 * 64, dtype=torch.int64, device="cuda")
lib = s.lib()
lib.sattn_debug_trace.argtypes = [ctypes.c_void_p]
for it in range(3):
    lib.sattn_debug_trace(ctypes.c_void_p(tr.data_ptr() if it == 2 else 0))
    s.llsa_backward(q, k, v, o, lse, do, L, R)
    torch.cuda.synchronize()
lib.sattn_debug_trace(None)
t = tr.view(16, 64).cpu().numpy().astype(np.int64)
names = ["start", "full", "stair", "sfull", "P", "dpfull", "dsfull", "hmma", "done", "tfree"]
n = int((t[9] > 0).sum())
base = t[0, 0]
print("items traced", n)
for k in range(min(n, 12)):
    print(k, " ".join(f"{names[e]}:{(t[e, k] - base):7d}" for e in range(10)))
d = np.diff(t[:10, 2:n], axis=0)
print("mean phase durations (cycles), items 2..:")
for e in range(9):
    print(f"  {names[e]}->{names[e+1]}: {d[e].mean():8.0f}")
print("item period per WG (start k -> start k+2):", np.mean(t[0, 4:n] - t[0, 2:n - 2]))
