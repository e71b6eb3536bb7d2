"""Phase timeline (clock64 cycles) of CTA 0 of the stored-band dK/dV kernel (K2) at the bench shape
(debug aid): per tile k, when the producer issued its loads, when the warpgroup passed full, read
the band window, saw dP, wrote P/dS, saw dV/dK, finished the epilogue."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
q, k, v, do = (torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse, pb = s.sa_forward_p(q, k, v, L, R, impl="tc")
buf = torch.zeros(1024 + 512, dtype=torch.int64, device="cuda")
lib = s.lib()
lib.sattn_debug_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    s.sa_backward_p(q, k, v, o, pb, do, L, R, impl="tc")
torch.cuda.synchronize()
lib.sattn_debug_trace(ctypes.c_void_p(buf.data_ptr()))
s.sa_backward_p(q, k, v, o, pb, do, L, R, impl="tc")
torch.cuda.synchronize()
lib.sattn_debug_trace(None)
t = buf[:1024].view(16, 64).cpu()
t0 = int(t[0, 0])
names = ["tma_issue", "full", "-", "P_read", "dpfull", "PdS_written", "kvfull", "epi_done"]
n = int((t[0] > 0).sum())
print("tile " + " ".join(f"{nm:>12s}" for nm in names))
for kk in range(n):
    print(f"{kk:4d} " + " ".join(f"{(int(t[e, kk]) - t0) if t[e, kk] else -1:12d}" for e in range(8)))
