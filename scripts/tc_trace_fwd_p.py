"""Phase timeline (clock64) of CTA 0 of the stored-band forward (sa_fwd_tc<CW, PST>) at the bench shape
(debug aid): QK issued, S waited/issued, softmax start / P written, PV ready / issued, O epilogue."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
q, k, v = (torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(3))
buf = torch.zeros(1024 + 512, dtype=torch.int64, device="cuda")
lib = s.lib()
lib.sattn_debug_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    s.sa_forward_p(q, k, v, L, R, impl="tc")
torch.cuda.synchronize()
lib.sattn_debug_trace(ctypes.c_void_p(buf.data_ptr()))
s.sa_forward_p(q, k, v, L, R, impl="tc")
torch.cuda.synchronize()
lib.sattn_debug_trace(None)
t = buf[:1024].view(16, 64).cpu()
t0 = int(t[0, 0])
names = ["qk_issue", "S_full", "S_issued", "PV_ready", "wg_sfull", "wg_pfull", "wg_ofull", "epi_done", "PV_issued", "v_issue"]
print("tile " + " ".join(f"{nm:>9s}" for nm in names))
for kk in range(10):
    print(f"{kk:4d} " + " ".join(f"{(int(t[e, kk]) - t0) if t[e, kk] else -1:9d}" for e in range(10)))
