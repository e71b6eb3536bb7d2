"""Phase timeline of CTA 0 of the fused tensor-core SA backward + per-CTA spans (debug aid)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
q, k, v, do = (torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4))
o, lse = s.sa_forward(q, k, v, L, R, impl="tc")
buf = torch.zeros(1024 + 512, dtype=torch.int64, device="cuda")
lib = s.lib()
lib.sattn_debug_trace.argtypes = [ctypes.c_void_p]
for _ in range(3):
    s.sa_backward(q, k, v, o, lse, do, L, R, impl="tc")
torch.cuda.synchronize()
lib.sattn_debug_trace(ctypes.c_void_p(buf.data_ptr()))
s.sa_backward(q, k, v, o, lse, do, L, R, impl="tc")
torch.cuda.synchronize()
lib.sattn_debug_trace(None)
t = buf[:1024].view(16, 64).cpu()
t0 = int(t[0, 0])
names = ["tma_issue", "rows_done", "sfull", "dpfull", "PdS_done", "kvfull", "dqfull", "epi_done"]
n = int((t[0] > 0).sum())
print("tile " + " ".join(f"{nm:>10s}" for nm in names))
for kk in range(n):
    print(f"{kk:4d} " + " ".join(f"{(int(t[e, kk]) - t0) if t[e, kk] else -1:10d}" for e in range(8)))
print("pre-grid-sync", int(t[8, 0]) - t0)
c = buf[1024:1024 + 296].view(148, 2).cpu().double()
st = (c[:, 0] - c[:, 0].min()) / 1e3; en = (c[:, 1] - c[:, 0].min()) / 1e3
print(f"CTA start min/med/max {st.min():.2f}/{st.median():.2f}/{st.max():.2f} us; end {en.min():.2f}/{en.median():.2f}/{en.max():.2f} us")
# untraced timing, L2-cold-ish distinct buffers (like the bench)
NL = 6
bufs = [[torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4)] for _ in range(NL)]
outs = [s.sa_forward(b[0], b[1], b[2], L, R, impl="tc") for b in bufs]
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for b, (oo, ll) in zip(bufs, outs):
        s.sa_backward(b[0], b[1], b[2], oo, ll, b[3], L, R, impl="tc")
    e1.record(); torch.cuda.synchronize()
    print(f"eager sa_backward x{NL}: {e0.elapsed_time(e1) * 1e3 / NL:.1f} us/call")
