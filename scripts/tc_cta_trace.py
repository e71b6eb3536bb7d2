"""Per-CTA start/end (globaltimer) of the tensor-core forward (debug aid)."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
q, k, v = (torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(3))
buf = torch.zeros(1024 + 512, dtype=torch.int64, device="cuda")
lib = s.lib(); lib.sattn_debug_trace.argtypes = [ctypes.c_void_p]
for _ in range(3): s.sa_forward(q, k, v, L, R, impl="tc")
torch.cuda.synchronize()
lib.sattn_debug_trace(ctypes.c_void_p(buf.data_ptr()))
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); s.sa_forward(q, k, v, L, R, impl="tc"); e1.record()
torch.cuda.synchronize(); lib.sattn_debug_trace(None)
t = buf[1024:1024 + 296].view(148, 2).cpu().double()
t0 = t[:, 0].min()
st = (t[:, 0] - t0) / 1e3; en = (t[:, 1] - t0) / 1e3
print(f"event time {e0.elapsed_time(e1)*1e3:.1f} us; CTA start min/med/max {st.min():.2f}/{st.median():.2f}/{st.max():.2f} us; end min/med/max {en.min():.2f}/{en.median():.2f}/{en.max():.2f} us")
print("durations (us) by CTA (first 12 have 10 tiles):", [round(float(x), 1) for x in (en - st)[:16]])
