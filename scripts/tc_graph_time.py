"""Per-kernel GPU time via CUDA graphs (removes host launch overhead): debug aid."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
N = 12
impl = sys.argv[1] if len(sys.argv) > 1 else "tc"
qs = [[torch.randn(B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4)] for _ in range(N)]
outs = [s.sa_forward(q, k, v, L, R, impl=impl) for q, k, v, _ in qs]
grads = [[torch.empty_like(q) for _ in range(3)] for q, *_ in qs]
ws = torch.empty(2 * B * H * ((T + 3) // 4 * 4) * 4, dtype=torch.uint8, device="cuda")
import ctypes
lib = s.lib()
d = s.make_desc(B, H, T, D, L, R, s.BF16, impl=impl)
P = lambda t: ctypes.c_void_p(t.data_ptr())
def fwd():
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for (q, k, v, _), (o, lse) in zip(qs, outs):
        assert lib.sa_forward(ctypes.byref(d), P(q), P(k), P(v), P(o), P(lse), sp) == 0
def bwd():
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for (q, k, v, do), (o, lse), (dq, dk, dv) in zip(qs, outs, grads):
        assert lib.sa_backward(ctypes.byref(d), P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk), P(dv), P(ws), ws.numel(), sp) == 0
fwd(); bwd(); torch.cuda.synchronize()
st = torch.cuda.Stream()
gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(gf, stream=st):
    fwd()
with torch.cuda.graph(gb, stream=st):
    bwd()
for _ in range(3):
    gf.replay(); gb.replay()
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
reps = 10
e[0].record()
for _ in range(reps): gf.replay()
e[1].record()
for _ in range(reps): gb.replay()
e[2].record()
torch.cuda.synchronize()
f = e[0].elapsed_time(e[1]) / reps / N * 1e3
b = e[1].elapsed_time(e[2]) / reps / N * 1e3
unit = B * H * T
print(f"{impl} graphs: fwd {f:.1f} us ({516*unit/f/1e3:.0f} GB/s)  bwd {b:.1f} us ({1028*unit/b/1e3:.0f} GB/s)  step {(f+b)*N/1e3:.3f} ms -> {B*T/((f+b)*N/1e6)/1e6:.2f} M frames/s")
