"""LLSA per-layer fwd / bwd GPU time (CUDA graphs) at the bench shape: debug aid."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L = 8, 12, 1750, 64, 32
R = int(sys.argv[1]) if len(sys.argv) > 1 else 8
C = R + 1
N = 4
x = [[torch.randn(C, B, H, T, D, device="cuda").to(torch.bfloat16) for _ in range(4)] for _ in range(N)]
outs = [s.llsa_forward(q, k, v, L, R) for q, k, v, _ in x]
g = [torch.empty_like(x[0][0]) for _ in range(3)]
lib = s.lib()
d = s.make_desc(B, H, T, D, L, R, s.BF16)
nws = lib.llsa_backward_workspace(ctypes.byref(d))
ws = torch.empty(nws, dtype=torch.uint8, device="cuda")
P = lambda t: ctypes.c_void_p(t.data_ptr())
def fwd():
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for (q, k, v, _), (o, lse) in zip(x, outs):
        assert lib.llsa_forward(ctypes.byref(d), P(q), P(k), P(v), P(o), P(lse), sp) == 0
def bwd():
    sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for (q, k, v, do), (o, lse) in zip(x, outs):
        assert lib.llsa_backward(ctypes.byref(d), P(q), P(k), P(v), P(o), P(lse), P(do), P(g[0]), P(g[1]), P(g[2]), P(ws), nws, sp) == 0
fwd(); bwd(); torch.cuda.synchronize()
st = torch.cuda.Stream()
gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
with torch.cuda.graph(gf, stream=st): fwd()
with torch.cuda.graph(gb, stream=st): bwd()
for _ in range(2): gf.replay(); gb.replay()
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record(); gf.replay(); e[1].record(); gb.replay(); e[2].record(); torch.cuda.synchronize()
f = e[0].elapsed_time(e[1]) / N * 1e3; b = e[1].elapsed_time(e[2]) / N * 1e3
unit = C * B * H * T
print(f"llsa: fwd {f:.1f} us ({516*unit/f/1e3:.0f} GB/s)  bwd {b:.1f} us ({1028*unit/b/1e3:.0f} GB/s)")
