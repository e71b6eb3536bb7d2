"""Experiment: stored-band SA backward (12 layers, bench shape) with each layer's call split into
`nc` batch chunks, so K2's re-reads of V / dO / band (read by K1 just before) can hit L2.
Prints per-layer backward time for nc in (1, 2, 3, 4, 8).  Debug aid."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
B, H, T, D, L, R, NL = 8, 12, 1750, 64, 32, 8, 12
lib = s.lib()
dev = torch.device("cuda", 0)
bf = torch.bfloat16
shp = (B, H, T, D)
d0 = s.make_desc(B, H, T, D, L, R, s.BF16)
ld = int(lib.sa_p_ld(ctypes.byref(d0)))
rnd = lambda *sh: torch.randn(*sh, device=dev).to(bf)
Q, K, V, dO = ([rnd(*shp) for _ in range(NL)] for _ in range(4))
O = [torch.empty(shp, device=dev, dtype=bf) for _ in range(NL)]
LSE = [torch.empty(shp[:-1], device=dev, dtype=torch.float32) for _ in range(NL)]
Pb = [torch.empty(shp[:-1] + (ld,), device=dev, dtype=bf) for _ in range(NL)]
dQ, dK, dV = ([torch.empty(shp, device=dev, dtype=bf) for _ in range(NL)] for _ in range(3))
P = lambda t: ctypes.c_void_p(t.data_ptr())
sp = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for l in range(NL):
    assert lib.sa_forward_p(ctypes.byref(d0), P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), P(Pb[l]), sp()) == 0
torch.cuda.synchronize()
for nc in (1, 2, 4, 8):
    bc = B // nc
    dc = s.make_desc(bc, H, T, D, L, R, s.BF16)
    nws = lib.sa_backward_p_workspace(ctypes.byref(dc))
    ws = torch.empty(max(nws, 1), device=dev, dtype=torch.uint8)
    def bwd():
        for l in reversed(range(NL)):
            for c in range(nc):
                sl = slice(c * bc, (c + 1) * bc)
                st = lib.sa_backward_p(ctypes.byref(dc), P(Q[l][sl]), P(K[l][sl]), P(V[l][sl]), P(O[l][sl]), P(Pb[l][sl]),
                                       P(dO[l][sl]), P(dQ[l][sl]), P(dK[l][sl]), P(dV[l][sl]), P(ws), nws, sp())
                assert st == 0
    bwd(); torch.cuda.synchronize()
    cap = torch.cuda.Stream(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        bwd()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): g.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 10 / NL
    print(f"chunks {nc}: backward {us:.1f} us/layer, frac {978 * B * H * T / (us * 1e-6) / 1e9 / 6556:.3f}", flush=True)
