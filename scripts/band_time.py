"""Time the stored-band mode (sa_forward_p + sa_backward_p) against the LSE-recompute path
at the bench shape: 12 layers of distinct buffers, each pass captured in a CUDA graph,
CUDA events around the replay, median of 10, reported per layer."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2302_13451_b200 as s

B, H, T, D, L, R = 8, 12, 1750, 64, 32, 8
if len(sys.argv) > 2:
    L, R = int(sys.argv[1]), int(sys.argv[2])
NL = 12
g = torch.Generator(device="cuda").manual_seed(0)
layers = [[torch.randn(B, H, T, D, device="cuda", generator=g).bfloat16() for _ in range(4)] for _ in range(NL)]


def graph_time(fn):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            fn()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / NL)
    return sorted(ts)[5]


res = {}
for impl in ("auto", "ffma"):
    outs = [s.sa_forward(q, k, v, L, R, impl=impl) for q, k, v, _ in layers]
    ws = torch.empty(s.lib().sa_backward_workspace(s.ctypes.byref(s.make_desc(B, H, T, D, L, R, s.BF16))),
                     device="cuda", dtype=torch.uint8)
    res[f"fwd_{impl}"] = graph_time(lambda: [s.sa_forward(q, k, v, L, R, impl=impl) for q, k, v, _ in layers])
    res[f"bwd_{impl}"] = graph_time(lambda: [s.sa_backward(q, k, v, o, l, do, L, R, impl=impl, ws=ws)
                                             for (q, k, v, do), (o, l) in zip(layers, outs)])
    outp = [s.sa_forward_p(q, k, v, L, R, impl=impl) for q, k, v, _ in layers]
    res[f"fwd_p_{impl}"] = graph_time(lambda: [s.sa_forward_p(q, k, v, L, R, impl=impl) for q, k, v, _ in layers])
    res[f"bwd_p_{impl}"] = graph_time(lambda: [s.sa_backward_p(q, k, v, o, p, do, L, R, impl=impl, ws=ws)
                                               for (q, k, v, do), (o, _, p) in zip(layers, outp)])
print(f"(L,R)=({L},{R}) per layer us:", {k_: round(v_, 1) for k_, v_ in res.items()},
      "band MB/layer", round(outp[0][2].numel() * 2 / 1e6, 1))
