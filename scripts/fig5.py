"""NEXT-1: the paper's Fig. 5 experiment on B200.

d_k = 64, N_T = 1000 frames, H in {8, 16} heads, receptive field W = A + B + 1 = 10 ... 490 in
steps of 10 (look-back B = ceil((W-1)/2), look-ahead A = floor((W-1)/2)), 5 repeats, mean.
For each point: peak device memory of one SA forward + backward through the C ABI (bf16; the
tensor-core kernels at every W: W <= 65 in one launch, wider bands as log-sum-exp-merged sub-bands
of width <= 49) per training vector (frame),
and its time, for both SA modes -- LSE + recompute (sa_forward / sa_backward) and the paper's own
stored band a_t (sa_forward_p / sa_backward_p; one tensor-core pass for W <= 49, 48-column sub-bands beyond) -- next to masked
acausal attention (MAA) as PyTorch computes it (dense T x T scores,
boolean band mask, softmax, autograd), which is what the paper compares against.  Writes
profiles/r1/fig5.json and prints a markdown table.  Inputs are synthetic (iid N(0,1))."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2302_13451_b200 as s

T, D, REP = 1000, 64, 5
dev = torch.device("cuda")


def band(W):
    Lb = W // 2
    return Lb, W - 1 - Lb          # (look-back L, look-ahead R)


def measure(fn, reps=REP):
    torch.cuda.synchronize()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated()
    fn()
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return peak, sum(ts) / len(ts)


def run(H, B=8):
    g = torch.Generator(device=dev).manual_seed(5)
    q, k, v, do = (torch.randn(B, H, T, D, device=dev, generator=g).to(torch.bfloat16) for _ in range(4))
    rows = []
    for W in range(10, 491, 10):
        L, R = band(W)

        def sa():
            o, lse = s.sa_forward(q, k, v, L, R)
            s.sa_backward(q, k, v, o, lse, do, L, R)

        def sa_band():
            o, lse, pb = s.sa_forward_p(q, k, v, L, R)
            s.sa_backward_p(q, k, v, o, pb, do, L, R)

        idx = torch.arange(T, device=dev)
        mask = (idx[None, :] >= idx[:, None] - L) & (idx[None, :] <= idx[:, None] + R)

        def maa():
            qq, kk, vv = (x.detach().requires_grad_(True) for x in (q, k, v))
            z = (qq @ kk.transpose(-1, -2)) * D ** -0.5
            z = z.masked_fill(~mask, float("-inf"))
            y = torch.softmax(z.float(), -1).to(torch.bfloat16) @ vv
            y.backward(do)

        m_sa, t_sa = measure(sa)
        m_sb, t_sb = measure(sa_band)
        m_maa, t_maa = measure(maa)
        frames = B * T
        rows.append({"H": H, "W": W, "L": L, "R": R, "kernels": "tcgen05" if W <= 65 else f"tcgen05 x {-(-W // 49)} sub-bands",
                     "band_kernels": "tcgen05" if W <= 49 else (f"tcgen05 fwd + tcgen05 x {-(-W // 48)} sub-band bwd" if W <= 64
                                                              else f"ffma fwd + tcgen05 x {-(-W // 48)} sub-band bwd"),
                     "sa_bytes_per_frame": m_sa / frames, "maa_bytes_per_frame": m_maa / frames,
                     "sa_band_bytes_per_frame": m_sb / frames,
                     "sa_ms": t_sa, "sa_band_ms": t_sb, "maa_ms": t_maa})
        del mask
    return rows


def main():
    out = {"what": "Fig. 5 (P:L344-354) on B200: SA vs MAA peak memory per training vector and time per fwd+bwd",
           "T": T, "D": D, "B": 8, "repeats": REP, "dtype": "bf16", "rows": []}
    for H in (8, 16):
        out["rows"] += run(H)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r2", "fig5.json")
    os.makedirs(os.path.dirname(path), exist_ok=True)
    json.dump(out, open(path, "w"), indent=1)
    lines = ["| H | W | kernels (lse / band) | SA KB/frame | SA-band KB/frame | MAA KB/frame | SA ms | SA-band ms | MAA ms |",
             "|---|---|---|---|---|---|---|---|---|"]
    for r in out["rows"]:
        if r["W"] in (10, 20, 40, 50, 70, 100, 150, 200, 300, 400, 490):
            lines.append(f"| {r['H']} | {r['W']} | {r['kernels']} / {r['band_kernels']} | {r['sa_bytes_per_frame'] / 1024:.1f} | "
                         f"{r['sa_band_bytes_per_frame'] / 1024:.1f} | {r['maa_bytes_per_frame'] / 1024:.1f} | "
                         f"{r['sa_ms']:.3f} | {r['sa_band_ms']:.3f} | {r['maa_ms']:.3f} |")
    slower = [(r["H"], r["W"]) for r in out["rows"] if r["sa_ms"] >= r["maa_ms"]]
    lines.append("")
    lines.append(f"SA (LSE mode) slower than MAA at: {slower or 'no W'}")
    print("\n".join(lines))
    open(path.replace(".json", ".md"), "w").write("# Fig. 5 sweep on B200 (scripts/fig5.py, round 2)\n\n" + "\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
