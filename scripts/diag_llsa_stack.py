"""Diagnostic: bf16 LLSA 12-layer stack backward vs the oracle — where is the error?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import oracle
import synth
import paper_2302_13451_b200 as s

B, H, T, D, L, R = 1, 2, 1750, 64, 32, 8
for n in (1, 2, 4, 8, 12):
    for dt in ("bf16", "f32"):
        tdt = torch.float32 if dt == "f32" else torch.bfloat16
        x = synth.round_to(synth.normal(8, "X", (B, H, T, D)), dt)
        dy = synth.round_to(synth.normal(8, "dY", (R + 1, B, H, T, D)), dt)
        tx = torch.tensor(x, dtype=tdt, device="cuda")
        tdy = torch.tensor(dy, dtype=tdt, device="cuda")
        y, saved = s.stack_forward(tx, L, R, n, s.MODE_LLSA)
        dx = s.stack_backward(tx, saved, tdy, L, R, n, s.MODE_LLSA)
        Y, _ = oracle.stack.stack_forward(x, L, R, n, "llsa")
        DX = oracle.stack.stack_backward(x, dy, L, R, n, "llsa")
        ey = np.abs(y.double().cpu().numpy() - Y)
        e = np.abs(dx.double().cpu().numpy() - DX)
        idx = np.argsort(e.ravel())[::-1][:6]
        pos = [np.unravel_index(i, e.shape) for i in idx]
        print(f"n={n} {dt}: Y err {ey.max():.3g} (|Y| {np.abs(Y).max():.3g}); dX err max {e.max():.3g} "
              f"p99.99 {np.quantile(e, 0.9999):.3g} median {np.median(e):.3g} |DX| max {np.abs(DX).max():.3g}")
        if dt == "bf16":
            print("   worst (b,h,t,d) err got ref:", [(tuple(int(v) for v in p), round(float(e[p]), 3),
                                                     round(float(dx.double().cpu().numpy()[p]), 3), round(float(DX[p]), 3)) for p in pos[:4]])
            # per-t error profile
            et = e.max(axis=(0, 1, 3))
            bad = np.where(et > 0.5)[0]
            print("   t with err > 0.5:", bad[:40], len(bad))
