"""Stream vs offline GPU stack / oracle error by depth (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2302_13451_b200 as s
B, H, T, D, L, R = 1, 2, 200, 64, 32, 8
x = synth.normal(6, "X", (B, H, T, D))
xr = synth.round_to(x, "bf16")
tx = torch.tensor(xr, dtype=torch.bfloat16, device="cuda")
for mode in ("llsa", "sa"):
    for n in (1, 2, 3, 4, 6, 8, 12):
        cls = s.LLSAStream if mode == "llsa" else s.SAStream
        st = cls(B, H, D, L, R, n, dtype=torch.bfloat16)
        ys = torch.full((B, H, T, D), float("nan"), device="cuda", dtype=torch.bfloat16)
        for h in range(T):
            r = st.step(tx[:, :, h].contiguous())
            if r is not None:
                ys[:, :, r[0]] = r[1]
        tail = st.flush()
        ys[:, :, T - tail.shape[0]:] = tail.permute(1, 2, 0, 3)
        y_off, _ = s.stack_forward(tx, L, R, n, s.MODE_LLSA if mode == "llsa" else s.MODE_SA)
        y_off = y_off[R] if mode == "llsa" else y_off
        Y = (oracle.stream.stream_all if mode == "llsa" else oracle.stream.sa_stream_all)(xr, L, R, n)[0]
        a = ys.double().cpu().numpy(); b = y_off.double().cpu().numpy()
        e = np.abs(a - b); eo = np.abs(a - Y); eoff = np.abs(b - Y)
        t_bad = np.unravel_index(e.argmax(), e.shape)
        print(mode, n, "stream-offline", round(e.max(), 4), "at", t_bad, "stream-oracle", round(eo.max(), 4),
              "offline-oracle", round(eoff.max(), 4), "max|Y|", round(np.abs(Y).max(), 3), flush=True)
