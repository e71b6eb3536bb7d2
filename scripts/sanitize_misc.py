"""Stack driver (SA and LLSA, fwd + bwd) and the incremental streams (LLSA, SA) at small sizes,
for compute-sanitizer."""
import os
import sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import torch
import paper_2302_13451_b200 as s

g = torch.Generator(device="cuda").manual_seed(0)
B, H, T, D, L, R, NLy = 1, 2, 200, 64, 16, 4, 3
for dt in (torch.bfloat16, torch.float32):
    x0 = torch.randn(B, H, T, D, device="cuda", generator=g).to(dt)
    for mode in (s.MODE_SA, s.MODE_LLSA):
        y, saved = s.stack_forward(x0, L, R, NLy, mode)
        dy = torch.randn(y.shape, device="cuda", generator=g).to(dt)
        s.stack_backward(x0, saved, dy, L, R, NLy, mode)
    for cls in (s.LLSAStream, s.SAStream):
        for (Ls, Rs) in ((L, R), (32, 16), (3, 1)):   # (32, 16): two query m-tiles on the mma.sync step
            st = cls(B, H, D, Ls, Rs, NLy, dtype=dt)
            for t in range(40):
                st.step(torch.randn(B, H, D, device="cuda", generator=g).to(dt))
            st.flush()
torch.cuda.synchronize()
print("done")
