"""Run a few incremental LLSA and SA steps (B=1 and B=64, 12 layers, base shape) for ncu (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2302_13451_b200 as s
for cls in (s.LLSAStream, s.SAStream):
    for nb in (1, 64):
        st = cls(nb, 12, 64, 32, 8, 12, dtype=torch.bfloat16, device="cuda")
        xs = torch.randn(64, nb, 12, 64, device="cuda").to(torch.bfloat16)
        y = torch.empty(nb, 12, 64, device="cuda", dtype=torch.bfloat16)
        for i in range(64):
            st.step_into(xs[i], y)
        torch.cuda.synchronize()
