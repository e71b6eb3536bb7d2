#!/bin/bash
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python - <<'PY'
import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2302_13451_b200 as s
B,H,T,D,L,R = 8,12,1750,64,32,32
g = torch.Generator("cuda").manual_seed(0)
q,k,v,do = (torch.randn(B,H,T,D,device="cuda",generator=g).to(torch.bfloat16) for _ in range(4))
for impl in ("auto","ffma"):
    o,lse = s.sa_forward(q,k,v,L,R,impl=impl)
    for _ in range(3): s.sa_backward(q,k,v,o,lse,do,L,R,impl=impl)
    torch.cuda.synchronize()
    e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): s.sa_backward(q,k,v,o,lse,do,L,R,impl=impl)
    e1.record(); torch.cuda.synchronize()
    f0=torch.cuda.Event(enable_timing=True); f1=torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(10): s.sa_forward(q,k,v,L,R,impl=impl)
    f1.record(); torch.cuda.synchronize()
    print(f"(32,32) {impl}: fwd {f0.elapsed_time(f1)/10*1e3:.1f} us, bwd {e0.elapsed_time(e1)/10*1e3:.1f} us")
PY
