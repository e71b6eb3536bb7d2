"""CPU oracle for the SA / LLSA hot path of arXiv 2302.13451 — TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct numpy fp64 implementations of what the GPU path
computes, each function citing the PAPER.md passage it follows (P:Lx = line x
of /root/reference/PAPER.md; SPEC S:Lx likewise; readings G1..G23 are listed in
DESIGN.md §3).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
/ --impl reference legs may import this package.  It shares no code with the
CUDA path (paper_2302_13451_b200/), and the CUDA path never imports it.

Modules
  sa       AA / MAA / SA forward+backward as dense masked attention (Eq. 1-13)
  llsa     LLSA forward+backward, gather form of Eq. 14-15 (+ flattened-mask form)
  stack    n-layer tied-QKV stack with the X_{l+1} = (X_l + Y_l)/2 rule (G12)
  stream   per-frame incremental LLSA recurrence over a ring of channel-R frames, and the
           incremental SA stack (infer_sa: latency n_layers x R)
  latency  structural receptive-field propagation and Table-3 latency arithmetic
  counts   score-element counts of P:L87 / P:L337-342

Parity status: every function here is pinned by a
`-m "not gpu"` test in tests/test_oracle_*.py to something other than itself,
except the LLSA q/k gradient *as the paper's supplementary writes it* (not in
the reference; we pin the exact gradient by finite differences instead).
"""
from . import sa, llsa, stack, stream, latency, counts  # noqa: F401
