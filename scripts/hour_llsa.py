"""Run only the M4 LLSA hour-stream measurement of bench.py (debug aid)."""
import json, os, sys, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2302_13451_b200 as s
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
rnd = lambda *sh: torch.randn(*sh, device=dev, generator=g).to(torch.bfloat16)  # noqa: E731
args = argparse.Namespace(steps=2, warmup=1)
print(json.dumps(bench.run_hour_llsa(args, s, dev, rnd, torch.cuda.synchronize, 1, 0, torch.cuda.current_stream(), 6556.0)))
