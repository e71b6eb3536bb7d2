#!/usr/bin/env python
"""bench.py — SA / LLSA fwd+bwd frames/s on B200 (BASELINE.json metric) + roofline + CPU-oracle baseline.

Step (one pass of the hot path over one batch): the attention core of a 12-layer
wav2vec2/HuBERT-base encoder, forward then backward —
    for l in 0..11:  sa_forward(Q_l, K_l, V_l) -> O_l, LSE_l
    for l in 11..0:  sa_backward(Q_l, K_l, V_l, O_l, LSE_l, dO_l) -> dQ_l, dK_l, dV_l
on synthetic iid N(0,1) bf16 activations, B=8 sequences x T=1750 frames (35 s at
50 Hz), H=12 heads, D=64, band (L, R) = (32, 8) (Table 3's l32_r8), distinct
per-layer tensors (2.3 GB working set >> 126 MB L2, so no L2 flush is needed).
A "frame" is one time step of one sequence carried through all heads and layers,
forward and backward: frames/step = B*T.  The same step with LLSA (C = R+1 = 9
channels per frame) is reported under "llsa".

Multi-GPU (one rank per GPU; `--gpus N` re-executes itself under torch.distributed.run when
it is not already a rank, and fails loudly if fewer than N GPUs are visible): batch x head
sharding is embarrassingly parallel - the headline has every rank run its own
B=8 batch, no data-path collective ("weak"); value = frames of all ranks / max-over-ranks
time.  Sub-objects: "llsa" = M2, the LLSA step with the B*H = 96 (b, h) units split over the
ranks (strong scaling); "large" = M3, wav2vec2-large (B=64, H=16, 24 layers) batch-sharded
(strong); "hour" = M4, one hour-long stream time-sharded through the library's NCCL halo
exchange (stored-band mode: sa_forward_p_tsharded / sa_backward_p_tsharded, strong; "hour.lse_mode" the
LSE-mode calls), with "hour.llsa" the same stream through the LLSA time-sharded calls
(llsa_forward_tsharded / llsa_backward_tsharded).

--impl reference runs the CPU oracle (oracle/, numpy fp64) on a bounded sample of
the same workload (the task's reference arm for this paper-only reference).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

B, H, T, D, L, R, NL = 8, 12, 1750, 64, 32, 8, 12
METRIC = "SA/LLSA fwd+bwd frames/sec (12L, H=12, D=64) at 1/2/4/8 B200; % HBM roofline"
UNIT = "frames/s"
# algorithmic bytes per head*layer*frame: bf16 activations, fp32 LSE
FWD_BYTES = 8 * D + 4            # read Q,K,V + write O (2 B each) + LSE (4 B)   = 516
BWD_BYTES = 16 * D + 4           # read Q,K,V,O,dO + LSE, write dQ,dK,dV        = 1028


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        j = json.load(open(p))
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------------- GPU arm

def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_2302_13451_b200 as sattn

    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        t = torch.ones(1, device=torch.device("cuda", local))
        dist.all_reduce(t)
        comm = {"backend": "nccl", "nranks": dist.get_world_size(), "all_reduce_check": int(t.item()),
                "nccl_version": ".".join(str(v) for v in torch.cuda.nccl.version())}
        print(f"[bench] rank {rank}: NCCL communicator up, nranks={comm['nranks']} (all_reduce of ones = "
              f"{comm['all_reduce_check']}), NCCL {comm['nccl_version']}", file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(1234 + rank)

    def rnd(*shape):
        return torch.randn(*shape, device=dev, generator=g, dtype=torch.float32).to(bf)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])
        torch.cuda.synchronize()

    # ---------------- SA workload: distinct per-layer tensors
    shp = (B, H, T, D)
    Qs, Ks, Vs, dOs = ([rnd(*shp) for _ in range(NL)] for _ in range(4))
    Os = [torch.empty(shp, device=dev, dtype=bf) for _ in range(NL)]
    LSEs = [torch.empty(shp[:-1], device=dev, dtype=torch.float32) for _ in range(NL)]
    dQs, dKs, dVs = ([torch.empty(shp, device=dev, dtype=bf) for _ in range(NL)] for _ in range(3))
    ws = torch.empty(sattn.lib().sa_backward_workspace(__import__("ctypes").byref(
        sattn.make_desc(B, H, T, D, L, R, sattn.BF16))), device=dev, dtype=torch.uint8)
    lib = sattn.lib()
    import ctypes
    desc = sattn.make_desc(B, H, T, D, L, R, sattn.BF16, impl=args.kernels)
    pd = ctypes.byref(desc)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    stream = torch.cuda.current_stream(dev)
    sp = ctypes.c_void_p(stream.cuda_stream)
    nws = ws.numel()

    def check(st, what):
        if st != 0:
            raise RuntimeError(f"{what}: {lib.sattn_last_error().decode()}")

    # mode "band" (default): the paper's stored a_t -- sa_forward_p keeps the band,
    # sa_backward_p reads it; mode "lse": LSE + recompute (sa_forward / sa_backward).  Same
    # outputs (dQ, dK, dV of the same SA layer), different memory / recompute trade-off.
    band = args.mode == "band"
    W = L + R + 1
    Pbs = [torch.empty(shp[:-1] + (int(lib.sa_p_ld(pd)),), device=dev, dtype=bf) for _ in range(NL)] if band else LSEs
    FB, BB = (FWD_BYTES + 2 * W, 896 + 2 * W) if band else (FWD_BYTES, BWD_BYTES)
    KF, KB = ("sa_forward_p", "sa_backward_p") if band else ("sa_forward", "sa_backward")

    def fcall(q, k, v, o, lse, pb, sp):
        if band:
            check(lib.sa_forward_p(pd, P(q), P(k), P(v), P(o), P(lse), P(pb), sp), KF)
        else:
            check(lib.sa_forward(pd, P(q), P(k), P(v), P(o), P(lse), sp), KF)

    def bcall(q, k, v, o, lse, pb, do, dq, dk, dv, sp):
        if band:
            check(lib.sa_backward_p(pd, P(q), P(k), P(v), P(o), P(pb), P(do), P(dq), P(dk), P(dv), P(ws), nws, sp), KB)
        else:
            check(lib.sa_backward(pd, P(q), P(k), P(v), P(o), P(lse), P(do), P(dq), P(dk), P(dv), P(ws), nws, sp), KB)

    def fwd_pass():
        sp = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        for l in range(NL):
            fcall(Qs[l], Ks[l], Vs[l], Os[l], LSEs[l], Pbs[l], sp)

    def bwd_pass():
        sp = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        for l in reversed(range(NL)):
            bcall(Qs[l], Ks[l], Vs[l], Os[l], LSEs[l], Pbs[l], dOs[l], dQs[l], dKs[l], dVs[l], sp)

    # The step is captured once as two CUDA graphs (forward pass, backward pass) so the timed
    # region measures GPU execution, not Python/ctypes launch overhead; an event between the two
    # replays splits the step into the per-call averages the roofline uses.
    fwd_pass(); bwd_pass()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(dev)
    gF, gB = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    n_cap0 = sattn.launch_count()
    with torch.cuda.graph(gF, stream=cap):
        fwd_pass()
    with torch.cuda.graph(gB, stream=cap):
        bwd_pass()
    launches_per_step = sattn.launch_count() - n_cap0
    ev = {"fwd": [], "bwd": []}

    def step(record=False):
        if record:
            e0 = torch.cuda.Event(enable_timing=True); e0.record(stream)
        gF.replay()
        if record:
            e1 = torch.cuda.Event(enable_timing=True); e1.record(stream)
        gB.replay()
        if record:
            e2 = torch.cuda.Event(enable_timing=True); e2.record(stream)
            ev["fwd"].append((e0, e1)); ev["bwd"].append((e1, e2))

    for _ in range(args.warmup):
        step()
    barrier()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    barrier()
    t0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    t1.record(stream)
    barrier()
    clocks = clk.stop()
    launches = launches_per_step * args.steps
    ms = t0.elapsed_time(t1)
    ms_max = ms
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms_max = float(tt.item())
    ms_per_step = ms_max / args.steps
    frames = world * B * T * args.steps
    value = frames / (ms_max / 1e3)

    fwd_ms = float(np.mean([a.elapsed_time(b) for a, b in ev["fwd"]])) / NL
    bwd_ms = float(np.mean([a.elapsed_time(b) for a, b in ev["bwd"]])) / NL
    units = B * H * T  # head-frames per launch
    hbm, tc_peak, peak_kind = load_peaks()
    kern = {KF: (fwd_ms, FB * units), KB: (bwd_ms, BB * units)}
    dom = max(kern, key=lambda k: kern[k][0])
    achieved = kern[dom][1] / (kern[dom][0] / 1e3) / 1e9
    tr = load_traffic(dom, args.kernels) or {}
    traffic = tr.get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4), "traffic": traffic, "peak_kind": peak_kind,
                "traffic_note": "dram read + max(dram write, output bytes) per launch (profiles/traffic.json)",
                "traffic_ratio": tr.get("traffic_ratio"), "dram_read_bytes": tr.get("dram_read_bytes"),
                "read_ratio_vs_algorithmic_reads": tr.get("read_ratio"),
                "algorithmic_bytes_per_launch": kern[dom][1],
                "per_call_ms": {k: round(v[0], 4) for k, v in kern.items()},
                "step_frac": {k: round(v[0] * NL / ms_per_step, 3) for k, v in kern.items()},
                "algorithmic_bytes_per_head_frame": {KF: FB, KB: BB},
                "step_hbm_frac": round((FB + BB) * units * NL / (ms_per_step / 1e3) / 1e9 / hbm, 4)}

    # ---------------- e2e through the public API with host buffers (pinned), H2D + D2H inside
    # Every step copies its inputs (all layers' Q, K, V, dO) from pinned host memory and reads
    # its results (dQ, dK, dV) back.  The copies are layer-granular on two copy streams
    # (PCIe is full duplex: the H2D of step i+1 overlaps the D2H of step i) and the compute
    # stream waits per layer on events, so each layer starts as soon as its own inputs landed.
    e2e = None
    if not args.no_e2e:
        hin = [[torch.empty(shp, dtype=bf, pin_memory=True) for _ in range(4)] for _ in range(NL)]
        hout = [[torch.empty(shp, dtype=bf, pin_memory=True) for _ in range(3)] for _ in range(NL)]
        for l in range(NL):
            for j, src in enumerate((Qs, Ks, Vs, dOs)):
                hin[l][j].copy_(src[l])
        # H2D on copy stream(s) (layers alternate when more than one), D2H on another
        n_in = 1   # 2-3 H2D copy streams measured no faster (PCIe-bound)
        s_ins = [torch.cuda.Stream(dev) for _ in range(n_in)]
        s_out = torch.cuda.Stream(dev)
        ev = lambda: torch.cuda.Event()  # noqa: E731
        # two device buffer sets, alternating by step: the H2D of step i+1 need not wait for
        # step i's compute to release its inputs
        sets = [(Qs, Ks, Vs, dOs, Os, LSEs, dQs, dKs, dVs, Pbs),
                tuple([torch.empty_like(t) for t in ts] for ts in (Qs, Ks, Vs, dOs, Os, LSEs, dQs, dKs, dVs, Pbs))]
        used = [[None] * NL for _ in range(2)]      # compute finished reading set p, layer l
        drained = [[None] * NL for _ in range(2)]   # D2H of set p, layer l finished
        par = [0]

        def e2e_step():
            p_ = par[0]; par[0] ^= 1
            q_, k_, v_, do_, o_, lse_, dq_, dk_, dv_, pb_ = sets[p_]
            landed = []
            for l in range(NL):
                s_in = s_ins[l % n_in]
                with torch.cuda.stream(s_in):
                    if used[p_][l] is not None:
                        s_in.wait_event(used[p_][l])
                    for j, dst in enumerate((q_, k_, v_, do_)):
                        dst[l].copy_(hin[l][j], non_blocking=True)
                    e = ev(); e.record(s_in); landed.append(e)
            spp = ctypes.c_void_p(stream.cuda_stream)
            for l in range(NL):
                stream.wait_event(landed[l])
                fcall(q_[l], k_[l], v_[l], o_[l], lse_[l], pb_[l], spp)
            for l in reversed(range(NL)):
                if drained[p_][l] is not None:
                    stream.wait_event(drained[p_][l])
                bcall(q_[l], k_[l], v_[l], o_[l], lse_[l], pb_[l], do_[l], dq_[l], dk_[l], dv_[l], spp)
                e = ev(); e.record(stream); used[p_][l] = e
                with torch.cuda.stream(s_out):
                    s_out.wait_event(e)
                    for j, src in enumerate((dq_, dk_, dv_)):
                        hout[l][j].copy_(src[l], non_blocking=True)
                    d = ev(); d.record(s_out); drained[p_][l] = d

        e2e_step()
        torch.cuda.synchronize()
        barrier()
        n_e2e = max(2, min(args.steps, 5))
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for s_in in s_ins:
            s_in.wait_event(a0)      # the first copies start after the start event
        for _ in range(n_e2e):
            e2e_step()
        for d in drained[0] + drained[1]:   # the end event follows every copy of the last steps
            stream.wait_event(d)
        a1.record(stream)
        barrier()
        e_ms = a0.elapsed_time(a1)
        if world > 1:
            tt = torch.tensor([e_ms], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e_ms = float(tt.item())
        el = 2 * B * H * T * D
        e2e = {"value": round(world * B * T * n_e2e / (e_ms / 1e3), 1), "unit": UNIT,
               "h2d_bytes_per_step": 4 * NL * el, "d2h_bytes_per_step": 3 * NL * el, "steps": n_e2e,
               "pipeline": f"layer-granular H2D ({n_in} copy streams) / compute / D2H streams (CUDA events), two "
                           "device buffer sets alternating by step"}
        del hin, hout, sets

    # ---------------- LLSA step (same shape, C = R+1 channels), reported alongside
    llsa = llsa_r16 = None
    if not args.no_llsa:
        del Qs, Ks, Vs, dOs, Os, dQs, dKs, dVs
        torch.cuda.empty_cache()
        try:
            llsa = run_llsa(args, sattn, dev, rnd, barrier, world, stream, hbm)
        except Exception as e:
            llsa = {"error": f"{type(e).__name__}: {e}"[:300]}
        torch.cuda.empty_cache()
        try:   # Table 3's second band, l32_r16 (C = 17 channels)
            llsa_r16 = run_llsa(args, sattn, dev, rnd, barrier, world, stream, hbm, R=16)
        except Exception as e:
            llsa_r16 = {"error": f"{type(e).__name__}: {e}"[:300]}

    alt = None   # the other SA mode, same workload
    if not args.no_alt:
        torch.cuda.empty_cache()
        try:
            alt = run_mode(args, sattn, dev, rnd, barrier, world, stream, hbm, "lse" if band else "band")
        except Exception as e:
            alt = {"error": f"{type(e).__name__}: {e}"[:300]}

    large = None
    if not args.no_large:
        torch.cuda.empty_cache()
        try:
            large = run_large(args, sattn, dev, rnd, barrier, world, stream, hbm)
        except Exception as e:
            large = {"error": f"{type(e).__name__}: {e}"[:300]}

    fa2 = None
    if not args.no_fa2 and world == 1:
        torch.cuda.empty_cache()
        try:
            fa2 = run_fa2(args, dev, rnd)
        except Exception as e:
            fa2 = {"error": f"{type(e).__name__}: {e}"[:300]}

    hour = None
    if not args.no_hour:
        torch.cuda.empty_cache()
        try:
            hour = run_hour(args, sattn, dev, rnd, barrier, world, rank, stream, hbm, band=True)
        except Exception as e:   # the headline line must not depend on this sub-measurement
            hour = {"error": f"{type(e).__name__}: {e}"[:300]}
        torch.cuda.empty_cache()
        try:
            hour_lse = run_hour(args, sattn, dev, rnd, barrier, world, rank, stream, hbm, band=False)
        except Exception as e:
            hour_lse = {"error": f"{type(e).__name__}: {e}"[:300]}
        if isinstance(hour, dict):
            hour["lse_mode"] = hour_lse
        torch.cuda.empty_cache()
        try:
            hour_llsa = run_hour_llsa(args, sattn, dev, rnd, barrier, world, rank, stream, hbm)
        except Exception as e:
            hour_llsa = {"error": f"{type(e).__name__}: {e}"[:300]}
        if isinstance(hour, dict):
            hour["llsa"] = hour_llsa

    enc = None
    if not args.no_encoder and world == 1:
        torch.cuda.empty_cache()
        try:
            enc = run_encoder(args, dev)
        except Exception as e:
            enc = {"error": f"{type(e).__name__}: {e}"[:300]}

    stream_lat = None
    if not args.no_stream:
        stream_lat = run_stream(sattn, dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.cpu_seconds)

    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    out = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic iid N(0,1) activations",
           "config": {"workload": "wav2vec2-base attention core: 12 layers x (SA fwd + SA bwd), untied per-layer "
                                  "Q/K/V/dO, bf16 in/out, fp32 accumulate",
                      "mode": "stored band a_t (P:L342): sa_forward_p + sa_backward_p" if band
                              else "LSE + recompute: sa_forward + sa_backward",
                      "B": B, "H": H, "T": T, "D": D, "L": L, "R": R, "layers": NL, "global_batch": B * world,
                      "frames_per_step": B * T * world, "parallelism": f"batch-sharded x{world} (no collective)",
                      "kernels": args.kernels, "l2": "working set 2.3 GB/rank >> 126 MB L2 (no flush)"},
           "roofline": roofline, "clocks": clocks, "gpu_launches": launches, "e2e": e2e, "llsa": llsa, "llsa_r16": llsa_r16, ("lse_mode" if band else "band_mode"): alt,
           "large": large, "hour": hour, "fa2_local_context": fa2, "comm": comm, "encoder": enc, "stream": stream_lat, "latency": latency_check(sattn, dev) if not args.no_stream else None,
           "cpu_baseline": cpu}
    print(json.dumps(out))


def _strong_batch(Btot, world):
    """Per-rank batch of a batch-sharded strong-scaling config (Btot sequences over the ranks)."""
    if Btot % world:
        raise ValueError(f"batch {Btot} does not split over {world} ranks")
    return Btot // world


def _max_ms(ms, world, dev):
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    tt = torch.tensor([ms], device=dev)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def run_llsa(args, sattn, dev, rnd, barrier, world, stream, hbm, R=R):
    """M2 (BASELINE configs[2]): the 12-layer LLSA step (C = R+1 = 9 channels) at the base shape with
    the B*H = 96 (b, h) units split over the ranks - strong scaling (B/N sequences per rank, every
    rank all H heads); value = B*T frames / max-over-ranks step time."""
    import ctypes
    import torch
    lib = sattn.lib()
    C = R + 1
    Br = _strong_batch(B, world)
    shp = (C, Br, H, T, D)
    bf = torch.bfloat16
    n_layers = NL
    Q, K, V, dO = ([rnd(*shp) for _ in range(n_layers)] for _ in range(4))
    O = [torch.empty(shp, device=dev, dtype=bf) for _ in range(n_layers)]
    LSE = [torch.empty(shp[:-1], device=dev, dtype=torch.float32) for _ in range(n_layers)]
    dQ, dK, dV = torch.empty(shp, device=dev, dtype=bf), torch.empty(shp, device=dev, dtype=bf), \
        torch.empty(shp, device=dev, dtype=bf)
    desc = sattn.make_desc(Br, H, T, D, L, R, sattn.BF16, impl=args.kernels)
    pd = ctypes.byref(desc)
    nws = lib.llsa_backward_workspace(pd)
    ws = torch.empty(nws, device=dev, dtype=torch.uint8)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def fwd():
        for l in range(n_layers):
            assert lib.llsa_forward(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0

    def bwd():
        for l in reversed(range(n_layers)):
            assert lib.llsa_backward(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), P(dO[l]), P(dQ), P(dK),
                                     P(dV), P(ws), nws, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0

    fwd(); bwd()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(dev)
    gF, gB = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gF, stream=cap):
        fwd()
    with torch.cuda.graph(gB, stream=cap):
        bwd()
    for _ in range(max(1, args.warmup)):
        gF.replay(); gB.replay()
    barrier()
    k = max(1, min(args.steps, 5))
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * k + 1)]
    evs[0].record(stream)
    for i in range(k):
        gF.replay(); evs[2 * i + 1].record(stream)
        gB.replay(); evs[2 * i + 2].record(stream)
    barrier()
    f_ms = sum(evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(k)) / k
    b_ms = sum(evs[2 * i + 1].elapsed_time(evs[2 * i + 2]) for i in range(k)) / k
    ms = _max_ms(f_ms + b_ms, world, dev)
    units = C * Br * H * T
    return {"value": round(B * T / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 3), "scaling": "strong",
            "channels": C, "steps": k, "bh_units_per_rank": Br * H,
            "hbm_frac": round((FWD_BYTES + BWD_BYTES) * units * n_layers / ((f_ms + b_ms) / 1e3) / 1e9 / hbm, 4),
            "per_call_ms": {"llsa_forward": round(f_ms / n_layers, 4), "llsa_backward": round(b_ms / n_layers, 4)},
            "hbm_frac_per_call": {"llsa_forward": round(FWD_BYTES * units / (f_ms / n_layers / 1e3) / 1e9 / hbm, 4),
                                  "llsa_backward": round(BWD_BYTES * units / (b_ms / n_layers / 1e3) / 1e9 / hbm, 4)},
            "band": [L, R],
            "workload": f"M2: 12 layers x (LLSA fwd + LLSA bwd), (L,R)=({L},{R}), untied per-layer [C,B,H,T,D] inputs, B*H = {B * H} "
                        f"(b,h) units split over {world} rank(s) ({Br * H} per rank)"}


def run_large(args, sattn, dev, rnd, barrier, world, stream, hbm):
    """M3 (BASELINE configs[3]): wav2vec2-large attention core, B=64, H=16, T=1750, D=64, 24 layers
    (reading G22), SA fwd + bwd in the headline mode, batch-sharded over the ranks (strong scaling:
    64/N sequences per rank); value = 64*T frames / max-over-ranks step time."""
    import ctypes
    import torch
    lib = sattn.lib()
    Bl, Hl, nl = 64, 16, 24
    Br = _strong_batch(Bl, world)
    shp = (Br, Hl, T, D)
    bf = torch.bfloat16
    band = args.mode == "band"
    desc = sattn.make_desc(Br, Hl, T, D, L, R, sattn.BF16, impl=args.kernels)
    pd = ctypes.byref(desc)
    ld = int(lib.sa_p_ld(pd))
    Q, K, V, dO = ([rnd(*shp) for _ in range(nl)] for _ in range(4))
    O = [torch.empty(shp, device=dev, dtype=bf) for _ in range(nl)]
    LSE = [torch.empty(shp[:-1], device=dev, dtype=torch.float32) for _ in range(nl)]
    Pb = [torch.empty(shp[:-1] + (ld,), device=dev, dtype=bf) for _ in range(nl)] if band else LSE
    dQ, dK, dV = (torch.empty(shp, device=dev, dtype=bf) for _ in range(3))
    nws = lib.sa_backward_p_workspace(pd) if band else lib.sa_backward_workspace(pd)
    ws = torch.empty(nws, device=dev, dtype=torch.uint8)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    sp = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731

    def fwd():
        for l in range(nl):
            st = (lib.sa_forward_p(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), P(Pb[l]), sp()) if band else
                  lib.sa_forward(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), sp()))
            assert st == 0, lib.sattn_last_error()

    def bwd():
        for l in reversed(range(nl)):
            st = (lib.sa_backward_p(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(Pb[l]), P(dO[l]), P(dQ), P(dK), P(dV),
                                    P(ws), nws, sp()) if band else
                  lib.sa_backward(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), P(dO[l]), P(dQ), P(dK), P(dV),
                                  P(ws), nws, sp()))
            assert st == 0, lib.sattn_last_error()

    fwd(); bwd()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cap):
        fwd(); bwd()
    for _ in range(max(1, min(args.warmup, 3))):
        g.replay()
    barrier()
    k = max(1, min(args.steps, 3))
    a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(k):
        g.replay()
    a1.record(stream)
    barrier()
    ms_loc = a0.elapsed_time(a1) / k
    ms = _max_ms(ms_loc, world, dev)
    W = L + R + 1
    fb, bb = (FWD_BYTES + 2 * W, 896 + 2 * W) if band else (FWD_BYTES, BWD_BYTES)
    units = Br * Hl * T
    return {"value": round(Bl * T / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 3), "scaling": "strong",
            "steps": k, "per_layer_ms": round(ms / nl, 4),
            "hbm_frac": round((fb + bb) * units * nl / (ms_loc / 1e3) / 1e9 / hbm, 4),
            "workload": f"M3: wav2vec2-large attention core B={Bl}, H={Hl}, T={T}, {nl} layers x (SA fwd + bwd, "
                        f"{'stored band' if band else 'LSE'} mode), batch-sharded over {world} rank(s) ({Br} "
                        f"sequences per rank)"}


def run_fa2(args, dev, rnd):
    """Context only: FlashAttention-2's local attention
    (flash_attn_func(..., window_size=(L, R)), a library kernel) fwd + bwd on the headline
    workload (12 distinct layers, [B, T, H, D] bf16), next to the repo's per-layer times."""
    import torch
    from flash_attn import flash_attn_func
    shp = (B, T, H, D)
    qs = [[rnd(*shp).requires_grad_(True) for _ in range(3)] for _ in range(NL)]
    dos = [rnd(*shp) for _ in range(NL)]

    def step():
        outs = [flash_attn_func(q, k, v, window_size=(L, R)) for q, k, v in qs]
        for o, do in zip(reversed(outs), reversed(dos)):
            o.backward(do)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    k = 3
    a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(k):
        step()
    a1.record()
    torch.cuda.synchronize()
    ms = a0.elapsed_time(a1) / k
    return {"value": round(B * T / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 3),
            "per_layer_fwd_bwd_ms": round(ms / NL, 4),
            "workload": f"flash_attn {__import__('flash_attn').__version__} flash_attn_func window_size=({L},{R}) "
                        f"fwd+bwd, 12 layers, B={B}, T={T}, H={H}, D={D}, bf16, eager autograd (context only)"}


def run_mode(args, sattn, dev, rnd, barrier, world, stream, hbm, mode):
    """The same 12-layer SA step in the other mode: "band" = the paper's stored a_t
    ([B,H,T,ld] bf16 kept by the forward and read by the backward; NEXT-4), "lse" =
    LSE + recompute.  Algorithmic bytes per head-frame: band forward 516 + 2W (the band write),
    backward Q,K,V,dO + band + dQ,dK,dV = 896 + 2W (no O, no LSE: delta = rowsum(P o dP));
    lse 516 / 1028."""
    import ctypes
    import torch
    lib = sattn.lib()
    shp = (B, H, T, D)
    bf = torch.bfloat16
    desc = sattn.make_desc(B, H, T, D, L, R, sattn.BF16, impl=args.kernels)
    pd = ctypes.byref(desc)
    ld = int(lib.sa_p_ld(pd))
    Q, K, V, dO = ([rnd(*shp) for _ in range(NL)] for _ in range(4))
    O = [torch.empty(shp, device=dev, dtype=bf) for _ in range(NL)]
    LSE = [torch.empty(shp[:-1], device=dev, dtype=torch.float32) for _ in range(NL)]
    Pb = [torch.empty(shp[:-1] + (ld,), device=dev, dtype=bf) for _ in range(NL)]
    dQ, dK, dV = ([torch.empty(shp, device=dev, dtype=bf) for _ in range(NL)] for _ in range(3))
    nws = lib.sa_backward_p_workspace(pd)
    ws = torch.empty(nws, device=dev, dtype=torch.uint8)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731
    sp = lambda: ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)  # noqa: E731

    bm = mode == "band"
    if not bm:
        nws = lib.sa_backward_workspace(pd)
        ws = torch.empty(nws, device=dev, dtype=torch.uint8)

    def fwd():
        for l in range(NL):
            st = (lib.sa_forward_p(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), P(Pb[l]), sp()) if bm else
                  lib.sa_forward(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), sp()))
            assert st == 0, lib.sattn_last_error()

    def bwd():
        for l in reversed(range(NL)):
            st = (lib.sa_backward_p(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(Pb[l]), P(dO[l]), P(dQ[l]), P(dK[l]),
                                    P(dV[l]), P(ws), nws, sp()) if bm else
                  lib.sa_backward(pd, P(Q[l]), P(K[l]), P(V[l]), P(O[l]), P(LSE[l]), P(dO[l]), P(dQ[l]), P(dK[l]),
                                  P(dV[l]), P(ws), nws, sp()))
            assert st == 0, lib.sattn_last_error()

    fwd(); bwd()
    torch.cuda.synchronize()
    cap = torch.cuda.Stream(dev)
    gF, gB = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(gF, stream=cap):
        fwd()
    with torch.cuda.graph(gB, stream=cap):
        bwd()
    for _ in range(max(3, args.warmup)):
        gF.replay(); gB.replay()
    barrier()
    k = max(2, min(args.steps, 10))
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * k + 1)]
    evs[0].record(stream)
    for i in range(k):
        gF.replay(); evs[2 * i + 1].record(stream)
        gB.replay(); evs[2 * i + 2].record(stream)
    barrier()
    f_ms = sum(evs[2 * i].elapsed_time(evs[2 * i + 1]) for i in range(k)) / k
    b_ms = sum(evs[2 * i + 1].elapsed_time(evs[2 * i + 2]) for i in range(k)) / k
    ms = f_ms + b_ms
    W = L + R + 1
    fb, bb = (FWD_BYTES + 2 * W, 896 + 2 * W) if bm else (FWD_BYTES, BWD_BYTES)
    kf, kb = ("sa_forward_p", "sa_backward_p") if bm else ("sa_forward", "sa_backward")
    units = B * H * T
    return {"mode": mode, "value": round(world * B * T / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 4),
            "steps": k, "per_call_ms": {kf: round(f_ms / NL, 4), kb: round(b_ms / NL, 4)},
            "algorithmic_bytes_per_head_frame": {kf: fb, kb: bb},
            "hbm_frac": {kf: round(fb * units / (f_ms / NL / 1e3) / 1e9 / hbm, 4),
                         kb: round(bb * units / (b_ms / NL / 1e3) / 1e9 / hbm, 4),
                         "step": round((fb + bb) * units * NL / (ms / 1e3) / 1e9 / hbm, 4)},
            "band_bytes_per_layer": units * ld * 2, "lse_bytes_per_layer": units * 4,
            "workload": f"12 layers x ({kf} + {kb}), untied per-layer inputs, bf16"}


def run_hour(args, sattn, dev, rnd, barrier, world, rank, stream, hbm, band=True):
    """M4 (BASELINE configs[4]): one hour-long stream (B=1, H=12, T=180,000 frames = 1 h at 50 Hz),
    12 layers x (SA fwd + SA bwd), bf16, time-sharded over the ranks through the library on margined
    shards (rank r owns frames [t0, t1), 128-aligned; each call exchanges the halo rows with its
    neighbours over NCCL on a library stream while the interior tiles run).  band=True: the stored-band
    mode (sa_forward_p_tsharded / sa_backward_p_tsharded, as the headline); False: LSE + recompute
    (sa_forward_tsharded / sa_backward_tsharded).  At N = 1 the same calls run with no neighbours.
    Strong scaling: value = T frames / max-over-ranks step time."""
    import ctypes
    import torch
    from paper_2302_13451_b200 import dist as sd
    from paper_2302_13451_b200 import tshard
    Th, Bh, n_layers = 180_000, 1, NL
    t0, t1 = tshard.shard_bounds(Th, world, rank, 128)
    n = t1 - t0
    d = sd.Dist()
    L_ = sd._lib()
    td = sd.tdesc(Bh, H, n, D, L, R, t0, Th)
    tdp = ctypes.byref(td)
    nws = int(L_.sa_tsharded_workspace(tdp, d._h))
    if nws == 0:
        raise RuntimeError(L_.sattn_last_error().decode())
    ws = torch.empty(nws, device=dev, dtype=torch.uint8)
    ld = (L + R + 1 + 7) // 8 * 8
    Qm, Km, Vm, dOm = ([sd.margined(Bh, H, n, D, device=dev) for _ in range(n_layers)] for _ in range(4))
    for bufs in (Qm, Km, Vm, dOm):
        for m in bufs:
            sd.local(m, n).copy_(rnd(Bh, H, n, D))
    Om = [sd.margined(Bh, H, n, D, device=dev) for _ in range(n_layers)]
    LSEm = [sd.margined(Bh, H, n, None, dtype=torch.float32, device=dev) for _ in range(n_layers)]
    Pm = [sd.margined(Bh, H, n, ld, device=dev) for _ in range(n_layers)] if band else None
    dQm, dKm, dVm = (sd.margined(Bh, H, n, D, device=dev) for _ in range(3))
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def step():
        sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for l in range(n_layers):
            st = (L_.sa_forward_p_tsharded(tdp, d._h, P(Qm[l]), P(Km[l]), P(Vm[l]), P(Om[l]), P(LSEm[l]), P(Pm[l]),
                                           P(ws), nws, sp) if band else
                  L_.sa_forward_tsharded(tdp, d._h, P(Qm[l]), P(Km[l]), P(Vm[l]), P(Om[l]), P(LSEm[l]), P(ws), nws, sp))
            assert st == 0, L_.sattn_last_error()
        for l in reversed(range(n_layers)):
            st = (L_.sa_backward_p_tsharded(tdp, d._h, P(Qm[l]), P(Km[l]), P(Vm[l]), P(Pm[l]), P(dOm[l]), P(dQm),
                                            P(dKm), P(dVm), P(ws), nws, sp) if band else
                  L_.sa_backward_tsharded(tdp, d._h, P(Qm[l]), P(Km[l]), P(Vm[l]), P(LSEm[l]), P(dOm[l]), P(dQm),
                                          P(dKm), P(dVm), P(ws), nws, sp))
            assert st == 0, L_.sattn_last_error()

    step()
    torch.cuda.synchronize()
    graph = None
    try:   # NCCL point-to-point and the library's fork/join streams are capturable
        cap = torch.cuda.Stream(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cap):
            step()
        graph = g
    except Exception:
        torch.cuda.synchronize()
        graph = None
    run = graph.replay if graph is not None else step
    for _ in range(max(1, min(args.warmup, 3))):
        run()
    barrier()
    k = max(1, min(args.steps, 5))
    a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(k):
        run()
    a1.record(stream)
    barrier()
    ms_loc = a0.elapsed_time(a1) / k
    ms = _max_ms(ms_loc, world, dev)
    d.close()
    graphed = graph is not None
    del graph
    units = Bh * H * n
    W = L + R + 1
    fb, bb = (FWD_BYTES + 2 * W, 896 + 2 * W) if band else (FWD_BYTES, BWD_BYTES)
    calls = ("sa_forward_p_tsharded / sa_backward_p_tsharded (stored band)" if band else
             "sa_forward_tsharded / sa_backward_tsharded (LSE + recompute)")
    return {"value": round(Bh * Th / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 3), "steps": k,
            "scaling": "strong", "mode": "band" if band else "lse",
            "hbm_frac": round((fb + bb) * units * n_layers / (ms_loc / 1e3) / 1e9 / hbm, 4),
            "workload": f"M4: hour-long stream B=1, H={H}, T={Th}, (L,R)=({L},{R}), {n_layers} layers x (SA fwd + bwd) "
                        f"through {calls}, time-sharded x{world} "
                        f"({'NCCL halo exchange overlapped with interior tiles' if world > 1 else 'no neighbours'}), "
                        f"{'CUDA graph' if graphed else 'eager'}",
            "frames_per_rank": n, "halo_exchange": "nccl" if world > 1 else None}


def run_hour_llsa(args, sattn, dev, rnd, barrier, world, rank, stream, hbm):
    """M4, LLSA: the hour-long stream (B=1, H=12, T=180,000) through 12 layers x (LLSA fwd + bwd),
    C = R+1 = 9 channels, bf16, time-sharded over the ranks through llsa_forward_tsharded /
    llsa_backward_tsharded (contiguous slabs with L+2R-frame margins exchanged over NCCL before
    each call; at N = 1 no neighbours).  One buffer set serves every layer (the 20 GB per-layer
    working set is far beyond L2 either way).  Strong scaling: value = T / max-over-ranks time."""
    import ctypes
    import torch
    from paper_2302_13451_b200 import dist as sd
    from paper_2302_13451_b200 import tshard
    Th, Bh, n_layers, C = 180_000, 1, NL, R + 1
    t0, t1 = tshard.shard_bounds(Th, world, rank, 1)
    n = t1 - t0
    hl, hr = sd.llsa_slab_rows(n, L, R, t0, Th)
    Ts = hl + n + hr
    d = sd.Dist()
    L_ = sd._lib()
    td = sd.tdesc(Bh, H, n, D, L, R, t0, Th)
    tdp = ctypes.byref(td)
    nws = int(L_.llsa_tsharded_workspace(tdp, d._h))
    if nws == 0:
        raise RuntimeError(L_.sattn_last_error().decode())
    ws = torch.empty(nws, device=dev, dtype=torch.uint8)
    shp = (C, Bh, H, Ts, D)
    Q, K, V, dO = (torch.zeros(shp, device=dev, dtype=torch.bfloat16) for _ in range(4))
    for x in (Q, K, V, dO):
        x[:, :, :, hl:hl + n].copy_(rnd(C, Bh, H, n, D))
    O, dQ, dK, dV = (torch.zeros(shp, device=dev, dtype=torch.bfloat16) for _ in range(4))
    LSE = torch.zeros(shp[:-1], device=dev, dtype=torch.float32)
    P = lambda t: ctypes.c_void_p(t.data_ptr())  # noqa: E731

    def step():
        sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        for _ in range(n_layers):
            st = L_.llsa_forward_tsharded(tdp, d._h, P(Q), P(K), P(V), P(O), P(LSE), P(ws), nws, sp)
            assert st == 0, L_.sattn_last_error()
        for _ in range(n_layers):
            st = L_.llsa_backward_tsharded(tdp, d._h, P(Q), P(K), P(V), P(O), P(LSE), P(dO), P(dQ), P(dK), P(dV),
                                           P(ws), nws, sp)
            assert st == 0, L_.sattn_last_error()

    step()
    torch.cuda.synchronize()
    barrier()
    k = max(1, min(args.steps, 3))
    a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(k):
        step()
    a1.record(stream)
    barrier()
    ms_loc = a0.elapsed_time(a1) / k
    ms = _max_ms(ms_loc, world, dev)
    d.close()
    units = Bh * H * n * C
    del Q, K, V, dO, O, dQ, dK, dV, LSE, ws
    torch.cuda.empty_cache()
    return {"value": round(Bh * Th / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 3), "steps": k,
            "scaling": "strong", "channels": C,
            "hbm_frac": round((FWD_BYTES + BWD_BYTES) * units * n_layers / (ms_loc / 1e3) / 1e9 / hbm, 4),
            "workload": f"M4 LLSA: hour-long stream B=1, H={H}, T={Th}, (L,R)=({L},{R}), C={C}, {n_layers} layers x "
                        f"(LLSA fwd + bwd) through llsa_forward_tsharded / llsa_backward_tsharded, time-sharded "
                        f"x{world} ({'NCCL halo exchange of L+2R-frame margins' if world > 1 else 'no neighbours'}), eager",
            "frames_per_rank": n, "halo_exchange": "nccl" if world > 1 else None}


def run_encoder(args, dev):
    """NEXT-3: a 12-layer wav2vec2/HuBERT-base encoder (d=768, H=12, FFN 3072, post-LN, bf16)
    training step (forward + backward, no optimizer) at B=8, T=1750, with the repo's SA
    attention vs the same layers with masked acausal attention (torch SDPA + band mask).
    Everything but the attention is torch / cuBLAS."""
    import torch
    from paper_2302_13451_b200 import encoder
    out = {}
    g = torch.Generator(device=dev).manual_seed(7)
    x = torch.randn(B, T, 768, device=dev, generator=g).to(torch.bfloat16)
    dy = torch.randn(B, T, 768, device=dev, generator=g).to(torch.bfloat16)
    for name, cls in (("sa", encoder.SAEncoderLayer), ("maa", encoder.MaskedEncoderLayer)):
        torch.manual_seed(0)
        layers = torch.nn.Sequential(*[cls(L=L, R=R) for _ in range(NL)]).to(dev).to(torch.bfloat16)

        def step():
            xi = x.detach().requires_grad_(True)
            layers(xi).backward(dy)

        for _ in range(2):
            step()
        torch.cuda.synchronize()
        torch.cuda.reset_peak_memory_stats()
        k = 3
        a0 = torch.cuda.Event(enable_timing=True); a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(k):
            step()
        a1.record()
        torch.cuda.synchronize()
        ms = a0.elapsed_time(a1) / k
        out[name] = {"ms_per_step": round(ms, 3), "frames_per_s": round(B * T / (ms / 1e3), 1),
                     "peak_mem_gb": round(torch.cuda.max_memory_allocated() / 2**30, 2)}
        del layers
        torch.cuda.empty_cache()
    out["speedup_vs_maa"] = round(out["maa"]["ms_per_step"] / out["sa"]["ms_per_step"], 3)
    out["workload"] = (f"{NL} x wav2vec2-base encoder layer (d=768, H=12, FFN 3072, post-LN), B={B}, T={T}, "
                       f"(L,R)=({L},{R}), bf16, fwd+bwd (no optimizer); projections/FFN/LN are torch (cuBLAS)")
    return out


def run_stream(sattn, dev, n_steps=10000, warm=1000):
    """Incremental LLSA (infer_llsa) and SA (infer_sa) inference: per-frame step latency, 12 layers,
    H=12, D=64, (L,R)=(32,8), bf16, one kernel launch per frame for all layers.
    device = CUDA-event time around one eager step (includes the Python binding's launch overhead, the
    GPU waits for the launch); host = ABI call + synchronize round trip; kernel_us_graph = the step
    kernel alone (64 consecutive steps in one CUDA graph, replayed)."""
    import torch
    res = {}
    for kind, nb, dt in (("llsa", 1, torch.bfloat16), ("llsa", 64, torch.bfloat16), ("sa", 1, torch.bfloat16),
                         ("sa", 64, torch.bfloat16), ("llsa", 1, torch.float32), ("sa", 1, torch.float32)):
        cls = sattn.LLSAStream if kind == "llsa" else sattn.SAStream
        st = cls(nb, H, D, L, R, NL, dtype=dt, device=dev)
        xs = torch.randn(warm + n_steps, nb, H, D, device=dev).to(dt)
        y = torch.empty(nb, H, D, device=dev, dtype=dt)
        for i in range(warm):
            st.step_into(xs[i], y)
        torch.cuda.synchronize()
        dev_us, host_us = [], []
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_steps)]
        for i in range(n_steps):
            t0 = time.perf_counter()
            ev[i][0].record()
            st.step_into(xs[warm + i], y)
            ev[i][1].record()
            torch.cuda.synchronize()
            host_us.append((time.perf_counter() - t0) * 1e6)
        dev_us = [a.elapsed_time(b) * 1e3 for a, b in ev]
        # the kernel alone: 64 consecutive steps captured in one CUDA graph (no host call between
        # steps), replayed; per-step device time = replay time / 64
        kern_us = None
        try:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(device=dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    for i in range(64):
                        st.step_into(xs[i], y)
            torch.cuda.current_stream(dev).wait_stream(side)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            kern_us = round(e0.elapsed_time(e1) * 1e3 / (20 * 64), 2)
            del g
        except Exception as ex:  # report, do not hide: the host-timed numbers above stand
            kern_us = f"unavailable: {type(ex).__name__}: {ex}"[:200]
        key = (f"B{nb}" if kind == "llsa" else f"sa_B{nb}") + ("" if dt == torch.bfloat16 else "_f32")
        res[key] = {"device_p50_us": round(float(np.percentile(dev_us, 50)), 2),
                         "device_p99_us": round(float(np.percentile(dev_us, 99)), 2),
                         "host_p50_us": round(float(np.percentile(host_us, 50)), 2),
                         "host_p99_us": round(float(np.percentile(host_us, 99)), 2),
                         "kernel_us_graph": kern_us,
                         "streams": nb, "steps": n_steps, "dtype": "bf16" if dt == torch.bfloat16 else "f32"}
        del st
    res["config"] = (f"{NL} layers, H={H}, D={D}, (L,R)=({L},{R}), bf16 (mma.sync step; *_f32: fp32 CUDA-core step), "
                     f"one launch per frame, {n_steps} steps after {warm} warm-up; B1/B64 = infer_llsa (latency R = {R} "
                     f"frames), sa_B1/sa_B64 = infer_sa (latency {NL}R = {NL * R} frames)")
    return res


def latency_check(sattn, dev):
    """Numeric witness probe: a 12-layer LLSA stack's designated output
    depends on frames <= t + R only; the masked-acausal (SA) stack's on frames <= t + 12 R."""
    import torch
    import synth
    T_, D_, tau = 400, 64, 350
    x = synth.witness(0, 1, 1, T_, D_, kappa=40.0)
    x2 = x.copy()
    x2[0, 0, tau] += 0.5
    out = {}
    for mode, m in (("sa", sattn.MODE_SA), ("llsa", sattn.MODE_LLSA)):
        ys = []
        for xx in (x, x2):
            y, _ = sattn.stack_forward(torch.tensor(xx, dtype=torch.float32, device=dev), L, R, NL, m)
            ys.append((y[R] if mode == "llsa" else y).double().cpu().numpy())
        d = np.abs(ys[1] - ys[0])[0, 0].max(-1)
        out[f"{mode}_frames"] = int(tau - np.nonzero(d > 0)[0][0])
    out["sa_seconds"] = round(out["sa_frames"] * 0.02, 4)
    out["llsa_seconds"] = round(out["llsa_frames"] * 0.02, 4)
    out["paper"] = "Table 3 l32_r8: infer_sa 1.92 s, infer_llsa 0.16 s (P:L391, P:L396)"
    return out


def load_traffic(kernel, impl):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        j = json.load(open(p))
        return j.get(f"{kernel}:{impl}") or j.get(kernel)
    except Exception:
        return None


# ----------------------------------------------------------------------------------- CPU oracle

def _oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(budget_s: float = 15.0, steps: int | None = None):
    """Time the oracle (as it stands) on host cores on a bounded sample: SA forward + backward of
    single (batch, head) planes of one layer at the bench shape; frames/s scaled to the metric
    (one frame = H heads x 12 layers of fwd+bwd)."""
    import oracle
    import synth
    q, k, v = synth.qkv(0, (T, D), "bf16")
    do = synth.grad_out(0, (T, D), "bf16")
    times = []
    t_start = time.perf_counter()
    n = 0
    while True:
        a = time.perf_counter()
        oracle.sa.sa_forward(q, k, v, L, R)
        oracle.sa.sa_backward(q, k, v, do, L, R)
        times.append(time.perf_counter() - a)
        n += 1
        if steps is not None and n >= steps:
            break
        if steps is None and time.perf_counter() - t_start > budget_s:
            break
    per_head_layer = float(np.mean(times))
    value = T / (per_head_layer * H * NL)
    return {"value": round(value, 3), "unit": UNIT, "cores": _oracle_threads(), "kind": "oracle",
            "sample": f"{n} x one (batch, head) plane, one layer, SA fwd+bwd at T={T}, D={D}, (L,R)=({L},{R}), "
                      f"numpy fp64 dense masked T x T; {per_head_layer:.3f} s each; scaled to H={H} x {NL} layers",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    for _ in range(args.warmup):
        cpu_baseline(steps=1)
    t0 = time.perf_counter()
    cb = cpu_baseline(steps=args.steps)
    wall = time.perf_counter() - t0
    out = {"impl": "reference", "metric": METRIC, "value": cb["value"], "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 1),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic iid N(0,1) activations (bf16-rounded)",
           "config": {"workload": "wav2vec2-base attention core: 12 layers x (SA fwd + SA bwd) — CPU oracle on a "
                                  "bounded sample (one (batch, head) plane of one layer per step)",
                      "B": B, "H": H, "T": T, "D": D, "L": L, "R": R, "layers": NL},
           "cpu_baseline": cb,
           "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernels", default="auto", choices=["auto", "ffma", "tc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-llsa", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stream", action="store_true")
    ap.add_argument("--no-hour", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other SA mode's sub-measurement")
    ap.add_argument("--mode", default="band", choices=["band", "lse"],
                    help="headline SA mode: stored band a_t (paper P:L342) or LSE + recompute")
    ap.add_argument("--no-encoder", action="store_true")
    ap.add_argument("--no-large", action="store_true")
    ap.add_argument("--no-fa2", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if "WORLD_SIZE" in os.environ:
        if int(os.environ["WORLD_SIZE"]) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
    elif args.gpus > 1:
        # not a rank yet: launch one rank per GPU (the driver's own torchrun command is equivalent)
        if args.impl == "ours":
            import torch
            n = torch.cuda.device_count()
            if n < args.gpus:
                sys.exit(f"bench.py: --gpus {args.gpus} requested but only {n} CUDA device(s) are visible")
        import socket
        so = socket.socket(); so.bind(("127.0.0.1", 0)); port = so.getsockname()[1]; so.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
