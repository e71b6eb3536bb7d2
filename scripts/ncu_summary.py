#!/usr/bin/env python
"""Summarise an ncu launch list (gpu__time_duration.sum CSV) and an optional `ncu --set full`
report into markdown + traffic.json entries.  Usage:
    python scripts/ncu_summary.py <dir with launches.csv [prof_full.ncu-rep]> <out.md>
"""
import collections
import csv
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]


def short(name):
    return name.split("(")[0].replace("void ", "").replace("sattn::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] != "gpu__time_duration.sum":
                continue
            scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "nsecond": 1e-3}.get(d["Metric Unit"], 1.0)
            agg.setdefault(short(d["Kernel Name"]), []).append(float(d["Metric Value"].replace(",", "")) * scale)
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, label in METRICS:
            if m in hdr:
                d[label] = (r[hdr.index(m)], units[hdr.index(m)])
        res.append(d)
    return res


def main():
    src, out = sys.argv[1], sys.argv[2]
    lines = [f"# ncu summary: {src}", ""]
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        agg = launches(lp)
        tot = sum(sum(v) for k, v in agg.items() if "at::" not in k and "elementwise" not in k)
        lines += ["## launch list (cold-cache, serialised; compare shares)", "",
                  "| kernel | launches | mean µs | share of our kernels |", "|---|---|---|---|"]
        for k, v in agg.items():
            share = sum(v) / tot if ("at::" not in k and tot) else float("nan")
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.1f} | {share:.3f} |")
        lines.append("")
    fp = os.path.join(src, "prof_full.ncu-rep")
    traffic = {}
    if os.path.exists(fp):
        res = full(fp)
        lines += ["## ncu --set full (per launch)", ""]
        for d in res:
            lines.append(f"### {d['kernel']}")
            for m, label in METRICS:
                if label in d:
                    lines.append(f"- {label}: {d[label][0]} {d[label][1]}")
            lines.append("")
            try:
                rd = float(d["DRAM read"][0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["DRAM read"][1]]
                wr = float(d["DRAM write"][0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[d["DRAM write"][1]]
                traffic.setdefault(d["kernel"], []).append(rd + wr)
            except Exception:
                pass
    open(out, "w").write("\n".join(lines) + "\n")
    if traffic:
        tj = {k: {"dram_bytes_per_launch": sum(v) / len(v), "launches": len(v)} for k, v in traffic.items()}
        open(os.path.splitext(out)[0] + "_traffic.json", "w").write(json.dumps(tj, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
