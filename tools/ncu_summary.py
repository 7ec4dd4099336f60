"""Summarise ncu outputs into profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py report <file.ncu-rep> [--out profiles/x.md]
  python tools/ncu_summary.py launches <launches.csv> [--out profiles/x.md]
"""
import argparse
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "SM Frequency"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "L1/TEX Cache Throughput"),
    ("GPU Speed Of Light Throughput", "L2 Cache Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("Compute Workload Analysis", "Issued Ipc Active"),
    ("Memory Workload Analysis", "Memory Throughput"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Scheduler Statistics", "No Eligible"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Warp State Statistics", "Avg. Active Threads Per Warp"),
    ("Instruction Statistics", "Executed Instructions"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Achieved Occupancy"),
    ("Source Counters", "Branch Efficiency"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "lts__t_sectors_op_atomic.sum",
       "lts__t_sectors_op_red.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
       "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
       "gpu__time_duration.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def _csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def report(path):
    rows = _csv([path, "--page", "details"])
    hdr = rows[0]
    d = [dict(zip(hdr, r)) for r in rows[1:]]
    kernel = d[0].get("Kernel Name", "?") if d else "?"
    lines = [f"### {kernel[:120]}", "", "| section | metric | value |", "|---|---|---|"]
    for sec, met in KEYS:
        for r in d:
            if r.get("Section Name") == sec and r.get("Metric Name") == met:
                lines.append(f"| {sec} | {met} | {r.get('Metric Value')} {r.get('Metric Unit')} |")
                break
    raw = _csv([path, "--page", "raw"])
    if len(raw) >= 3:
        h, units, vals = raw[0], raw[1], raw[2]
        lines += ["", "| raw metric | value |", "|---|---|"]
        for k in RAW:
            if k in h:
                i = h.index(k)
                lines.append(f"| {k} | {vals[i]} {units[i]} |")
    return "\n".join(lines) + "\n"


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki][:90]][0] += 1
            agg[r[ki][:90]][1] += float(r[vi].replace(",", ""))
    tot = sum(v for _, v in agg.values())
    lines = ["| launches | total ms | share | kernel |", "|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {c} | {v / 1e6:.3f} | {100 * v / tot:.1f}% | `{k}` |")
    return "\n".join(lines) + "\n"


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["report", "launches"])
    ap.add_argument("path")
    ap.add_argument("--out")
    a = ap.parse_args()
    text = report(a.path) if a.kind == "report" else launches(a.path)
    if a.out:
        with open(a.out, "a") as f:
            f.write(text + "\n")
    sys.stdout.write(text)
