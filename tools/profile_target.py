#!/usr/bin/env python
"""Short launch driver for ncu captures (replaces profile_batch /
profile_groups / profile_sweep): builds one workload and launches its kernel
a few times, so `ncu -k regex:... -c N` can pick a warm launch.

  python tools/profile_target.py city_batch|metro_batch [--reps 2]
  python tools/profile_target.py single:CFG[:kernel] [--reps 2]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_00966_b200 import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--subtrips", type=int, default=3)
args = ap.parse_args()
if args.workload in ("city_batch", "metro_batch"):
    tt = synth.generate(args.workload.split("_")[0])
    src, ts = synth.queries(tt, *((1000, 10) if args.workload == "city_batch" else (256, 4)))
    eng = Engine.from_timetable(tt, subtrips=args.subtrips)
    d_src = torch.tensor(src.astype(np.int32), device="cuda")
    d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
    out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
    for _ in range(args.reps):
        eng.query_many_device(d_src, d_ts, out)
else:
    parts = args.workload.split(":")
    tt = synth.generate(parts[1])
    eng = Engine.from_timetable(tt, subtrips=args.subtrips, kernel=parts[2] if len(parts) > 2 else "auto")
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    for _ in range(args.reps):
        eng.query_device(*synth.SINGLE_QUERY, out)
torch.cuda.synchronize()
print("done", args.workload, eng.stats()["kernel_name"])
