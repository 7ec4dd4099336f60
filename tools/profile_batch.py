"""Short driver for ncu captures: build the city index and launch the batched
kernel (BASELINE configs[2]) a few times.  Usage:
  python tools/profile_batch.py [--nq 10000] [--reps 2] [--kernel-single cta|frontier]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1912_00966_b200 import Engine

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="city")
ap.add_argument("--nq", type=int, default=10000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--single", default="")
ap.add_argument("--subwarp", type=int, default=8)
ap.add_argument("--window", type=int, default=0)
ap.add_argument("--subtrips", type=int, default=3)
a = ap.parse_args()
tt = synth.generate(a.config)
if a.single:
    eng = Engine.from_timetable(tt, kernel=a.single, subwarp=a.subwarp, window=a.window, subtrips=a.subtrips)
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    for _ in range(a.reps):
        eng.query_device(*synth.SINGLE_QUERY, out)
    torch.cuda.synchronize()
    print("sweeps", eng.stats()["last_sweeps"])
else:
    eng = Engine.from_timetable(tt, subwarp=a.subwarp, window=a.window, subtrips=a.subtrips)
    src, ts = synth.queries(tt, a.nq // 10, 10)
    d_src = torch.tensor(src.astype(np.int32), device="cuda")
    d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
    out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
    for _ in range(a.reps):
        eng.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize()
print("done")
