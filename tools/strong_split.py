#!/usr/bin/env python
"""One rank's share of the strong-scaled city batch (BASELINE configs[2]:
10k queries split over N GPUs): device time of query_many_device on the
first 10k/N queries of the bench's batch, N = 1, 2, 4, 8, on this one GPU.
Shows the tail of the last CTA wave that the N-GPU bench line will see
(the driver computes scaling efficiency from the per-N values).

  python tools/strong_split.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_00966_b200 import Engine  # noqa: E402

tt = synth.generate("city")
src, ts = synth.queries(tt, 1000, 10)
eng = Engine.from_timetable(tt, subtrips=3)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
base = None
for N in (1, 2, 4, 8):
    nq = src.size // N
    d_src = torch.tensor(src[:nq].astype(np.int32), device="cuda")
    d_ts = torch.tensor(ts[:nq].astype(np.int32), device="cuda")
    out = torch.empty((nq, tt.num_vertices), dtype=torch.int32, device="cuda")
    eng.query_many_device(d_src, d_ts, out)
    ms = []
    for i in range(7):
        flush.fill_(i)
        a.record()
        eng.query_many_device(d_src, d_ts, out)
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
    m = float(np.median(ms))
    if base is None:
        base = m
    print(json.dumps({"N": N, "queries_per_gpu": nq, "ms": m, "qps_per_gpu": nq / m * 1e3,
                      "efficiency_vs_N1": base / (m * N), "cta_grid": eng.stats()["cta_grid"]}), flush=True)
