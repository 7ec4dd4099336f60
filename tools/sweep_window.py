"""Sweep the CTA schedule's time window on the city batch: time + work counters."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1912_00966_b200 import Engine

tt = synth.generate(sys.argv[1] if len(sys.argv) > 1 else "city")
src, ts = synth.queries(tt, 1000, 10)
d_src = torch.tensor(src.astype(np.int32), device="cuda")
d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
ref = None
for window in [0x7FFFFFFF, 3600, 1800, 900, 600, 300, 120, 60]:
    eng = Engine.from_timetable(tt, window=window)
    for _ in range(2):
        eng.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        eng.query_many_device(d_src, d_ts, out)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 3
    chk = out[:64].cpu().numpy()
    if ref is None:
        ref = chk
    same = bool(np.array_equal(ref, chk))
    o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    eng1 = Engine.from_timetable(tt, window=window, kernel="cta")
    for _ in range(3):
        eng1.query_device(*synth.SINGLE_QUERY, o1)
    torch.cuda.synchronize()
    a.record()
    for _ in range(20):
        eng1.query_device(*synth.SINGLE_QUERY, o1)
    b.record()
    b.synchronize()
    single = a.elapsed_time(b) / 20
    e2 = Engine.from_timetable(tt, window=window, counters=True)
    e2.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize()
    st = e2.stats()
    cnt = {k: st[k] / src.size for k in ("vertex_visits", "type_evals", "cluster_reads", "improvements", "sweeps_total")}
    print(json.dumps({"window": window, "batch_ms": ms, "qps": src.size / ms * 1e3, "single_ms": single,
                      "single_sweeps": eng1.stats()["last_sweeps"], "same_rows": same, "per_query": cnt}), flush=True)
