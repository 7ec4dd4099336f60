"""Warp-local continuation on/off x window: city batch throughput, work counters, single-query latency."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1912_00966_b200 import Engine


def timed(fn, reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


tt = synth.generate("city")
src, ts = synth.queries(tt, 1000, 10)
d_src = torch.tensor(src.astype(np.int32), device="cuda")
d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
ref = None
for cont in (True, False):
    for window in (1800, 3600, 900, 0x7FFFFFFF):
        kw = dict(subtrips=2, window=window, continuation=cont)
        eng = Engine.from_timetable(tt, **kw)
        for _ in range(2):
            eng.query_many_device(d_src, d_ts, out)
        ms = timed(lambda: eng.query_many_device(d_src, d_ts, out), 3)
        chk = out[:256].cpu().numpy()
        ref = chk if ref is None else ref
        sms = timed(lambda: eng.query_device(*synth.SINGLE_QUERY, o1), 20)
        e2 = Engine.from_timetable(tt, counters=True, **kw)
        e2.query_many_device(d_src, d_ts, out)
        torch.cuda.synchronize()
        st = e2.stats()
        per = {k: st[k] / src.size for k in ("vertex_visits", "type_evals", "cluster_reads", "improvements", "sweeps_total")}
        print(json.dumps({"cont": cont, "window": window, "batch_ms": ms, "qps": src.size / ms * 1e3, "single_ms": sms,
                          "single_sweeps": eng.stats()["last_sweeps"], "same_rows": bool(np.array_equal(ref, chk)),
                          "per_query": per}), flush=True)
        eng.close()
        e2.close()
