#!/usr/bin/env python
"""Query-order experiment behind the batched kernel's departure-time
hand-out (profiles/r02_order_by_time.jsonl): device time of the N = 8 share
(1,250 queries) of the city batch in several orders, and the cost of 740
queries drawn from each 3-hour departure band.  EAT_SORT_BATCHES=0 to time
the orders as given (the library otherwise re-orders by departure time).

  EAT_SORT_BATCHES=0 python tools/order_experiment.py
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1912_00966_b200 import Engine
tt = synth.generate("city")
src, ts = synth.queries(tt, 1000, 10)
eng = Engine.from_timetable(tt, subtrips=3)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
# per-query cost: time each query alone? use single-query CTA via batch of 1 -- too slow; use sweeps proxy via batches of 740
def timeit(s_, t_):
    d_src = torch.tensor(s_.astype(np.int32), device="cuda"); d_ts = torch.tensor(t_.astype(np.int32), device="cuda")
    out = torch.empty((s_.size, tt.num_vertices), dtype=torch.int32, device="cuda")
    eng.query_many_device(d_src, d_ts, out)
    ms = []
    for i in range(7):
        flush.fill_(i); a.record(); eng.query_many_device(d_src, d_ts, out); b.record(); b.synchronize(); ms.append(a.elapsed_time(b))
    return float(np.median(ms))
nq = 1250
s8, t8 = src[:nq], ts[:nq]
h = (t8 // 3600).astype(int)
orders = {
  "as_is": np.arange(nq),
  "ts_asc": np.argsort(t8, kind="stable"),
  "ts_desc": np.argsort(-t8.astype(np.int64), kind="stable"),
  # hours 0-5 (wait for morning, then explore the whole day) first, then daytime by ascending time, late evening last
  "night_first": np.argsort(np.where(h < 5, -1, np.where(h >= 21, 100, h)) * 100000 + t8 % 100000, kind="stable"),
  "late_last": np.argsort(np.where(h >= 21, 1, 0), kind="stable"),
}
for k, o in orders.items():
    print(json.dumps({"order": k, "ms": timeit(s8[o], t8[o])}), flush=True)
# per-hour cost: batches of 740 queries all from one hour band (repeat sources)
for band in range(0, 24, 3):
    sel = np.nonzero((ts // 3600 >= band) & (ts // 3600 < band + 3))[0][:740]
    print(json.dumps({"band": band, "n": int(sel.size), "ms": timeit(src[sel], ts[sel])}), flush=True)
