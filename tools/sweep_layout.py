"""Dense vs compact cluster directory: city batch (CTA kernel) and metro single query (grid kernel)."""
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
ref = None
for cd in ("dense", "compact"):
    for threads in (256, 384):
        for bits in (32, 16):
            eng = Engine.from_timetable(tt, cta_threads=threads, arr_bits=bits, subtrips=2, cluster_dir=cd)
            for _ in range(2):
                eng.query_many_device(d_src, d_ts, out)
            ms = timed(lambda: eng.query_many_device(d_src, d_ts, out), 3)
            chk = out[:256].cpu().numpy()
            ref = chk if ref is None else ref
            o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
            sms = timed(lambda: eng.query_device(*synth.SINGLE_QUERY, o1), 20)
            print(json.dumps({"config": "city", "dir": cd, "threads": threads, "bits": bits, "batch_ms": ms,
                              "qps": src.size / ms * 1e3, "single_ms": sms, "index_MB": eng.stats()["index_bytes"] / 1e6,
                              "same_rows": bool(np.array_equal(ref, chk))}), flush=True)
            eng.close()
tt = synth.generate("metro")
o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
for cd in ("dense", "compact"):
    for sub in (2, 0):
        eng = Engine.from_timetable(tt, subtrips=sub, cluster_dir=cd)
        for _ in range(3):
            eng.query_device(*synth.SINGLE_QUERY, o1)
        ms = timed(lambda: eng.query_device(*synth.SINGLE_QUERY, o1), 10)
        print(json.dumps({"config": "metro", "dir": cd, "subtrips": sub, "single_ms": ms,
                          "sweeps": eng.stats()["last_sweeps"], "index_MB": eng.stats()["index_bytes"] / 1e6}), flush=True)
        eng.close()
