"""Sub-trip schemes (NEXT-1): sweeps, latency, batch throughput."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1912_00966_b200 import Engine

for name in sys.argv[1:] or ["city", "metro"]:
    tt = synth.generate(name)
    src, ts = synth.queries(tt, 1000, 10)
    ref = None
    for scheme in (0, 1, 2, 3, 4, 6):
        row = {"config": name, "subtrips": scheme}
        eng = Engine.from_timetable(tt, subtrips=scheme)
        st = eng.stats()
        row.update(kernel=st["kernel_name"], shortcuts=st["num_shortcuts"], types=st["num_types"])
        out1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
        for _ in range(3):
            eng.query_device(*synth.SINGLE_QUERY, out1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            eng.query_device(*synth.SINGLE_QUERY, out1)
        b.record()
        b.synchronize()
        row.update(single_ms=a.elapsed_time(b) / 10, single_sweeps=eng.stats()["last_sweeps"])
        got = out1.cpu().numpy()
        ref = got if ref is None else ref
        row["same_as_scheme0"] = bool(np.array_equal(ref, got))
        if name == "city":
            d_src = torch.tensor(src.astype(np.int32), device="cuda")
            d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
            out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
            for _ in range(2):
                eng.query_many_device(d_src, d_ts, out)
            torch.cuda.synchronize()
            a.record()
            for _ in range(3):
                eng.query_many_device(d_src, d_ts, out)
            b.record()
            b.synchronize()
            row.update(batch_ms=a.elapsed_time(b) / 3, qps=src.size / (a.elapsed_time(b) / 3) * 1e3)
        print(json.dumps(row), flush=True)
        eng.close()
