"""Sweep CTA-kernel variants (threads per query x e[] width) on the city batch."""
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
for subtrips in (2, 0):
    for bits in (16, 32):
        for threads in (512, 384, 256, 192, 128):
            try:
                eng = Engine.from_timetable(tt, cta_threads=threads, arr_bits=bits, subtrips=subtrips)
            except Exception as e:
                print(json.dumps({"threads": threads, "bits": bits, "error": str(e)[:100]}), flush=True)
                continue
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
            chk = out[:256].cpu().numpy()
            ref = chk if ref is None else ref
            print(json.dumps({"subtrips": subtrips, "bits": bits, "threads": threads, "batch_ms": ms,
                              "qps": src.size / ms * 1e3, "same_rows": bool(np.array_equal(ref, chk))}), flush=True)
            eng.close()
