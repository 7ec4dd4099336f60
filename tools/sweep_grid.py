"""Sweep the grid (single-query, global e[]) kernel variants on one config."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1912_00966_b200 import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "metro"
tt = synth.generate(name)
s, t_s = synth.SINGLE_QUERY
out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
ref = None
variants = [dict(subwarp=8, window=0x7FFFFFFF), dict(subwarp=0, window=0x7FFFFFFF), dict(subwarp=0, window=7200),
            dict(subwarp=0, window=3600), dict(subwarp=0, window=1800), dict(subwarp=0, window=900),
            dict(subwarp=32, window=0x7FFFFFFF), dict(subwarp=1, window=0x7FFFFFFF)]
for kw in variants:
    eng = Engine.from_timetable(tt, kernel="frontier", **kw)
    for _ in range(3):
        eng.query_device(s, t_s, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        eng.query_device(s, t_s, out)
    b.record()
    b.synchronize()
    got = out.cpu().numpy()
    ref = got if ref is None else ref
    print(json.dumps({"config": name, **kw, "ms": a.elapsed_time(b) / 10, "sweeps": eng.stats()["last_sweeps"],
                      "same": bool(np.array_equal(ref, got))}), flush=True)
    eng.close()
