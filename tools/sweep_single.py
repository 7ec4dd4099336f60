"""Single-query latency of the global-e[] kernels (frontier, async, edge partition P=1) on one config."""
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
out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
ref = None
rng = np.random.default_rng(5)
queries = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(4)]
for kw in [dict(kernel="frontier"), dict(kernel="async"), dict(mode="edge_partitioned", part_count=1),
           dict(kernel="cta")]:
    try:
        eng = Engine.from_timetable(tt, **kw)
    except Exception as e:
        print(json.dumps({"config": name, **kw, "error": str(e)[:120]}), flush=True)
        continue
    for (s, t_s) in queries:
        for _ in range(2):
            eng.query_device(s, t_s, out)
        torch.cuda.synchronize()
        ms = []
        for _ in range(5):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            eng.query_device(s, t_s, out)
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
        st = eng.stats()
        print(json.dumps({"config": name, **kw, "q": [s, t_s], "ms": float(np.median(ms)), "sweeps": st["last_sweeps"],
                          "rounds": st["last_rounds"], "reached": int((out.cpu().numpy().astype(np.uint32) < 0x7FFFFFFF).sum())}),
              flush=True)
    eng.close()
