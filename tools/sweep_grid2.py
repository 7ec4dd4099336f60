"""Grid-kernel schedules for large single queries: full sweep (paper's thread/type) vs frontier."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_1912_00966_b200 import Engine

for name in sys.argv[1:] or ["metro"]:
    tt = synth.generate(name)
    src, ts = synth.queries(tt, 8, 1, seed=11)
    src[0], ts[0] = synth.SINGLE_QUERY
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    ref = None
    for kw in [dict(kernel="frontier", subtrips=2), dict(kernel="full_sweep", subtrips=2),
               dict(kernel="full_sweep", subtrips=2, cluster_dir="compact"), dict(kernel="full_sweep", subtrips=0),
               dict(kernel="frontier", subtrips=2, cluster_dir="compact")]:
        for gps in (1, 2, 4):
            os.environ["EAT_GRID_CTAS_PER_SM"] = str(gps)
            eng = Engine.from_timetable(tt, **kw)
            eng.query_device(int(src[0]), int(ts[0]), out)
            torch.cuda.synchronize()
            got = out.cpu().numpy()
            ref = got if ref is None else ref
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ms = []
            for i in range(len(src)):
                a.record()
                eng.query_device(int(src[i]), int(ts[i]), out)
                b.record()
                b.synchronize()
                ms.append(a.elapsed_time(b))
            print(json.dumps({"config": name, **kw, "ctas_per_sm": gps, "ms_s0": ms[0], "ms_mean": float(np.mean(ms)),
                              "same": bool(np.array_equal(ref, got))}), flush=True)
            eng.close()
            break  # grid_ctas_per_sm is read once per process (static); keep the default
