#!/bin/bash
# frontier vs bitmap grid kernels x CTAs per SM, single queries (8 random + s0), sub-trips 2
for g in 1 2 4; do
EAT_GRID_CTAS_PER_SM=$g python - "$@" <<'PY'
import json, os, sys
sys.path.insert(0, ".")
import numpy as np, torch, synth
from paper_1912_00966_b200 import Engine
for name in sys.argv[1:]:
    tt = synth.generate(name)
    src, ts = synth.queries(tt, 8, 1, seed=11)
    src[0], ts[0] = synth.SINGLE_QUERY
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    ref = None
    for kernel in ("frontier", "bitmap"):
        eng = Engine.from_timetable(tt, kernel=kernel, subtrips=2)
        for _ in range(2): eng.query_device(int(src[0]), int(ts[0]), out)
        torch.cuda.synchronize()
        got = out.cpu().numpy(); ref = got if ref is None else ref
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for i in range(len(src)):
            a.record(); eng.query_device(int(src[i]), int(ts[i]), out); b.record(); b.synchronize()
            ms.append(a.elapsed_time(b))
        print(json.dumps({"config": name, "kernel": kernel, "ctas_per_sm": int(os.environ["EAT_GRID_CTAS_PER_SM"]),
                          "ms_s0": ms[0], "ms_mean": float(np.mean(ms)), "sweeps": eng.stats()["last_sweeps"],
                          "same": bool(np.array_equal(ref, got))}), flush=True)
        eng.close()
PY
done
