#!/bin/bash
# frontier-kernel single-query latency vs CTAs per SM (grid barrier cost)
for g in 1 2 4 8; do
  EAT_GRID_CTAS_PER_SM=$g python - <<'PY'
import json, os, sys
sys.path.insert(0, ".")
import numpy as np, torch, synth
from paper_1912_00966_b200 import Engine
for name in ("city", "metro"):
    tt = synth.generate(name)
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    for sw in (32, 8):
        eng = Engine.from_timetable(tt, kernel="frontier", subwarp=sw)
        for _ in range(3): eng.query_device(*synth.SINGLE_QUERY, out)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10): eng.query_device(*synth.SINGLE_QUERY, out)
        b.record(); b.synchronize()
        print(json.dumps({"ctas_per_sm": int(os.environ["EAT_GRID_CTAS_PER_SM"]), "config": name, "subwarp": sw,
                          "ms": a.elapsed_time(b) / 10, "sweeps": eng.stats()["last_sweeps"]}), flush=True)
        eng.close()
PY
done
