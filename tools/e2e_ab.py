"""e2e A/B of eat_query_many with a pinned host output: direct (kernel stores
rows into the mapped host buffer) vs the two-stream chunk pipeline."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1912_00966_b200 import Engine
from paper_1912_00966_b200.engine import pinned_empty
tt = synth.generate("city")
src, ts = synth.queries(tt, 1000, 10)
ref = None
for direct in (1, 0, 1):
    os.environ["EAT_E2E_DIRECT"] = str(direct)
    eng = Engine.from_timetable(tt, subtrips=2)
    out = pinned_empty((src.size, tt.num_vertices))
    hs = pinned_empty(src.shape); hs[:] = src
    ht = pinned_empty(ts.shape); ht[:] = ts
    for _ in range(3):
        eng.query_many(hs, ht, out=out)
    t = []
    for _ in range(5):
        t0 = time.perf_counter(); eng.query_many(hs, ht, out=out); t.append(time.perf_counter() - t0)
    ref = out.copy() if ref is None else ref
    print(json.dumps({"direct": direct, "ms": 1e3 * float(np.median(t)), "qps": src.size / float(np.median(t)),
                      "same": bool(np.array_equal(ref, out))}), flush=True)
    eng.close()
