#!/usr/bin/env python
"""e2e A/B of eat_query_many into a page-locked host buffer (the bench's e2e
leg, city batch 10k): EAT_E2E_MODE 0 = two-stream chunk pipeline, 1 = direct
(kernel stores rows into the mapped host buffer), 2 = streamed (rows to device
memory, copy engine moves each finished 256-query chunk while the kernel runs).
Rows are checked identical across modes.  One JSON line per mode."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from paper_1912_00966_b200 import _lib  # noqa: E402

if os.environ.get("EAT_AB_LIB"):  # A/B of a libeat build (tools/build_variant.py)
    _lib.LIB_PATH = os.path.abspath(os.environ["EAT_AB_LIB"])
from paper_1912_00966_b200 import Engine, pinned_empty  # noqa: E402

tt = synth.generate("city")
src, ts = synth.queries(tt, 1000, 10)
h_src, h_ts = pinned_empty((src.size,)), pinned_empty((src.size,))
h_src[:] = src
h_ts[:] = ts
ref = None
for mode in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,0,2,1").split(",")]:
    os.environ["EAT_E2E_MODE"] = str(mode)
    eng = Engine.from_timetable(tt, subtrips=3)
    out = pinned_empty((src.size, tt.num_vertices))
    eng.query_many(h_src, h_ts, out=out)
    t0 = time.perf_counter()
    reps = 5
    for _ in range(reps):
        eng.query_many(h_src, h_ts, out=out)
    dt = (time.perf_counter() - t0) / reps
    if ref is None:
        ref = out.copy()
    print(json.dumps({"mode": mode, "e2e_qps": src.size / dt, "ms": dt * 1e3, "same_rows": bool(np.array_equal(ref, out))}),
          flush=True)
    eng.close()
