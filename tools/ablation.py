"""NEXT-3: the paper's incremental versions on B200 (Table II
shape) + cluster-size and virtual-warp sweeps (Figs. 3-4).
Mean ms per query over random queries (the paper's protocol),
device time, plus serial CSA on one host core.  Every variant's rows are
checked against the oracle."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import synth
from paper_1912_00966_b200 import Engine

name = sys.argv[1] if len(sys.argv) > 1 else "city"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 20
tt = synth.generate(name)
src, ts = synth.queries(tt, nq, 1, seed=11)
csa = oracle.CSA(tt.num_vertices, *tt.arrays())
t0 = time.perf_counter()
want = csa.query_many(src, ts)
cpu_ms = (time.perf_counter() - t0) * 1e3 / nq
print(json.dumps({"config": name, "variant": "serial CSA (oracle, 1 core)", "ms": cpu_ms}), flush=True)
out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")

VARIANTS = [
    ("Connection (Alg. 4, thread/connection, full sweep)", dict(kernel="connection")),
    ("Connection-type (Alg. 5, linear, thread/type)", dict(kernel="full_sweep", lookup="linear")),
    ("Connection-type-AP (Alg. 6 over all APs, thread/type)", dict(kernel="full_sweep", lookup="ap")),
    ("Cluster-AP (thread/type, full sweep)", dict(kernel="full_sweep")),
    ("Edge-like (thread/vertex, frontier)", dict(kernel="frontier", subwarp=1)),
    ("Warps (warp/vertex, frontier)", dict(kernel="frontier", subwarp=32)),
    ("Warps + sub-trips", dict(kernel="frontier", subwarp=32, subtrips=2)),
    ("CTA kernel (1 CTA, e[] in smem, window)", dict(kernel="cta")),
    ("CTA kernel + sub-trips", dict(kernel="cta", subtrips=2)),
]
VARIANTS += [(f"Cluster size {cs // 60} min (Warps)", dict(kernel="frontier", subwarp=32, cluster_seconds=cs))
             for cs in (1800, 900, 300)]
VARIANTS += [(f"Virtual warp {sw} lanes", dict(kernel="frontier", subwarp=sw)) for sw in (2, 4, 8, 16)]
for label, kw in VARIANTS:
    try:
        eng = Engine.from_timetable(tt, **kw)
    except Exception as e:
        print(json.dumps({"config": name, "variant": label, "error": str(e)[:120]}), flush=True)
        continue
    ok = True
    for i in range(min(nq, 3)):
        eng.query_device(int(src[i]), int(ts[i]), out)
        ok &= bool(np.array_equal(out.cpu().numpy().astype(np.uint32), want[i]))
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for i in range(nq):
        eng.query_device(int(src[i]), int(ts[i]), out)
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / nq
    print(json.dumps({"config": name, "variant": label, "ms": ms, "speedup_vs_csa": cpu_ms / ms,
                      "sweeps_last": eng.stats()["last_sweeps"], "parity": ok}), flush=True)
    eng.close()
