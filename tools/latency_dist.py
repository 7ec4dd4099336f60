"""Single-query latency distribution (100 seeded (s, t_s) per
config, p50/p90): device time per query (CUDA events; L2 flushed before each
query), sweeps, parity against the oracle on the first K queries.
Usage: python tools/latency_dist.py city,metro,country [nq] [parity_k] [kernel]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
from paper_1912_00966_b200 import Engine

cfgs = (sys.argv[1] if len(sys.argv) > 1 else "city,metro").split(",")
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 100
pk = int(sys.argv[3]) if len(sys.argv) > 3 else 10
kernel = sys.argv[4] if len(sys.argv) > 4 else "auto"
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
for cfg in cfgs:
    tt = synth.generate(cfg)
    eng = Engine.from_timetable(tt, subtrips=3, kernel=kernel)
    rng = np.random.default_rng(7)
    qs = [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(nq)]
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    for s, t in qs[:3]:
        eng.query_device(s, t, out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms, sweeps = [], []
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    ok = True
    cpu_ms = []
    for i, (s, t) in enumerate(qs):
        flush.fill_(i)
        a.record(); eng.query_device(s, t, out); b.record(); b.synchronize()
        ms.append(a.elapsed_time(b))
        sweeps.append(eng.stats()["last_sweeps"])
        if i < pk:
            t0 = time.perf_counter()
            want = csa.query(s, t)
            cpu_ms.append((time.perf_counter() - t0) * 1e3)
            ok &= bool(np.array_equal(out.cpu().numpy().astype(np.uint32), want))
    ms = np.array(ms)
    print(json.dumps({"config": cfg, "kernel": eng.stats()["kernel_name"], "queries": nq, "seed": 7, "subtrips": 3,
                      "l2": "flushed before each query", "p50_ms": float(np.percentile(ms, 50)),
                      "p90_ms": float(np.percentile(ms, 90)), "mean_ms": float(ms.mean()), "max_ms": float(ms.max()),
                      "sweeps_p50": float(np.median(sweeps)), "sweeps_max": int(max(sweeps)),
                      "parity_checked": pk, "parity": ok, "oracle_ms_mean_1core": float(np.mean(cpu_ms)) if cpu_ms else None}),
          flush=True)
    eng.close()
