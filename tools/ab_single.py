"""Single-query latency (s=0, 06:00) of the grid frontier kernel on a config,
with a given libeat.so build; parity against the oracle.
Usage: python tools/ab_single.py path/to/libeat.so config [kernel]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1912_00966_b200 import _lib
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_1912_00966_b200 import Engine
cfg = sys.argv[2]
kernel = sys.argv[3] if len(sys.argv) > 3 else "auto"
subwarp = int(sys.argv[4]) if len(sys.argv) > 4 else 0
tt = synth.generate(cfg)
eng = Engine.from_timetable(tt, subtrips=int(os.environ.get("EAT_AB_SUBTRIPS", "3")), kernel=kernel, subwarp=subwarp,
                            continuation=int(os.environ["EAT_AB_CONT"]) if "EAT_AB_CONT" in os.environ else None)
o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
src, ts = synth.queries(tt, 4, 1, seed=11)
qs = [synth.SINGLE_QUERY] + list(zip(src.tolist(), ts.tolist()))
res = {}
import oracle
csa = oracle.CSA(tt.num_vertices, *tt.arrays())
for (s, t) in qs:
    for _ in range(2):
        eng.query_device(s, t, o1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(5):
        flush.fill_(1)
        a.record(); eng.query_device(s, t, o1); b.record(); b.synchronize()
        ms.append(a.elapsed_time(b))
    ok = bool(np.array_equal(o1.cpu().numpy().astype(np.uint32), csa.query(s, t)))
    res[f"{s}@{t}"] = {"ms": float(np.median(ms)), "sweeps": eng.stats()["last_sweeps"], "parity": ok}
print(json.dumps({"lib": os.path.basename(sys.argv[1]), "config": cfg, "kernel": kernel, "subwarp": subwarp, "cont": os.environ.get("EAT_AB_CONT"),
                  "mean_ms": float(np.mean([v["ms"] for v in res.values()])), "queries": res}), flush=True)
