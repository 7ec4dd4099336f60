"""Batched queries on graphs whose e[] does not fit shared memory (metro):
CTA groups of the grid kernel (EAT_BATCH_GROUPS) x queries; q/s and parity
of sampled rows against the oracle.  Usage: python tools/sweep_groups.py [config] [nq]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1912_00966_b200 import _lib
if os.environ.get("EAT_AB_LIB"):
    _lib.LIB_PATH = os.path.abspath(os.environ["EAT_AB_LIB"])
from paper_1912_00966_b200 import Engine
cfg = sys.argv[1] if len(sys.argv) > 1 else "metro"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 256
tt = synth.generate(cfg)
src, ts = synth.queries(tt, nq // 4, 4)
csa = oracle.CSA(tt.num_vertices, *tt.arrays())
want = {i: csa.query(int(src[i]), int(ts[i])) for i in range(0, nq, nq // 8)}
d_src = torch.tensor(src.astype(np.int32), device="cuda")
d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
out = torch.empty((nq, tt.num_vertices), dtype=torch.int32, device="cuda")
for g in [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4,8,16,37,74").split(",")]:
    os.environ["EAT_BATCH_GROUPS"] = str(g)
    eng = Engine.from_timetable(tt, subtrips=3)
    eng.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); eng.query_many_device(d_src, d_ts, out); b.record(); b.synchronize()
    ms = a.elapsed_time(b)
    ok = all(np.array_equal(out[i].cpu().numpy().astype(np.uint32), w) for i, w in want.items())
    print(json.dumps({"lib": os.path.basename(os.environ.get("EAT_AB_LIB", "libeat.so")), "config": cfg, "groups": g, "queries": nq, "ms": ms, "qps": nq / ms * 1e3, "parity_sampled": ok}), flush=True)
    eng.close()
