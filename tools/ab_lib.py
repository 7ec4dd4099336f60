"""Time the city batch (10k queries, device buffers) with a given libeat.so
build (A/B of kernel versions on one box).  Usage: python tools/ab_lib.py path/to/libeat.so"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1912_00966_b200 import _lib
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_1912_00966_b200 import Engine
tt = synth.generate("city")
src, ts = synth.queries(tt, 1000, 10)
d_src = torch.tensor(src.astype(np.int32), device="cuda")
d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
subtrips = int(sys.argv[2]) if len(sys.argv) > 2 else 2
eng = Engine.from_timetable(tt, subtrips=subtrips, window=int(os.environ.get("EAT_AB_WINDOW", "0")),
                            cta_threads=int(os.environ.get("EAT_AB_THREADS", "0")))
for _ in range(3):
    eng.query_many_device(d_src, d_ts, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ms = []
for _ in range(7):
    a.record(); eng.query_many_device(d_src, d_ts, out); b.record(); b.synchronize()
    ms.append(a.elapsed_time(b))
o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
for _ in range(3):
    eng.query_device(*synth.SINGLE_QUERY, o1)
a.record()
for _ in range(20):
    eng.query_device(*synth.SINGLE_QUERY, o1)
b.record(); b.synchronize()
print(json.dumps({"lib": os.path.basename(sys.argv[1]), "subtrips": subtrips, "window": int(os.environ.get("EAT_AB_WINDOW", "0")), "threads": int(os.environ.get("EAT_AB_THREADS", "0")), "shortcuts": eng.stats()["num_shortcuts"], "batch_ms_med": float(np.median(ms)), "qps": src.size / float(np.median(ms)) * 1e3,
                  "single_ms": a.elapsed_time(b) / 20, "crc": int(out[::97].sum().item()), "crc1": int(o1.sum().item())}), flush=True)
