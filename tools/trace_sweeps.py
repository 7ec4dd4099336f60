"""Per-sweep timeline of the grid frontier kernel (EAT_EXP_TRACE build):
sweep start, slowest CTA's work end, barrier exit (globaltimer ns), frontier size.
Usage: python tools/trace_sweeps.py ab/libeat_trace.so metro"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1912_00966_b200 import _lib
_lib.LIB_PATH = os.path.abspath(sys.argv[1])
from paper_1912_00966_b200 import Engine
tt = synth.generate(sys.argv[2] if len(sys.argv) > 2 else "metro")
eng = Engine.from_timetable(tt, subtrips=2, kernel="frontier")
o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
L = _lib.lib()
buf = (ctypes.c_ulonglong * (4096 * 4))()
for rep in range(3):
    L.eat_debug_trace(buf, 1)
    eng.query_device(*synth.SINGLE_QUERY, o1)
    torch.cuda.synchronize()
L.eat_debug_trace(buf, 0)
a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, 4).astype(np.int64)
ns = eng.stats()["last_sweeps"]
a = a[:ns]
work = a[:, 1] - a[:, 0]
bar = a[:, 2] - a[:, 1]
gap = np.r_[a[1:, 0] - a[:-1, 2], 0]
tot = a[-1, 2] - a[0, 0]
print(json.dumps({"sweeps": int(ns), "total_us": tot / 1e3, "work_us_mean": work.mean() / 1e3, "work_us_p50": float(np.median(work)) / 1e3,
                  "barrier_tail_us_mean": bar.mean() / 1e3, "gap_us_mean": gap[:-1].mean() / 1e3,
                  "frontier_mean": float(a[:, 3].mean()), "frontier_max": int(a[:, 3].max())}))
for i in list(range(0, ns, max(1, ns // 25))):
    print(i, int(a[i, 3]), round(work[i] / 1e3, 2), round(bar[i] / 1e3, 2))

buf2 = (ctypes.c_ulonglong * (4096 * 8))()
L.eat_debug_trace2(buf2)
b = np.frombuffer(buf2, dtype=np.uint64).reshape(-1, 8).astype(np.int64)[:ns]
print("warp 0 of CTA 0 (frontier entry 0): ns from its start: [h0 loads, h0 relaxed, h0 ballot, h1 loads, h1 relaxed, h1 ballot]; sweep start->entry start")
for i in list(range(0, ns, max(1, ns // 25))):
    r = b[i]
    if r[0] == 0:
        continue
    print(i, [int(v - r[0]) if v else None for v in r[1:7]], int(r[0] - a[i, 0]))
