"""Where does a CTA-kernel sweep go? select vs relaxation-phase cycles (instrumented build), city."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1912_00966_b200 import Engine
tt = synth.generate("city")
src, ts = synth.queries(tt, 1000, 10)
d_src = torch.tensor(src.astype(np.int32), device="cuda"); d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
for kw in (dict(subtrips=2), dict(subtrips=2, cta_threads=512), dict(subtrips=0)):
    e = Engine.from_timetable(tt, counters=True, **kw)
    e.query_many_device(d_src, d_ts, out); torch.cuda.synchronize()
    st = e.stats(); sw = st["sweeps_total"]
    print(json.dumps({**kw, "sweeps_per_query": sw / src.size, "select_cycles_per_sweep": st["select_cycles"] / sw,
                      "pair_cycles_per_sweep": st["pair_cycles"] / sw,
                      "select_loop_per_sweep": st["select_loop_cycles"] / sw, "pair_loop_per_sweep": st["pair_loop_cycles"] / sw,
                      "type_evals_per_sweep": st["type_evals"] / sw, "visits_per_sweep": st["vertex_visits"] / sw}), flush=True)
    # single query (1024-thread CTA is uninstrumented): batch of 1 through the device batch path
    e1 = Engine.from_timetable(tt, counters=True, **kw)
    one_s = torch.tensor([0], dtype=torch.int32, device="cuda"); one_t = torch.tensor([21600], dtype=torch.int32, device="cuda")
    o1 = torch.empty((1, tt.num_vertices), dtype=torch.int32, device="cuda")
    e1.query_many_device(one_s, one_t, o1); torch.cuda.synchronize()
    st = e1.stats(); sw = st["sweeps_total"]
    print(json.dumps({**kw, "alone": True, "sweeps": sw, "select_cycles_per_sweep": st["select_cycles"] / sw,
                      "pair_cycles_per_sweep": st["pair_cycles"] / sw, "select_loop_per_sweep": st["select_loop_cycles"] / sw,
                      "pair_loop_per_sweep": st["pair_loop_cycles"] / sw, "type_evals_per_sweep": st["type_evals"] / sw}), flush=True)
