"""ncu driver: one batched metro launch through k_query_groups (e[] in global memory)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_1912_00966_b200 import Engine
tt = synth.generate("metro")
eng = Engine.from_timetable(tt, subtrips=3)
src, ts = synth.queries(tt, 256, 4)
d_src = torch.tensor(src.astype(np.int32), device="cuda")
d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
for _ in range(2):
    eng.query_many_device(d_src, d_ts, out)
torch.cuda.synchronize()
