"""Country/metro single query with the full-sweep (thread per type) grid kernel -- the
HBM-streaming schedule of SURVEY 8(d) -- for an ncu dram__bytes capture."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_1912_00966_b200 import Engine
name = sys.argv[1] if len(sys.argv) > 1 else "country"
kernel = sys.argv[2] if len(sys.argv) > 2 else "full_sweep"
tt = synth.generate(name)
eng = Engine.from_timetable(tt, kernel=kernel, subtrips=2)
out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
for _ in range(2):
    eng.query_device(*synth.SINGLE_QUERY, out)
torch.cuda.synchronize()
st = eng.stats()
print("sweeps", st["last_sweeps"], "types", st["num_types"], "index_bytes", st["index_bytes"])
