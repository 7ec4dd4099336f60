"""Edge-partitioned single query on one GPU: P partitions with the NCCL-style
allreduce rounds (device min-merge) vs the in-kernel peer exchange (NEXT-2),
parity-checked against the oracle.  Usage: python tools/peer_loopback.py config [P,...]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth, oracle
from paper_1912_00966_b200 import Engine
cfg = sys.argv[1] if len(sys.argv) > 1 else "metro"
Ps = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
tt = synth.generate(cfg)
csa = oracle.CSA(tt.num_vertices, *tt.arrays())
s, t = synth.SINGLE_QUERY
want = csa.query(s, t)
o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
for P in Ps:
    for ex in ("allreduce", "peer"):
        eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=P, exchange=ex, subtrips=2)
        for _ in range(2):
            eng.query_device(s, t, o1)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for _ in range(5):
            a.record(); eng.query_device(s, t, o1); b.record(); b.synchronize()
            ms.append(a.elapsed_time(b))
        st = eng.stats()
        print(json.dumps({"config": cfg, "P": P, "exchange": ex, "ms": float(np.median(ms)), "rounds": st["last_rounds"],
                          "sweeps": st["last_sweeps"], "parity": bool(np.array_equal(o1.cpu().numpy().astype(np.uint32), want))}), flush=True)
        eng.close()
