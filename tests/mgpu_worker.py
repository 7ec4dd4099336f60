"""Worker of tests/test_multigpu.py, run under torchrun with one process per
GPU (NCCL): the edge-partitioned single query across real devices with the
NCCL min-allreduce exchange (to local quiescence and one allreduce per
sweep) and with the in-kernel peer exchange over NVLink; every rank
compares its rows with the oracle and prints one JSON line."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import numpy as np, torch, torch.distributed as dist
import synth, oracle
from paper_1912_00966_b200.parallel import edge_partitioned_engine, peer_partitioned_engine

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
cfg = sys.argv[1] if len(sys.argv) > 1 else "tiny"
tt = synth.generate(cfg)
csa = oracle.CSA(tt.num_vertices, *tt.arrays())
qs = [synth.SINGLE_QUERY, (5, 30000), (17, 70000)]
want = [csa.query(*q) for q in qs]
res = {"rank": rank, "world": world, "config": cfg, "device": dev}
for name, mk in (("allreduce", lambda: edge_partitioned_engine(tt, device=dev)),
                 ("allreduce_per_sweep", lambda: edge_partitioned_engine(tt, device=dev, local_sweeps=1)),
                 ("peer", lambda: peer_partitioned_engine(tt, device=dev))):
    eng = mk()
    ok = all(np.array_equal(eng.query(*q), w) for q, w in zip(qs, want))
    res[name] = {"parity": bool(ok), "rounds": eng.stats()["last_rounds"]}
    eng.close()
    dist.barrier()
print(json.dumps(res), flush=True)
dist.destroy_process_group()
