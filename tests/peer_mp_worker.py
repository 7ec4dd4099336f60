"""Worker of test_peer_exchange_two_processes (tests/test_gpu_parity.py), run
under torchrun; ranks may share one GPU: build with EAT_BUILD_MULTIPROCESS, exchange CUDA IPC handles over
torch.distributed (gloo), run collective queries, compare with the oracle."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import numpy as np, torch, torch.distributed as dist
import synth, oracle
from paper_1912_00966_b200.parallel import peer_partitioned_engine
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count())
dist.init_process_group("gloo")
cfg = sys.argv[1] if len(sys.argv) > 1 else "tiny"
tt = synth.generate(cfg)
eng = peer_partitioned_engine(tt)
csa = oracle.CSA(tt.num_vertices, *tt.arrays())
ok = True
t0 = time.perf_counter()
for s, t_s in [synth.SINGLE_QUERY, (5, 30000), (17, 70000)]:
    got = eng.query(s, t_s)
    ok &= bool(np.array_equal(got, csa.query(s, t_s)))
dt = time.perf_counter() - t0
print(json.dumps({"rank": rank, "world": world, "config": cfg, "parity": ok, "rounds": eng.stats()["last_rounds"],
                  "s_per_query": dt / 3}), flush=True)
dist.barrier()
dist.destroy_process_group()
