"""Multi-GPU parity (needs >= 2 devices; skipped otherwise): the N > 1 code
paths of SURVEY 8(e) on real devices, one process per GPU.

* e2 edge-partitioned single query: NCCL min-allreduce of e[] per exchange
  round (libeat's own communicator) and the in-kernel peer exchange (CUDA IPC
  mapped blocks, system-scope atomics over NVLink) -- tests/mgpu_worker.py;
* e1 query sharding inside one process: a multi-device handle
  (eat_build_opts.devices) on the city batch.
Every row is compared with the oracle."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ndev():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.fixture(scope="module", autouse=True)
def _need_two():
    if _ndev() < 2:
        pytest.skip("needs >= 2 CUDA devices")


@pytest.mark.timeout(600)
@pytest.mark.parametrize("cfg", ["tiny", "city"])
def test_edge_partitioned_across_gpus(cfg):
    world = min(_ndev(), 4)
    port = 29500 + os.getpid() % 2000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mgpu_worker.py"), cfg]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=540, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert sorted(d["rank"] for d in lines) == list(range(world))
    for d in lines:
        for k in ("allreduce", "allreduce_per_sweep", "peer"):
            assert d[k]["parity"], (k, d)


def test_multi_device_batch_city():
    import oracle
    import synth
    from paper_1912_00966_b200 import Engine

    tt = synth.generate("city")
    devs = list(range(_ndev()))
    eng = Engine.from_timetable(tt, devices=devs, subtrips=3)
    src, ts = synth.queries(tt, 100, 4)
    got = eng.query_many(src, ts)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    rows = np.arange(0, src.size, 7)
    assert np.array_equal(got[rows], csa.query_many(src[rows], ts[rows]))
