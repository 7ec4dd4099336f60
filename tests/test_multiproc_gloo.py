"""world_size-2 CPU tests (gloo) of the multi-GPU host logic.

1. Query-parallel sharding: contiguous shards, all-gather
   in query order == the full batch (solver injected: the oracle on CPU,
   Engine.query_many on GPUs).
2. Edge-partitioned exchange protocol (e2), as run by libeat's
   part_query: each rank owns the out-types of the internal vertex range
   given by eat_partition_range; per round it relaxes from the owned
   vertices lowered since the last exchange to local quiescence, flags any
   lowered non-owned vertex, then min-allreduces e[] ++ flag; it stops when
   no rank flagged.  The relaxation here is a plain test-side model on the
   raw connections (the CUDA local phase is covered by the GPU parity tests);
   what is checked is the partition cut and the round/termination protocol.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INF = 0x7FFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    import sys

    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    return res


def _sharded_batch(rank, world):
    import oracle
    import synth
    from paper_1912_00966_b200.parallel import query_many_sharded, shard_range

    tt = synth.generate("tiny")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    src, ts = synth.queries(tt, 13, 3)  # 39 queries: uneven shards
    lo, hi = shard_range(src.size, rank, world)
    full = query_many_sharded(csa.query_many, src, ts)
    want = csa.query_many(src, ts)
    return bool(np.array_equal(full, want)) and (hi - lo) in (19, 20)


def _edge_protocol(rank, world):
    import oracle
    import synth
    from paper_1912_00966_b200 import Engine

    tt = synth.generate("tiny")
    eng = Engine.from_timetable(tt, host_only=True)
    perm = eng.export()["perm"].astype(np.int64)
    lo, hi = eng.partition_range(rank, world)
    owned = (perm >= lo) & (perm < hi)  # caller ids owned by this rank
    n = tt.num_vertices
    out_edges = {}
    for i in np.nonzero(owned[tt.u])[0]:
        out_edges.setdefault(int(tt.u[i]), []).append((int(tt.v[i]), int(tt.dep[i]), int(tt.dur[i])))
    ok = True
    # local_sweeps (eat_build_opts): 0 = local phase to quiescence; k = at
    # most k sweeps per round, vertices left on the local frontier keep
    # prev = INF (so they re-enter next round) and force another round
    for local_sweeps, (s, t_s) in [(ls, q) for ls in (0, 1, 2) for q in [(0, 21600), (57, 30000), (199, 80000)]]:
        arr = np.full(n + 1, INF, dtype=np.int64)
        arr[s] = t_s
        prev = np.full(n, INF, dtype=np.int64)
        rounds = 0
        while True:
            rounds += 1
            work = [x for x in range(n) if owned[x] and arr[x] < prev[x]]
            remote = False
            sweeps = 0
            while work and not (local_sweeps and sweeps >= local_sweeps):
                nxt = set()
                for x in work:
                    for (v, d, lam) in out_edges.get(x, []):
                        if arr[x] <= d and d + lam < arr[v]:
                            arr[v] = d + lam
                            if owned[v]:
                                nxt.add(v)
                            else:
                                remote = True
                work = sorted(nxt)
                sweeps += 1
            prev[:] = arr[:n]
            for x in work:  # left on a bounded local frontier
                prev[x] = INF
            arr[n] = 0 if (remote or work) else 1
            t = torch.from_numpy(arr.copy())
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            arr = t.numpy().astype(np.int64)
            if arr[n] == 1:
                break
            assert rounds < 4 * n
        ok &= np.array_equal(arr[:n].astype(np.uint32), oracle.csa(n, *tt.arrays(), s, t_s))
    # the partition cut covers every type exactly once across ranks
    cnt = torch.tensor([int(eng.export()["type_ptr"][hi]) - int(eng.export()["type_ptr"][lo])])
    dist.all_reduce(cnt)
    ok &= int(cnt.item()) == int(eng.stats()["num_types"])
    return bool(ok)


def _peer_handles(rank, world):
    from paper_1912_00966_b200.parallel import exchange_peer_handles

    got = exchange_peer_handles(bytes([rank + 1]) * 64)
    return got == [bytes([r + 1]) * 64 for r in range(world)]


def test_peer_handle_exchange_gloo():
    """NEXT-2 plumbing: every rank gets all exchange-block handles in rank order."""
    assert _run(_peer_handles) == {0: True, 1: True}


def test_query_sharding_gloo():
    assert _run(_sharded_batch) == {0: True, 1: True}


def test_edge_partition_protocol_gloo():
    assert _run(_edge_protocol) == {0: True, 1: True}


def test_peer_exchange_protocol_model():
    """NEXT-2 round protocol (peer.cu), modelled on the raw connections with a
    random relaxation order: each partition drains its inbox, relaxes owned
    vertices to local quiescence, lowers a remote vertex in its replica and in
    the owner's e[] and, if the owner's value dropped, queues it once per round
    in the owner's inbox; the query ends after a round with no message.  The
    result must be the oracle's for every partition count and order."""
    import sys

    sys.path.insert(0, ROOT)
    import oracle
    import synth
    from paper_1912_00966_b200 import Engine

    for seed in range(30):
        tt = synth.random_small(7000 + seed)
        n = tt.num_vertices
        eng = Engine.from_timetable(tt, host_only=True)
        perm = eng.export()["perm"].astype(np.int64)
        rng = np.random.default_rng(seed)
        for P in (1, 2, 3, 5):
            rngs = [eng.partition_range(p, P) for p in range(P)]
            owner = np.empty(n, np.int64)
            for p, (lo, hi) in enumerate(rngs):
                owner[(perm >= lo) & (perm < hi)] = p
            out = {}
            for i in range(tt.u.size):
                out.setdefault(int(tt.u[i]), []).append((int(tt.v[i]), int(tt.dep[i]), int(tt.dur[i])))
            s, t_s = int(rng.integers(n)), int(rng.integers(0, 2 * 86400))
            arr = [np.full(n, INF, np.int64) for _ in range(P)]  # replicas
            arr[owner[s]][s] = t_s
            inbox = [set() for _ in range(P)]
            frontier = [{s} if owner[s] == p else set() for p in range(P)]
            rounds = 0
            while True:
                rounds += 1
                new_inbox = [set() for _ in range(P)]
                for p in rng.permutation(P):
                    work = frontier[p] | inbox[p]
                    while work:
                        x = int(rng.choice(sorted(work)))
                        work.discard(x)
                        for (v, d, lam) in out.get(x, []):
                            if arr[p][x] <= d and d + lam < arr[p][v]:
                                arr[p][v] = d + lam
                                o = owner[v]
                                if o == p:
                                    work.add(v)
                                elif d + lam < arr[o][v]:
                                    arr[o][v] = d + lam
                                    new_inbox[o].add(v)
                    frontier[p] = set()
                inbox = new_inbox
                if not any(inbox):
                    break
                assert rounds < 4 * n + 8
            got = np.array([arr[owner[v]][v] for v in range(n)], np.uint32)
            assert np.array_equal(got, oracle.csa(n, *tt.arrays(), s, t_s)), (seed, P)
