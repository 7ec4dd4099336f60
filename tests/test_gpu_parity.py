"""GPU parity: the CUDA path (through the C ABI) against the oracle, element
by element, bit-exact (integer seconds; EAT_INF for unreachable).

Run on a B200 via gpurun:  python -m pytest tests -m gpu -x -q
"""
import numpy as np
import pytest

import oracle
import synth
from oracle import INF

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1912_00966_b200 import Engine, EatError, _lib  # noqa: E402

KERNELS = ["cta", "frontier", "full_sweep", "async", "bitmap", "cluster", "grid_async"]


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _types_raw(tt):
    """(u, v, lambda) -> sorted departures, from the RAW timetable (caller ids)."""
    order = np.lexsort((tt.dep, tt.dur, tt.v, tt.u))
    u, v, d, t = tt.u[order], tt.v[order], tt.dur[order], tt.dep[order]
    key = np.stack([u, v, d], 1)
    brk = np.nonzero(np.any(key[1:] != key[:-1], axis=1))[0] + 1
    starts = np.concatenate([[0], brk])
    ends = np.concatenate([brk, [len(u)]])
    return {(int(u[a]), int(v[a]), int(d[a])): t[a:b] for a, b in zip(starts, ends)}


def _assert_rows(got, want, what):
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)
        i = tuple(x[0] for x in bad)
        raise AssertionError(f"{what}: {len(bad[0])} mismatches, first at {i}: got {got[i]} want {want[i]}")


# ----------------------------------------------------------------------------- lookup kernel
@pytest.mark.parametrize("name,cs", [("tiny", 3600), ("tiny", 900), ("city", 3600)])
def test_lookup_kernel_vs_get_connection(name, cs):
    tt = synth.generate(name)
    eng = Engine.from_timetable(tt, cluster_seconds=cs)
    ex = eng.export()
    inv = np.empty(tt.num_vertices, np.int64)
    inv[ex["perm"].astype(np.int64)] = np.arange(tt.num_vertices)
    raw = _types_raw(tt)
    rng = np.random.default_rng(1)
    T = ex["type_rec"].shape[0]
    ts = rng.choice(T, min(T, 3000), replace=False)
    types, bounds, want = [], [], []
    for t in ts:
        rec = ex["type_rec"][t]
        deps = raw[(int(inv[rec[6]]), int(inv[rec[0]]), int(rec[1]))]
        cand = np.concatenate([deps, deps + 1, deps - 1, [0, deps[-1] + 1, int(rng.integers(0, 100000))]])
        cand = np.unique(cand[cand >= 0])
        for b in cand:
            g = oracle.get_connection(deps.tolist(), int(b))
            types.append(t)
            bounds.append(b)
            want.append(INF if g is None else g)
    dt = torch.tensor(np.array(types, np.int64).astype(np.int32), device="cuda")
    db = torch.tensor(np.array(bounds, np.int64).astype(np.int32), device="cuda")
    out = torch.empty_like(dt)
    eng.lookup_device(dt, db, out)
    torch.cuda.synchronize()
    _assert_rows(out.cpu().numpy().astype(np.uint32), np.array(want, np.uint32), f"lookup {name} cs={cs}")


def test_device_selftest():
    """eat_selftest: the fp32 ceil-division of Algorithm 6 (every 12-bit
    operand pair) and the reciprocal-multiply hour cluster (every e < 2^31,
    for several cluster widths) are exact on this device."""
    tt = synth.generate("tiny")
    for cs in (3600, 1, 7, 60, 900, 4095, 4096):
        eng = Engine.from_timetable(tt, cluster_seconds=cs)
        assert eng.selftest() == (0, 0), cs
        eng.close()


# ----------------------------------------------------------------------------- single queries
@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("subwarp", [0, 1, 8, 64])
def test_tiny_single_queries(kernel, subwarp):
    tt = synth.generate("tiny")
    eng = Engine.from_timetable(tt, kernel=kernel, subwarp=subwarp)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    rng = np.random.default_rng(subwarp)
    qs = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 90000))) for _ in range(30)]
    for s, t_s in qs:
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"tiny {kernel}/{subwarp} q=({s},{t_s})")
    st = eng.stats()
    assert st["kernel_name"] == kernel and st["last_sweeps"] >= 1


@pytest.mark.parametrize("kernel", KERNELS)
def test_random_small_instances(kernel):
    """>= 1000 (instance, query) pairs with lambda=0, duplicates, self-loops,
    multi-day departures (SPEC S:348 engine-equivalence property)."""
    npairs = 0
    for seed in range(400 if kernel != "full_sweep" else 150):
        tt = synth.random_small(seed)
        eng = Engine.from_timetable(tt, kernel=kernel, cluster_seconds=[3600, 600, 4096, 60][seed % 4],
                                    subwarp=[1, 2, 4, 8, 16, 32, 0, 64][seed % 8],
                                    cta_threads=[256, 384, 512, 192, 128][seed % 5], arr_bits=[16, 32][seed % 2],
                                    cluster_dir=["auto", "dense", "compact"][seed % 3],
                                    continuation=[None, 0, 2, 4, 64, 1, 16][seed % 7],
                                    cluster_ctas=[0, 2, 4, 8, 16, 16][seed % 6],
                                    window=[0, 60, 0x7FFFFFFF][seed % 3] if kernel == "cluster" else 0)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        rng = np.random.default_rng(seed)
        for _ in range(3):
            s, t_s = int(rng.integers(tt.num_vertices)), int(rng.integers(0, 2 * 86400))
            _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"seed {seed} {kernel} q=({s},{t_s})")
            npairs += 1
        eng.close()
    assert npairs >= 450


def test_edge_cases():
    # one vertex, no connections (every single-query kernel)
    eng = Engine(1, [], [], [], [])
    assert eng.query(0, 5).tolist() == [5]
    for kernel in KERNELS:
        if kernel == "connection":
            continue
        e1 = Engine(1, [], [], [], [], kernel=kernel)
        assert e1.query(0, 5).tolist() == [5], kernel
        e1.close()
    # a few vertices, one connection (bitmap words beyond the graph on most CTAs)
    for kernel in KERNELS:
        e3 = Engine(3, [0], [2], [10], [5], kernel=kernel)
        assert e3.query(0, 7).tolist() == [7, INF, 15], kernel
        assert e3.query(0, 11).tolist() == [11, INF, INF], kernel
        e3.close()
    # isolated source, late start, t_s = 0, t_s = INF-1
    tt = synth.generate("tiny")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    for kernel in KERNELS:
        eng = Engine.from_timetable(tt, kernel=kernel)
        for s, t_s in [(0, 0), (0, 200000), (5, INF - 1), (199, 86399)]:
            _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"edge {kernel} ({s},{t_s})")
        with pytest.raises(EatError) as e:
            eng.query(tt.num_vertices, 0)
        assert e.value.status == _lib.EAT_EINVAL
        with pytest.raises(EatError) as e:
            eng.query(0, INF)
        assert e.value.status == _lib.EAT_ERANGE


def test_query_device_and_stream():
    tt = synth.generate("tiny")
    eng = Engine.from_timetable(tt)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        eng.query_device(3, 30000, out, stream=s)
    s.synchronize()
    _assert_rows(out.cpu().numpy().astype(np.uint32), csa.query(3, 30000), "query_device")


# ----------------------------------------------------------------------------- batched
def test_tiny_batched_all_rows():
    tt = synth.generate("tiny")
    eng = Engine.from_timetable(tt)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    src, ts = synth.queries(tt, 100, 10)
    _assert_rows(eng.query_many(src, ts), csa.query_many(src, ts), "tiny batch host")
    d_src = torch.tensor(src.astype(np.int32), device="cuda")
    d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
    out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
    eng.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize()
    _assert_rows(out.cpu().numpy().astype(np.uint32), csa.query_many(src, ts), "tiny batch device")


def test_batched_invalid_rows_on_device():
    tt = synth.generate("tiny")
    eng = Engine.from_timetable(tt)
    d_src = torch.tensor([0, tt.num_vertices + 3, 1], dtype=torch.int32, device="cuda")
    d_ts = torch.tensor([100, 100, -1], dtype=torch.int32, device="cuda")  # -1 -> 0xFFFFFFFF >= INF
    out = torch.zeros((3, tt.num_vertices), dtype=torch.int32, device="cuda")
    eng.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize()
    o = out.cpu().numpy().astype(np.uint32)
    assert np.all(o[1] == INF) and np.all(o[2] == INF) and o[0][0] == 100
    assert eng.stats()["invalid_queries"] >= 2


def test_city_batch_full_size_sampled():
    """BASELINE configs[2]: city network, 10k queries (1000 sources x 10
    times, seed 7) in the bench's launch configuration (kernel auto -> the
    batched CTA kernel, 256 threads, window 1200 s, sub-trips r = 3, as
    bench.py builds it); 120 sampled rows compared with the oracle one by
    one (bench.py itself compares every row its CPU baseline solved)."""
    tt = synth.generate("city")
    eng = Engine.from_timetable(tt, kernel="auto", subtrips=3)
    st = eng.stats()
    assert st["cta_grid"] > 0 and st["num_shortcuts"] > 0
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    src, ts = synth.queries(tt, 1000, 10)
    d_src = torch.tensor(src.astype(np.int32), device="cuda")
    d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
    out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
    eng.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize()
    rows = np.random.default_rng(7).choice(src.size, 120, replace=False)
    got = out[torch.tensor(rows, device="cuda")].cpu().numpy().astype(np.uint32)
    _assert_rows(got, csa.query_many(src[rows], ts[rows]), "city batch sampled rows")
    # host e2e paths (pageable -> pinned staging; pinned -> direct), several pipeline chunks
    want = csa.query_many(src[:2500:5], ts[:2500:5])
    _assert_rows(eng.query_many(src[:2500:5], ts[:2500:5]), want, "city batch host pageable")
    from paper_1912_00966_b200 import pinned_empty

    pin = pinned_empty((500, tt.num_vertices))
    _assert_rows(eng.query_many(src[:2500:5], ts[:2500:5], out=pin), want, "city batch host pinned")
    full = pinned_empty((src.size, tt.num_vertices))
    eng.query_many(src, ts, out=full)
    _assert_rows(full[rows], csa.query_many(src[rows], ts[rows]), "city batch host pinned, all 10k")


@pytest.mark.parametrize("kernel", KERNELS)
def test_city_single_query(kernel):
    """BASELINE configs[1]: s=0, t_s=06:00, plus 10 seeded queries."""
    tt = synth.generate("city")
    eng = Engine.from_timetable(tt, kernel=kernel)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    rng = np.random.default_rng(11)
    qs = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(10)]
    for s, t_s in qs:
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"city {kernel} ({s},{t_s})")


def test_metro_single_query():
    """BASELINE configs[3]: metro network, global e[] (frontier kernel)."""
    tt = synth.generate("metro")
    eng = Engine.from_timetable(tt)
    assert eng.stats()["kernel_name"] in ("frontier", "cta", "async", "cluster", "grid_async")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    for s, t_s in [synth.SINGLE_QUERY, (777, 30000)]:
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"metro ({s},{t_s})")
    for kernel in ("frontier", "async", "cluster", "grid_async"):
        e2 = Engine.from_timetable(tt, kernel=kernel)
        for s, t_s in [synth.SINGLE_QUERY, (91, 50000)]:
            _assert_rows(e2.query(s, t_s), csa.query(s, t_s), f"metro {kernel} ({s},{t_s})")


@pytest.mark.parametrize("name,kernel,nq", [("city", "cluster", 300), ("metro", "grid_async", 100),
                                             ("city", "grid_async", 100)])
def test_async_kernels_many_queries(name, kernel, nq):
    """The asynchronous single-query kernels (the bench's AUTO choice for
    city / metro) on many seeded queries at full size, every stop of every
    row against the oracle (their termination is timing-dependent: many
    queries exercise many interleavings)."""
    tt = synth.generate(name)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    eng = Engine.from_timetable(tt, kernel=kernel, subtrips=3)
    rng = np.random.default_rng(2024)
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
    for i in range(nq):
        s, t_s = int(rng.integers(tt.num_vertices)), int(rng.integers(0, 2 * 86400))
        eng.query_device(s, t_s, out)
        _assert_rows(out.cpu().numpy().view(np.uint32), csa.query(s, t_s), f"{name} {kernel} q{i}=({s},{t_s})")
    eng.close()
    csa.close()


@pytest.mark.parametrize("stops,irregular", [(3000, 0.0), (30000, 0.3), (60000, 0.3)])
def test_auto_single_query_sizes(stops, irregular):
    """AUTO's single-query choice across graph sizes (cluster kernel with the
    whole index on chip, cluster with type ranges only, grid-async): every
    row vs the oracle on seeded queries."""
    tt = synth.generate("custom", stops=stops, edges=3 * stops, conns=60 * stops, irregular=irregular, seed=stops)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    eng = Engine.from_timetable(tt, subtrips=3)
    st = eng.stats()
    assert st["kernel_name"] in ("cluster", "grid_async"), st["kernel_name"]
    rng = np.random.default_rng(stops)
    for _ in range(12):
        s, t_s = int(rng.integers(tt.num_vertices)), int(rng.integers(0, 2 * 86400))
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"{stops} stops {st['kernel_name']} ({s},{t_s})")
    eng.close()
    csa.close()


@pytest.mark.parametrize("ctas", [2, 4, 8, 16])
def test_cluster_kernel_sizes(ctas):
    """EAT_KERNEL_CLUSTER with every cluster size: e[] spread over 2..16
    CTAs' shared memory (DSMEM), tiny + city queries incl. invalid-free
    repeats on one handle, sub-trips r = 3."""
    for name in ("tiny", "city"):
        tt = synth.generate(name)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        eng = Engine.from_timetable(tt, kernel="cluster", cluster_ctas=ctas, subtrips=3,
                                    cluster_sync=(ctas == 4))  # the synchronous variant too
        st = eng.stats()
        assert st["kernel_name"] == "cluster" and st["cluster_ctas"] == ctas
        rng = np.random.default_rng(ctas)
        qs = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(6)]
        for s, t_s in qs:
            _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"{name} cluster{ctas} ({s},{t_s})")
        eng.close()


def test_metro_batched_groups():
    """a12 with e[] in global memory: batched metro queries run as CTA groups
    of one launch (several queries in flight); every row equals the oracle's,
    invalid queries give INF rows (device path)."""
    import torch

    tt = synth.generate("metro")
    eng = Engine.from_timetable(tt, subtrips=3)
    assert eng.stats()["cta_grid"] == 0  # e[] exceeds shared memory
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    src, ts = synth.queries(tt, 12, 3)
    _assert_rows(eng.query_many(src, ts), csa.query_many(src, ts), "metro batch (host)")
    bad_s = src.astype(np.int64).copy()
    bad_s[5] = tt.num_vertices + 3
    d_src = torch.tensor(bad_s.astype(np.int32), device="cuda")
    d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
    out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
    eng.query_many_device(d_src, d_ts, out)
    got = out.cpu().numpy().astype(np.uint32)
    assert (got[5] == INF).all()
    keep = np.arange(src.size) != 5
    want = csa.query_many(src[keep], ts[keep])
    _assert_rows(got[keep], want, "metro batch (device)")
    # goal-directed on the same path: e[dst] only
    dst = (np.arange(src.size, dtype=np.int64) * 7919) % tt.num_vertices
    tgt = eng.query_targets(src, ts, dst.astype(np.uint32))
    full = csa.query_many(src, ts)
    assert np.array_equal(tgt, full[np.arange(src.size), dst])


@pytest.mark.timeout(600)
def test_metro_batched_chunked_pipeline():
    """eat_query_many with more queries than one pipeline chunk (640 metro
    rows): chunk kernels share one compute stream (cooperative grid-group
    launches must not overlap), row copies overlap on the copy stream;
    pageable and page-locked outputs; sampled rows equal the oracle's."""
    from paper_1912_00966_b200 import pinned_empty

    tt = synth.generate("metro")
    eng = Engine.from_timetable(tt, subtrips=3)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    src, ts = synth.queries(tt, 350, 4, seed=5)  # 1,400 queries: 3 chunks
    pin = pinned_empty((src.size, tt.num_vertices))
    for out in (None, pin):
        got = eng.query_many(src, ts, out=out)
        for i in list(range(0, src.size, 173)) + [src.size - 1]:
            _assert_rows(got[i:i + 1], csa.query_many(src[i:i + 1], ts[i:i + 1]), f"metro chunked row {i}")


def test_device_calls_on_two_streams_are_ordered():
    """Device calls on one handle from different streams (no user sync in
    between) run one after another: rows stay exact, and cooperative grid
    kernels never overlap (they would deadlock)."""
    import torch

    tt = synth.generate("metro")
    eng = Engine.from_timetable(tt, subtrips=3)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    qs = [synth.SINGLE_QUERY, (4242, 40000), (99, 70000)]
    outs = [torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda") for _ in qs]
    src, ts = synth.queries(tt, 4, 2, seed=9)
    d_src = torch.tensor(src.astype(np.int32), device="cuda")
    d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
    rows = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
    for k, (q, o) in enumerate(zip(qs, outs)):
        eng.query_device(*q, o, stream=s1 if k % 2 == 0 else s2)
        if k == 1:
            eng.query_many_device(d_src, d_ts, rows, stream=s1)
    torch.cuda.synchronize()
    for q, o in zip(qs, outs):
        _assert_rows(o.cpu().numpy().astype(np.uint32)[None], csa.query(*q)[None], f"two streams {q}")
    _assert_rows(rows.cpu().numpy().astype(np.uint32), csa.query_many(src, ts), "two streams batch")


def test_grouped_batches_random_small():
    """k_query_groups on adversarial small instances (explicit FRONTIER kernel
    routes batches to the grouped grid kernel even when e[] fits shared
    memory): every row equals the oracle's, invalid rows are INF."""
    import torch

    for seed in range(120):
        tt = synth.random_small(9000 + seed)
        eng = Engine.from_timetable(tt, kernel="frontier", subwarp=[32, 16, 8, 1][seed % 4],
                                    continuation=[None, 0, 2][seed % 3])
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        rng = np.random.default_rng(seed)
        nq = int(rng.integers(1, 70))
        src = rng.integers(0, tt.num_vertices, nq).astype(np.uint32)
        ts = rng.integers(0, 2 * 86400, nq).astype(np.uint32)
        _assert_rows(eng.query_many(src, ts), csa.query_many(src, ts), f"groups seed {seed}")
        if seed % 10 == 0:  # device path with an invalid query
            bad = src.astype(np.int64)
            bad[0] = tt.num_vertices
            out = torch.empty((nq, tt.num_vertices), dtype=torch.int32, device="cuda")
            eng.query_many_device(torch.tensor(bad.astype(np.int32), device="cuda"),
                                  torch.tensor(ts.astype(np.int32), device="cuda"), out)
            got = out.cpu().numpy().astype(np.uint32)
            assert (got[0] == INF).all()
            if nq > 1:
                _assert_rows(got[1:], csa.query_many(src[1:], ts[1:]), f"groups device seed {seed}")
        eng.close()


# ----------------------------------------------------------------------------- edge partition
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_edge_partitioned_loopback(P):
    """e2 on one GPU: P edge partitions (eat_partition_range slices) with the
    exchange as a device min-merge instead of NCCL -- same local-phase kernel,
    same round/termination protocol as the multi-GPU path."""
    for name in ("tiny", "city"):
        tt = synth.generate(name)
        eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=P)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        rng = np.random.default_rng(P)
        qs = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(4)]
        for s, t_s in qs:
            _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"loopback P={P} {name} ({s},{t_s})")
        assert eng.stats()["last_rounds"] >= 1
    for seed in range(40):
        tt = synth.random_small(3000 + seed)
        eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=P)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        s, t_s = seed % tt.num_vertices, (seed * 7919) % 86400
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"loopback P={P} seed {seed}")


@pytest.mark.parametrize("local_sweeps", [1, 2, 5])
def test_edge_partitioned_bounded_rounds_loopback(local_sweeps):
    """e2 with at most `local_sweeps` local sweeps per exchange round
    (eat_build_opts.local_sweeps; 1 = the north star's one allreduce(min)
    per sweep): vertices left on a bounded local frontier re-enter the next
    round; e[] equals the oracle's and the round count grows as the bound
    tightens."""
    for name in ("tiny", "city"):
        tt = synth.generate(name)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        free = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=2)
        eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=2, local_sweeps=local_sweeps)
        rng = np.random.default_rng(local_sweeps)
        qs = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(3)]
        for s, t_s in qs:
            _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"bounded {local_sweeps} {name} ({s},{t_s})")
        free.query(*synth.SINGLE_QUERY)
        eng.query(*synth.SINGLE_QUERY)
        assert eng.stats()["last_rounds"] >= free.stats()["last_rounds"]
        if local_sweeps == 1:  # one exchange per sweep
            assert eng.stats()["last_rounds"] >= eng.stats()["last_sweeps"] // 2
    for seed in range(30):
        tt = synth.random_small(3100 + seed)
        eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=[2, 3, 4][seed % 3],
                                    local_sweeps=local_sweeps, subwarp=[32, 8, 1][seed % 3])
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        s, t_s = seed % tt.num_vertices, (seed * 7919) % (2 * 86400)
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"bounded {local_sweeps} seed {seed}")
    with pytest.raises(EatError) as e:  # replicated handles have no exchange rounds
        Engine.from_timetable(synth.generate("tiny"), local_sweeps=1)
    assert e.value.status == _lib.EAT_EINVAL


def test_multi_device_handle():
    """eat_build_opts.devices: one replica per listed
    device, eat_query_many shards the batch over them in-library (one host
    thread per device).  With one GPU the list is [0]; with two or more the
    batch really spans devices.  Rows equal the oracle's."""
    tt = synth.generate("tiny")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    src, ts = synth.queries(tt, 50, 3)
    want = csa.query_many(src, ts)
    ndev = torch.cuda.device_count()
    devs = list(range(min(ndev, 4)))
    eng = Engine.from_timetable(tt, devices=devs)
    assert eng.stats()["num_devices"] == len(devs)
    _assert_rows(eng.query_many(src, ts), want, f"devices {devs}")
    dst = (np.arange(src.size) * 13 % tt.num_vertices).astype(np.uint32)
    assert np.array_equal(eng.query_targets(src, ts, dst), want[np.arange(src.size), dst])
    _assert_rows(eng.query(*synth.SINGLE_QUERY), csa.query(*synth.SINGLE_QUERY), "multi-device handle single")
    eng.close()
    with pytest.raises(EatError) as e:
        Engine.from_timetable(tt, devices=[0, 0])
    assert e.value.status == _lib.EAT_EINVAL
    with pytest.raises(EatError) as e:
        Engine.from_timetable(tt, devices=[0, 1], mode="edge_partitioned", part_count=2)
    assert e.value.status == _lib.EAT_EUNSUPPORTED


@pytest.mark.parametrize("P", [1, 2, 3, 4, 8, 16])
def test_edge_partitioned_peer_exchange_loopback(P):
    """NEXT-2 on one GPU: P edge partitions as P CTA groups of one launch, the
    exchange in-kernel (peer atomicMin on the owner's e[] + owner inbox +
    cross-partition barrier in device memory) -- the code path a multi-GPU
    run takes with IPC-mapped peer pointers."""
    for name in ("tiny", "city"):
        tt = synth.generate(name)
        eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=P, exchange="peer",
                                    subtrips=2 if name == "city" else 0)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        rng = np.random.default_rng(100 + P)
        qs = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(6)]
        for s, t_s in qs:  # repeated queries on one handle: round base / message slots carry over
            _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"peer P={P} {name} ({s},{t_s})")
            st = eng.stats()
            assert st["last_rounds"] >= 1 and st["last_sweeps"] >= 1
        eng.close()
    for seed in range(60):
        tt = synth.random_small(5000 + seed)
        eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=P, exchange="peer",
                                    subwarp=[32, 8, 1, 4][seed % 4], continuation=[None, 0, 3][seed % 3])
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        for k in range(2):
            s, t_s = (seed + k) % tt.num_vertices, (seed * 7919 + k * 3001) % (2 * 86400)
            _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"peer P={P} seed {seed}")
        eng.close()


def test_peer_exchange_api_errors():
    tt = synth.generate("tiny")
    loop = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=2, exchange="peer")
    with pytest.raises(EatError) as e:
        loop.peer_export()
    assert e.value.status == _lib.EAT_ESTATE
    rank1 = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=1, part_count=2, exchange="peer",
                                  multiprocess=True)
    assert len(rank1.peer_export()) == _lib.EAT_PEER_HANDLE_BYTES
    with pytest.raises(EatError) as e:  # not connected yet
        rank1.query(*synth.SINGLE_QUERY)
    assert e.value.status == _lib.EAT_ESTATE
    with pytest.raises(EatError) as e:
        rank1.peer_connect([b"\0" * 64] * 3)
    assert e.value.status == _lib.EAT_EINVAL
    with pytest.raises(EatError) as e:
        Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=17, exchange="peer")
    assert e.value.status == _lib.EAT_EINVAL


def test_edge_partitioned_single_rank():
    tt = synth.generate("tiny")
    eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=0, part_count=1)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    for s, t_s in [synth.SINGLE_QUERY, (17, 40000)]:
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), "edge-partitioned P=1")
    assert eng.stats()["last_rounds"] == 1


@pytest.mark.parametrize("window", [0, 60, 600, 3600])
def test_window_schedules_same_fixpoint(window):
    """The CTA schedule's time window only reorders relaxations (R12): the
    fixpoint, and so e[], is identical for every window."""
    tt = synth.generate("tiny")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    eng = Engine.from_timetable(tt, window=window if window else 0x7FFFFFFF, cta_threads=[256, 384, 512][window % 3],
                                arr_bits=[16, 32][window % 2])
    src, ts = synth.queries(tt, 50, 4)
    _assert_rows(eng.query_many(src, ts), csa.query_many(src, ts), f"window {window}")
    for seed in range(60):
        t2 = synth.random_small(1000 + seed)
        c2 = oracle.CSA(t2.num_vertices, *t2.arrays())
        e2 = Engine.from_timetable(t2, window=window if window else 0x7FFFFFFF, kernel="cta")
        rng = np.random.default_rng(seed)
        s, t_s = int(rng.integers(t2.num_vertices)), int(rng.integers(0, 86400))
        _assert_rows(e2.query(s, t_s), c2.query(s, t_s), f"window {window} seed {seed}")


@pytest.mark.timeout(900)
def test_country_single_query():
    """BASELINE configs[4] at N=1: country (1M stops, ~300M connections),
    s=0 at 06:00 plus 3 seeded queries, every stop compared with the oracle:
    replicated frontier kernel (the bench's single-query configuration,
    sub-trips r = 3), the edge-partitioned code path at P=1, NCCL-free
    loopback P=2 (device min-merge rounds) and the in-kernel peer exchange
    at P=2 (loopback)."""
    tt = synth.generate("country")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    rng = np.random.default_rng(44)
    qs = [synth.SINGLE_QUERY] + [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(3)]
    want = [csa.query(*q) for q in qs]
    # the bench's kernel (AUTO = grid_async here) on 12 more seeded queries
    more = [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 2 * 86400))) for _ in range(12)]
    want_more = [csa.query(*q) for q in more]
    csa.close()
    eng = Engine.from_timetable(tt, subtrips=3)
    assert eng.stats()["kernel_name"] in ("grid_async", "frontier")
    for q, w in zip(more, want_more):
        _assert_rows(eng.query(*q), w, f"country auto {q}")
    eng.close()
    for kw in ({"subtrips": 3, "kernel": "frontier"}, {"subtrips": 3, "kernel": "grid_async"}, {"mode": "edge_partitioned", "part_count": 1},
               {"mode": "edge_partitioned", "part_count": 2, "subtrips": 3},
               {"mode": "edge_partitioned", "part_count": 2, "exchange": "peer", "subtrips": 3}):
        eng = Engine.from_timetable(tt, **kw)
        for q, w in zip(qs, want):
            _assert_rows(eng.query(*q), w, f"country {kw} {q}")
        eng.close()


@pytest.mark.parametrize("kw", [dict(kernel="connection"), dict(kernel="full_sweep", lookup="linear"),
                                dict(kernel="full_sweep", lookup="ap"), dict(kernel="frontier", lookup="linear"),
                                dict(kernel="frontier", lookup="ap", subwarp=4)])
def test_ablation_versions(kw):
    """NEXT-3: the paper's incremental versions (Alg. 4, Alg. 5 linear, Alg. 6
    over all APs) give the oracle's arrival times too."""
    tt = synth.generate("tiny")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    eng = Engine.from_timetable(tt, **kw)
    for s, t_s in [synth.SINGLE_QUERY, (50, 40000), (199, 80000)]:
        _assert_rows(eng.query(s, t_s), csa.query(s, t_s), f"ablation {kw} ({s},{t_s})")
    for seed in range(60):
        t2 = synth.random_small(7000 + seed)
        c2 = oracle.CSA(t2.num_vertices, *t2.arrays())
        e2 = Engine.from_timetable(t2, cluster_seconds=[3600, 600][seed % 2], **kw)
        s, t_s = seed % t2.num_vertices, (seed * 4099) % 86400
        _assert_rows(e2.query(s, t_s), c2.query(s, t_s), f"ablation {kw} seed {seed}")


def test_arr16_overflow_recompute():
    """uint16 e[] offsets: queries whose arrivals pass t_s + 65534 s are
    recomputed with uint32 e[] (multi-day timetable, t_s = 0); rows exact."""
    rng = np.random.default_rng(9)
    n, m = 300, 6000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    dep = rng.integers(0, 3 * 86400, m)
    dur = rng.choice([60, 600, 3600, 7200], m)
    tt = synth.Timetable(n, *(np.asarray(x, np.uint32) for x in (u, v, dep, dur)))
    csa = oracle.CSA(n, *tt.arrays())
    src = rng.integers(0, n, 64).astype(np.uint32)
    ts = np.where(np.arange(64) % 2 == 0, 0, rng.integers(0, 2 * 86400, 64)).astype(np.uint32)
    want = csa.query_many(src, ts)
    assert ((want != INF) & (want - ts[:, None] >= 0xFFFF)).any(), "fixture must overflow uint16 offsets"
    for bits in (16, 32):
        eng = Engine.from_timetable(tt, arr_bits=bits)
        _assert_rows(eng.query_many(src, ts), want, f"arr_bits={bits} multi-day")
        d = [torch.tensor(x.astype(np.int32), device="cuda") for x in (src, ts)]
        out = torch.empty((64, n), dtype=torch.int32, device="cuda")
        eng.query_many_device(d[0], d[1], out)
        torch.cuda.synchronize()
        _assert_rows(out.cpu().numpy().astype(np.uint32), want, f"arr_bits={bits} multi-day device")


def test_goal_directed_targets():
    """NEXT-4: eat_query_many_target returns the oracle's e[dst] (pruned
    search on the CTA kernel; full query + gather on the grid path)."""
    for name, nq in (("tiny", 400), ("city", 300), ("metro", 6)):
        tt = synth.generate(name)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        rng = np.random.default_rng(17)
        src, ts = synth.queries(tt, nq, 1, seed=3)
        dst = rng.integers(0, tt.num_vertices, src.size).astype(np.uint32)
        dst[::7] = src[::7]  # target == source
        want = csa.query_many(src, ts)[np.arange(src.size), dst]
        for kw in ({}, {"window": 0x7FFFFFFF}, {"subtrips": 2}):
            eng = Engine.from_timetable(tt, **kw)
            _assert_rows(eng.query_targets(src, ts, dst), want, f"targets {name} {kw}")
            eng.close()
    for seed in range(80):
        tt = synth.random_small(5000 + seed)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        eng = Engine.from_timetable(tt)
        rng = np.random.default_rng(seed)
        src = rng.integers(0, tt.num_vertices, 5).astype(np.uint32)
        ts = rng.integers(0, 86400, 5).astype(np.uint32)
        dst = rng.integers(0, tt.num_vertices, 5).astype(np.uint32)
        want = csa.query_many(src, ts)[np.arange(5), dst]
        _assert_rows(eng.query_targets(src, ts, dst), want, f"targets seed {seed}")


@pytest.mark.parametrize("scheme", [1, 2, 3, 1003])
def test_subtrips_parity(scheme):
    """NEXT-1: the index with sub-trip shortcuts gives the oracle's arrival
    times of the ORIGINAL timetable (batched + single kernels)."""
    for name in ("tiny", "city"):
        tt = synth.generate(name)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        src, ts = synth.queries(tt, 40, 5)
        for kernel in ("cta", "frontier"):
            eng = Engine.from_timetable(tt, subtrips=scheme, kernel=kernel)
            assert eng.stats()["num_shortcuts"] > 0
            _assert_rows(eng.query(*synth.SINGLE_QUERY), csa.query(*synth.SINGLE_QUERY), f"subtrips {name} {kernel}")
        _assert_rows(eng.query_many(src, ts), csa.query_many(src, ts), f"subtrips {name} batch")


def test_peer_exchange_two_processes():
    """EAT_EXCHANGE_PEER across processes: two torchrun ranks (sharing the
    GPU when there is only one) map each other's exchange blocks with CUDA
    IPC handles exchanged over torch.distributed and run collective queries
    through system-scope peer atomics; every rank must return the oracle's e[]."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    port = 29000 + os.getpid() % 2000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), os.path.join(root, "tests", "peer_mp_worker.py"), "tiny"]
    env = dict(os.environ, EAT_GRID_CTAS_PER_SM="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=240, env=env, cwd=root)
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert r.returncode == 0, r.stderr[-2000:]
    assert sorted(d["rank"] for d in lines) == [0, 1] and all(d["parity"] for d in lines), lines


def test_query_into_caller_buffers():
    """eat_query writes a page-locked caller buffer directly and a pageable one
    through the pinned stage; both equal the oracle."""
    from paper_1912_00966_b200 import pinned_empty

    tt = synth.generate("tiny")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    for kernel in ("cta", "frontier"):
        eng = Engine.from_timetable(tt, kernel=kernel)
        pin = pinned_empty((tt.num_vertices,))
        page = np.zeros(tt.num_vertices, np.uint32)
        for s, t_s in [synth.SINGLE_QUERY, (9, 50000)]:
            want = csa.query(s, t_s)
            assert eng.query(s, t_s, out=pin) is pin and np.array_equal(pin, want)
            assert eng.query(s, t_s, out=page) is page and np.array_equal(page, want)
        with pytest.raises(ValueError):
            eng.query(0, 0, out=np.zeros(3, np.uint32))
        eng.close()
