"""Pins for oracle/ (CPU only, no GPU).

Every check here compares the oracle against something other than itself:
values printed in the paper / SPEC (tests/golden/paper_examples.json),
brute-force enumeration of the EAT definition, an independent label-setting
algorithm, a textbook shortest-path routine (scipy) on a reduction, a closed
form, and invariants.  A dropped term, a wrong inequality (<= vs <), a wrong
index or the missing lambda=0 closure each fail at least one of them.
"""
import json
import os
import random

import numpy as np
import pytest

import oracle
from oracle import INF

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")


def _values(spec):
    if isinstance(spec, str):
        assert spec.startswith("range(")
        return list(eval(spec, {"range": range}))  # fixture-controlled literal
    return list(spec)


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _csa_conns(n, conns, s, ts, with_parent=False):
    a = np.array(conns, dtype=np.uint32).reshape(-1, 4)
    return oracle.csa(n, a[:, 0], a[:, 1], a[:, 2], a[:, 3], s, ts, with_parent)


# --------------------------------------------------------------------- paper values
def test_golden_csa(golden):
    for ex in golden["csa"]:
        e = _csa_conns(ex["n"], ex["conns"], ex["s"], ex["t_s"])
        assert e.tolist() == ex["e"], ex["cite"]
        assert oracle.brute_force_eat(ex["n"], ex["conns"], ex["s"], ex["t_s"]) == ex["e"], ex["cite"]


def test_golden_ap_cover(golden):
    for ex in golden["ap_cover"]:
        vals = _values(ex["values"])
        got = oracle.greedy_ap_cover(vals)
        assert [list(t) for t in got] == ex["aps"], ex["cite"]
        assert sorted(oracle.expand_aps(got)) == sorted(vals)


def test_golden_alg6(golden):
    for ex in golden["alg6"]:
        aps = [tuple(t) for t in ex["aps"]]
        assert oracle.get_connection_from_aps(aps, ex["bound"]) == ex["t_c"], ex["cite"]
        assert oracle.get_connection(oracle.expand_aps(aps), ex["bound"]) == ex["t_c"], ex["cite"]


def test_golden_cluster_lookup(golden):
    for ex in golden["cluster_lookup"]:
        deps = _values(ex["departures"])
        assert oracle.cluster_ap_lookup(deps, ex["bound"]) == ex["t_c"], ex["cite"]
        assert oracle.get_connection(deps, ex["bound"]) == ex["t_c"], ex["cite"]


def test_plain_alg1_needs_tie_closure():
    """The tie fixture would FAIL under a literal single pass of Algorithm 1:
    (1,2,100,5) is scanned before (0,1,100,0).  Guards reading R1."""
    conns = [(1, 2, 100, 5), (0, 1, 100, 0)]
    e = [INF, INF, INF]
    e[0] = 50
    for (u, v, t, lam) in conns:  # literal Alg. 1 order, no closure
        if e[u] <= t and t + lam < e[v]:
            e[v] = t + lam
    assert e[2] == INF
    assert _csa_conns(3, conns, 0, 50).tolist() == [50, 100, 105]


# --------------------------------------------------------------------- brute force
def _rand_instance(rng, nmax=7, cmax=9, tmax=30, lams=(0, 1, 2, 5, 10)):
    n = rng.randint(1, nmax)
    m = rng.randint(0, cmax)
    conns = [(rng.randrange(n), rng.randrange(n), rng.randint(0, tmax), rng.choice(lams)) for _ in range(m)]
    return n, conns


def test_csa_equals_brute_force_random():
    rng = random.Random(1912)
    for _ in range(2500):
        n, conns = _rand_instance(rng)
        s, ts = rng.randrange(n), rng.randint(0, 20)
        want = oracle.brute_force_eat(n, conns, s, ts)
        if conns:
            got = _csa_conns(n, conns, s, ts).tolist()
        else:
            got = oracle.csa(n, [], [], [], [], s, ts).tolist()
        assert got == want, (n, conns, s, ts)


def test_td_dijkstra_equals_brute_force_random():
    rng = random.Random(77)
    for _ in range(1500):
        n, conns = _rand_instance(rng)
        s, ts = rng.randrange(n), rng.randint(0, 20)
        assert oracle.td_dijkstra(n, conns, s, ts) == oracle.brute_force_eat(n, conns, s, ts)


def test_csa_equals_td_dijkstra_medium():
    rng = random.Random(2024)
    for it in range(200):
        n = rng.randint(2, 50)
        m = rng.randint(1, 2000)
        conns = [(rng.randrange(n), rng.randrange(n), rng.randint(0, 5000), rng.choice((0, 1, 30, 60, 300, 900)))
                 for _ in range(m)]
        for _q in range(3):
            s, ts = rng.randrange(n), rng.randint(0, 3000)
            assert _csa_conns(n, conns, s, ts).tolist() == oracle.td_dijkstra(n, conns, s, ts)


# --------------------------------------------------------------------- textbook reduction
def test_static_shortest_path_reduction():
    """If every edge departs every 60 s over the whole horizon with one
    duration w (a multiple of 60) and t_s is a multiple of 60, waiting is
    never needed beyond 0 s, so e[v] = t_s + dist(s, v) where dist is the
    static shortest-path distance (scipy.sparse.csgraph.dijkstra)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra

    rng = np.random.default_rng(5)
    n, m_edges = 30, 80
    W = np.full((n, n), np.inf)
    for _ in range(m_edges):
        a, b = rng.integers(0, n, 2)
        if a != b:
            W[a, b] = min(W[a, b], 60 * int(rng.integers(1, 11)))
    ts = 60 * 100
    horizon = ts + 60 * 10 * n + 60
    us, vs, ds, ws = [], [], [], []
    for a in range(n):
        for b in range(n):
            if np.isfinite(W[a, b]):
                deps = np.arange(0, horizon + 1, 60)
                us.append(np.full(len(deps), a)); vs.append(np.full(len(deps), b))
                ds.append(deps); ws.append(np.full(len(deps), int(W[a, b])))
    u, v, d, w = (np.concatenate(x).astype(np.uint32) for x in (us, vs, ds, ws))
    rows, cols = np.nonzero(np.isfinite(W))
    G = csr_matrix((W[rows, cols], (rows, cols)), shape=(n, n))
    for s in range(0, n, 3):
        dist = dijkstra(G, directed=True, indices=s)
        want = [ts + int(x) if np.isfinite(x) else INF for x in dist]
        assert oracle.csa(n, u, v, d, w, s, ts).tolist() == want


# --------------------------------------------------------------------- closed form
def test_chain_closed_form():
    """Chain 0->1->...->k, edge i has one AP (f_i, p_i, c_i terms) and
    duration l_i: e[i+1] = next_i(e[i]) + l_i, next(x) = f if x <= f,
    f + ceil((x-f)/p)*p if x <= last, else unreachable."""
    rng = np.random.default_rng(11)
    for _ in range(50):
        k = int(rng.integers(1, 12))
        us, vs, ds, ls, aps = [], [], [], [], []
        for i in range(k):
            f, p, c, lam = int(rng.integers(0, 4000)), int(rng.integers(1, 900)), int(rng.integers(1, 30)), int(rng.integers(0, 700))
            aps.append((f, p, c, lam))
            for j in range(c):
                us.append(i); vs.append(i + 1); ds.append(f + j * p); ls.append(lam)
        ts = int(rng.integers(0, 5000))
        want = [INF] * (k + 1)
        want[0] = ts
        for i, (f, p, c, lam) in enumerate(aps):
            x, last = want[i], f + (c - 1) * p
            if x == INF or x > last:
                break
            nxt = f if x <= f else f + -(-(x - f) // p) * p
            want[i + 1] = nxt + lam
        got = oracle.csa(k + 1, us, vs, ds, ls, 0, ts).tolist()
        assert got == want


# --------------------------------------------------------------------- invariants
def test_invariants_witness_and_monotone():
    rng = np.random.default_rng(3)
    for _ in range(40):
        n, m = int(rng.integers(5, 80)), int(rng.integers(10, 3000))
        u = rng.integers(0, n, m).astype(np.uint32)
        v = rng.integers(0, n, m).astype(np.uint32)
        dep = rng.integers(0, 86400, m).astype(np.uint32)
        dur = rng.choice([0, 60, 120, 300, 1800], m).astype(np.uint32)
        c = oracle.CSA(n, u, v, dep, dur)
        s = int(rng.integers(0, n))
        prev = None
        for ts in sorted(int(x) for x in rng.integers(0, 86400, 6)):
            e, par = c.query(s, ts, with_parent=True)
            assert e[s] == ts
            assert np.all((e >= ts) | (e == INF)) and np.all(e <= INF)
            assert oracle.witness_ok(n, u, v, dep, dur, s, ts, e, par)
            if prev is not None:
                mask = np.arange(n) != s
                assert np.all(prev[mask] <= e[mask])  # t1 <= t2 => e_t1 <= e_t2
            prev = e
        c.close()


def test_witness_ok_rejects_bad_witnesses():
    """Negative pins for oracle.witness_ok: a valid
    parent chain passes; each way a chain can fail to be a time-respecting
    path ending exactly at e[x] is rejected."""
    #            u  v  dep  dur
    conns = [(0, 1, 100, 10),    # 0: e[1] = 110
             (1, 2, 120, 10),    # 1: e[2] = 130
             (2, 3, 140, 10),    # 2: e[3] = 150
             (1, 2, 105, 5),     # 3: arrives 110 at 2 but departs before e[1] = 110
             (0, 4, 100, 100),   # 4: e[4] = 200
             (4, 5, 200, 0),     # 5: e[5] = 200
             (5, 4, 200, 0)]     # 6: 5 -> 4 at the same instant (a cycle with 5)
    a = np.array(conns, dtype=np.uint32)
    u, v, dep, dur = a[:, 0], a[:, 1], a[:, 2], a[:, 3]
    n, s, ts = 6, 0, 100
    e_ok = [100, 110, 130, 150, 200, 200]
    par_ok = [-1, 0, 1, 2, 4, 5]

    def ok(e, par):
        return oracle.witness_ok(n, u, v, dep, dur, s, ts, np.array(e, np.uint32), np.array(par, np.int64))

    assert ok(e_ok, par_ok)
    # the oracle's own parent output is this chain
    e, par = oracle.csa(n, u, v, dep, dur, s, ts, with_parent=True)
    assert e.tolist() == e_ok and ok(e, par)
    bad = {
        "parent into another vertex": (e_ok, [-1, 0, 2, 2, 4, 5]),
        "departure before e[u] (1 -> 2 at 105 < e[1] = 110)": ([100, 110, 110, 150, 200, 200], [-1, 0, 3, 2, 4, 5]),
        "arrival != dep + dur": ([100, 110, 130, 151, 200, 200], par_ok),
        "cycle 4 <-> 5 never reaching s": (e_ok, [-1, 0, 1, 2, 6, 5]),
        "finite e[x] without parent": (e_ok, [-1, 0, 1, -1, 4, 5]),
        "INF vertex with a parent": ([100, 110, 130, INF, 200, 200], par_ok),
        "e[s] != t_s": ([101, 110, 130, 150, 200, 200], par_ok),
    }
    for what, (e, par) in bad.items():
        assert not ok(e, par), what


def test_query_many_equals_single():
    rng = np.random.default_rng(9)
    n, m = 40, 2000
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    dep, dur = rng.integers(0, 86400, m), rng.integers(0, 3000, m)
    c = oracle.CSA(n, u, v, dep, dur)
    src, ts = rng.integers(0, n, 20), rng.integers(0, 86400, 20)
    many = c.query_many(src, ts)
    for i in range(20):
        assert np.array_equal(many[i], c.query(int(src[i]), int(ts[i])))
    with pytest.raises(ValueError):
        c.query(n, 0)
    with pytest.raises(ValueError):
        c.query(0, INF)


# --------------------------------------------------------------------- lookups
def test_alg6_equals_linear_every_bound():
    rng = random.Random(6)
    for _ in range(300):
        aps = []
        for _k in range(rng.randint(1, 4)):
            f, d, c = rng.randint(0, 200), rng.randint(1, 40), rng.randint(1, 8)
            aps.append((f, f + (c - 1) * d, d))
        aps.sort()
        deps = oracle.expand_aps(aps)
        for b in range(0, max(deps) + 3):
            assert oracle.get_connection_from_aps(aps, b) == oracle.get_connection(deps, b)


def test_greedy_cover_roundtrip_and_cluster_lookup_every_bound():
    rng = random.Random(8)
    for it in range(100):
        cs = rng.choice([3600, 1800, 900, 300])
        horizon = rng.choice([86400, 3 * 86400 // 2])
        m = rng.randint(1, 30)
        if it % 3 == 0:  # periodic with jitter: AP-friendly
            start, h = rng.randint(0, 20000), rng.choice([300, 600, 900])
            deps = [start + i * h + (rng.randint(-60, 60) if rng.random() < 0.3 else 0) for i in range(m)]
            deps = [max(0, d) for d in deps]
        else:
            deps = [rng.randint(0, horizon) for _ in range(m)]
        if it % 5 == 0:
            deps += deps[: rng.randint(0, 3)]  # duplicate connections
        cover = oracle.greedy_ap_cover(deps)
        assert sorted(oracle.expand_aps(cover)) == sorted(deps)
        top = max(deps) + 2
        bounds = list(range(0, top, 37)) + [d + o for d in deps for o in (-1, 0, 1)] + [top]
        for b in bounds:
            if b < 0:
                continue
            assert oracle.cluster_ap_lookup(deps, b, cs) == oracle.get_connection(deps, b)
