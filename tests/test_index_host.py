"""CPU checks of the host compressor inside libeat.so (eat_build with
EAT_BUILD_HOST_ONLY) and of the C ABI surface.  No GPU needed.

The packed index is decoded HERE, in test code, from the layout documented in
include/eat.h, and compared with the raw connection multiset (north star:
"the compressed timetable decodes back to exactly the original connection
multiset") and, through a test-side lookup over the decoded layout, with
oracle.get_connection for every bound.
"""
import ctypes
import json
import os
import re
import subprocess
from collections import Counter

import numpy as np
import pytest

import oracle
import synth
from oracle import INF

pkg = pytest.importorskip("paper_1912_00966_b200")
from paper_1912_00966_b200 import Engine, EatError, _lib  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _decode(ex, cs):
    """-> list of (u_int, v_int, lam, dep) from the exported arrays, plus per-type departure lists."""
    trec, crec, pool, tptr = ex["type_rec"], ex["crec"], ex["pool"], ex["type_ptr"]
    out, per_type = [], []
    for t in range(trec.shape[0]):
        v, lam, first, last, cbase, cfirst, u, _ = (int(x) for x in trec[t])
        assert tptr[u] <= t < tptr[u + 1], "type stored under the wrong source vertex"
        deps = []
        # compact layout: c_first = first // cs, records crec_base + (k - c_first);
        # dense directory (the paper's CL[y*i + j]): c_first = 0, crec_base = t * y
        assert cfirst in (first // cs, 0)
        for k in range(first // cs, last // cs + 1):
            r = crec[cbase + k - cfirst]
            if r[1] == 0xFFFFFFFE:
                items = [int(x) for x in pool[r[2]:r[2] + r[3]]]
            else:
                items = [int(x) for x in r[1:] if x != 0xFFFFFFFF]
            for it in items:
                off, stride, cnt = it & 0xFFF, (it >> 12) & 0xFFF, (it >> 24) + 1
                assert off + (cnt - 1) * stride < cs, "item leaves its cluster"
                deps.extend(k * cs + off + i * stride for i in range(cnt))
        deps.sort()
        assert deps[0] == first and deps[-1] == last
        per_type.append((u, v, lam, deps))
        out.extend((u, v, lam, d) for d in deps)
    return out, per_type


def _lookup_on_layout(ex, cs, t, b):
    """Test-side reading of the layout: Cluster-AP rule."""
    v, lam, first, last, cbase, cfirst, u, _ = (int(x) for x in ex["type_rec"][t])
    if b > last:
        return None
    if b <= first:
        return first
    k = b // cs
    r = ex["crec"][cbase + k - cfirst]
    items = [int(x) for x in (ex["pool"][r[2]:r[2] + r[3]] if r[1] == 0xFFFFFFFE else r[1:]) if x != 0xFFFFFFFF]
    best = None
    for it in items:
        off, stride, cnt = it & 0xFFF, (it >> 12) & 0xFFF, (it >> 24) + 1
        terms = [k * cs + off + i * stride for i in range(cnt)]
        hit = [x for x in terms if x >= b]
        if hit and (best is None or hit[0] < best):
            best = hit[0]
    if best is not None:
        return best
    return None if r[0] == INF else int(r[0])


def _check_roundtrip(tt, cs=3600, renumber="auto", cluster_dir="auto"):
    eng = Engine.from_timetable(tt, host_only=True, cluster_seconds=cs, renumber=renumber, cluster_dir=cluster_dir)
    ex = eng.export()
    perm = ex["perm"].astype(np.int64)
    assert sorted(perm.tolist()) == list(range(tt.num_vertices))
    dec, per_type = _decode(ex, cs)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    got = Counter((int(inv[u]), int(inv[v]), lam, d) for (u, v, lam, d) in dec)
    want = Counter(zip(tt.u.tolist(), tt.v.tolist(), tt.dur.tolist(), tt.dep.tolist()))
    assert got == want
    keys = [(u, v, lam) for (u, v, lam, _d) in per_type]
    assert len(keys) == len(set(keys)), "connection types must be unique per (u, v, lambda)"
    st = eng.stats()
    assert st["num_types"] == len(per_type)
    assert st["num_connections"] == tt.num_connections
    return eng, ex, per_type


def test_abi_symbols_exported():
    lib = _lib.lib()
    for name in _lib.EXPORTED:
        assert hasattr(lib, name), name
    hdr = open(os.path.join(ROOT, "include", "eat.h")).read()
    declared = set(re.findall(r"^\s*(?:eat_status|void|const char \*|uint32_t)\s*\**\s*(eat_\w+)\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED)
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", nm, re.M), f"{name} not exported by libeat.so"
    assert _lib.eat_abi_version() == 4


def test_roundtrip_tiny_and_lookup_every_bound():
    tt = synth.generate("tiny")
    eng, ex, per_type = _check_roundtrip(tt)
    rng = np.random.default_rng(0)
    for t in rng.choice(len(per_type), 60, replace=False):
        deps = per_type[t][3]
        bounds = sorted(set([0, deps[-1] + 1] + [d + o for d in deps for o in (-1, 0, 1) if d + o >= 0]))
        for b in bounds:
            assert _lookup_on_layout(ex, 3600, int(t), b) == oracle.get_connection(deps, b)


@pytest.mark.parametrize("cs", [3600, 1800, 900, 300, 4096, 60])
def test_roundtrip_random_small_cluster_sizes(cs):
    for seed in range(12 if cs >= 300 else 3):
        tt = synth.random_small(seed)
        if tt.num_connections == 0:
            continue
        eng, ex, per_type = _check_roundtrip(tt, cs=cs, renumber=["none", "bfs", "auto"][seed % 3],
                                             cluster_dir=["auto", "dense", "compact"][seed % 3])
        for t in range(min(len(per_type), 25)):
            deps = per_type[t][3]
            for b in list(range(0, deps[-1] + 2, max(1, cs // 7))) + deps + [d + 1 for d in deps]:
                assert _lookup_on_layout(ex, cs, t, b) == oracle.get_connection(deps, b)


def test_paper_ap_examples_compress_to_one_item():
    """PAPER.md:142 (10,15,...,35) -> (10,35,5) and PAPER.md:259 every 15 min
    8:00-18:00 -> one AP per hour cluster (clusters split the AP)."""
    u = [0] * 6
    tt = synth.Timetable(2, np.array(u, np.uint32), np.ones(6, np.uint32), np.arange(10, 36, 5, dtype=np.uint32),
                         np.full(6, 60, np.uint32))
    ex = Engine.from_timetable(tt, host_only=True, renumber="none", cluster_dir="compact").export()
    items = [int(x) for x in ex["crec"][0][1:] if x != 0xFFFFFFFF]
    assert items == [10 | (5 << 12) | (5 << 24)]  # first 10, difference 5, 6 terms
    deps = np.arange(28800, 64801, 900, dtype=np.uint32)
    tt = synth.Timetable(2, np.zeros(deps.size, np.uint32), np.ones(deps.size, np.uint32), deps,
                         np.full(deps.size, 300, np.uint32))
    ex = Engine.from_timetable(tt, host_only=True, renumber="none", cluster_dir="compact").export()
    for r in ex["crec"][:-1]:  # hours 8..17: 4 departures each -> one AP item
        assert sum(1 for x in r[1:] if x != 0xFFFFFFFF) == 1
    assert ex["crec"].shape[0] == 11  # clusters 8..18


def test_next_nonempty_cluster_fallback_layout():
    """SPEC S:242 / PAPER.md:306: cluster 0 empty -> first of the next non-empty
    cluster; records exist from c_first to c_last with next_min precomputed."""
    deps = np.array([100, 3 * 3600 + 5, 3 * 3600 + 65], np.uint32)
    tt = synth.Timetable(2, np.zeros(3, np.uint32), np.ones(3, np.uint32), deps, np.full(3, 60, np.uint32))
    ex = Engine.from_timetable(tt, host_only=True, renumber="none", cluster_dir="compact").export()
    assert ex["crec"].shape[0] == 4
    assert ex["crec"][0][0] == 3 * 3600 + 5 and ex["crec"][1][0] == 3 * 3600 + 5 and ex["crec"][3][0] == INF
    assert _lookup_on_layout(ex, 3600, 0, 101) == 3 * 3600 + 5
    assert _lookup_on_layout(ex, 3600, 0, 3 * 3600 + 6) == 3 * 3600 + 65


def test_build_errors():
    u = np.array([0, 5], np.uint32)
    with pytest.raises(EatError) as e:
        Engine(3, u, np.array([1, 1], np.uint32), np.array([0, 0], np.uint32), np.array([1, 1], np.uint32),
               host_only=True)
    assert e.value.status == _lib.EAT_EINVAL
    with pytest.raises(EatError) as e:
        Engine(3, [0], [1], [INF - 5], [10], host_only=True)
    assert e.value.status == _lib.EAT_ERANGE
    with pytest.raises(EatError) as e:
        Engine(0, [], [], [], [], host_only=True)
    assert e.value.status == _lib.EAT_EINVAL
    with pytest.raises(EatError) as e:
        Engine(3, [0], [1], [5], [10], host_only=True, cluster_seconds=5000)
    assert e.value.status == _lib.EAT_EINVAL
    with pytest.raises(EatError) as e:
        Engine(3, [0], [1], [5], [10], host_only=True, subwarp=3)
    assert e.value.status == _lib.EAT_EINVAL
    for bad in (1, 3, 32):  # EAT_KERNEL_CLUSTER sizes: 2, 4, 8 or 16 CTAs
        with pytest.raises(EatError) as e:
            Engine(3, [0], [1], [5], [10], host_only=True, cluster_ctas=bad)
        assert e.value.status == _lib.EAT_EINVAL
    with pytest.raises(EatError) as e:
        Engine(3, [0], [1], [5], [10], host_only=True, cta_threads=300)
    assert e.value.status == _lib.EAT_EINVAL
    eng = Engine(3, [0], [1], [5], [10], host_only=True)
    with pytest.raises(EatError) as e:
        eng.query(0, 0)
    assert e.value.status == _lib.EAT_ESTATE
    _lib.lib().eat_free(None)  # no-op


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(EatError) as e:
        Engine(3, [0], [1], [5], [10])
    assert e.value.status == _lib.EAT_ECUDA


def test_partition_ranges_cover_vertices():
    """Host side of the edge partition: the C++ partition_range slices are
    exercised on the GPU; here the exported type_ptr gives the same cut rule
    (balanced by type count, contiguous internal ranges)."""
    tt = synth.generate("tiny")
    ex = Engine.from_timetable(tt, host_only=True).export()
    tptr = ex["type_ptr"].astype(np.int64)
    T = int(tptr[-1])
    for P in (1, 2, 3, 8):
        cuts = [0] + [int(np.searchsorted(tptr[:-1], T * r // P, side="left")) for r in range(1, P)] + [tt.num_vertices]
        assert cuts == sorted(cuts)
        owned = sum(int(tptr[cuts[r + 1]] - tptr[cuts[r]]) for r in range(P))
        assert owned == T


def _expected_shortcuts(tt, scheme):
    """Test-side statement of PAPER.md:349-354: trips ordered by departure,
    blocks of r connections, one shortcut (v_i, v_{j+1}, t_i, t_j + l_j - t_i)
    per block of >= 2 connections."""
    import math

    out = []
    by_trip = {}
    for i in range(tt.num_connections):
        by_trip.setdefault(int(tt.trip[i]), []).append(i)
    lens = []
    trips = []
    for t, idx in sorted(by_trip.items()):
        idx.sort(key=lambda i: (int(tt.dep[i]), i))
        ok = all(tt.v[a] == tt.u[b] and int(tt.dep[a]) + int(tt.dur[a]) <= int(tt.dep[b]) for a, b in zip(idx, idx[1:]))
        if ok and len(idx) >= 2:
            trips.append(idx)
            lens.append(len(idx))
    hier = scheme >= 1000  # EAT_SUBTRIPS_HIER + r: blocks of r, r^2, ... (ours, not the paper's)
    rg = round(math.sqrt(sum(lens) / len(lens))) if scheme == 2 else (scheme - 1000 if hier else scheme)
    for idx in trips:
        k = len(idx)
        r = round(math.sqrt(k)) if scheme == 1 else rg
        if r < 2:
            continue
        blocks = set()
        size = r
        while True:
            for i in range(0, k, size):
                blocks.add((i, min(k, i + size) - 1))
            if not hier or size >= k:
                break
            size *= r
        for i, j in sorted(blocks):  # a block equal to a smaller level's counts once
            if j > i:
                a, b = idx[i], idx[j]
                out.append((int(tt.u[a]), int(tt.v[b]), int(tt.dur[b]) + int(tt.dep[b]) - int(tt.dep[a]), int(tt.dep[a])))
    return out


@pytest.mark.parametrize("scheme", [1, 2, 4, 1002, 1003])
def test_subtrip_shortcuts_and_invariance(scheme):
    """NEXT-1: the index holds the original connections
    plus exactly the paper's shortcuts, and the oracle's arrival times on the
    enhanced connection set equal those on the original one."""
    tt = synth.generate("tiny")
    eng = Engine.from_timetable(tt, host_only=True, subtrips=scheme)
    ex = eng.export()
    dec, _ = _decode(ex, 3600)
    perm = ex["perm"].astype(np.int64)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    got = Counter((int(inv[u]), int(inv[v]), lam, d) for (u, v, lam, d) in dec)
    want = Counter(zip(tt.u.tolist(), tt.v.tolist(), tt.dur.tolist(), tt.dep.tolist()))
    sc = Counter(_expected_shortcuts(tt, scheme))
    assert got == want + sc
    assert eng.stats()["num_shortcuts"] == sum(sc.values()) > 0
    e = np.array([(u, v, d, lam) for (u, v, lam, d), c in got.items() for _ in range(c)], np.uint32)
    enh = oracle.CSA(tt.num_vertices, e[:, 0], e[:, 1], e[:, 2], e[:, 3])
    base = oracle.CSA(tt.num_vertices, *tt.arrays())
    src, ts = synth.queries(tt, 30, 3)
    assert np.array_equal(enh.query_many(src, ts), base.query_many(src, ts))


def test_subtrips_need_trip_ids():
    tt = synth.generate("tiny")
    with pytest.raises(EatError) as e:
        Engine(tt.num_vertices, tt.u, tt.v, tt.dep, tt.dur, host_only=True, subtrips=1)
    assert e.value.status == _lib.EAT_EINVAL
