"""Seeded synthetic public-transport timetables (input generator only).

This module is shared by the oracle side (tests, cpu baseline) and the CUDA
side (bench, parity tests).  It holds NONE of the method's arithmetic: it
only emits raw connections ``(u, v, dep, dur)`` (+ ``trip`` ids and stop
coordinates), in the shape of the paper's city networks.  Recipe (DESIGN.md
"Input recipe"):

* stops uniform in a square with ~400 m mean spacing; proximity graph =
  6 nearest neighbours (scipy cKDTree);
* lines = random non-backtracking simple walks of 10-40 stops over that
  graph, each run in both directions; walks start at not-yet-served stops;
  lines are added until the target number of distinct directed edges
  exists (then short feeder lines serve any stop still unserved);
* segment duration = distance / 8 m/s rounded to 60 s, minimum 60 s (so
  lambda >= 60); a peak variant adds 60 s on 60 % of segments for trips
  starting in 07-09 h or 16-19 h (~1.7 connection types per edge, the
  paper's Table I shape); dwell 0 or 60 s per stop;
* service starts 05-07 h and ends 22-24 h, hour aligned; headway from
  {5,6,10,12,15,20,30,60} min chosen to hit |C|, halved in peak hours when
  the half is still in the set; downstream departures may pass 24:00, so
  more than 24 hour clusters appear (Table I);
* an ``irregular`` fraction of trips is shifted by U[-120, 120] s
  ("mixed periodic/irregular" metro and country configs).

Times are integer seconds.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Optional, Tuple

import numpy as np

HEADWAYS = (300, 360, 600, 720, 900, 1200, 1800, 3600)
PEAK_BANDS = ((7 * 3600, 9 * 3600), (16 * 3600, 19 * 3600))

CONFIGS: Dict[str, dict] = {
    # BASELINE.json configs[0..4]
    "tiny": dict(stops=200, edges=600, conns=20_000, irregular=0.0, seed=1),
    "city": dict(stops=10_000, edges=30_000, conns=2_000_000, irregular=0.0, seed=2),
    "metro": dict(stops=100_000, edges=300_000, conns=30_000_000, irregular=0.3, seed=3),
    "country": dict(stops=1_000_000, edges=3_000_000, conns=300_000_000, irregular=0.3, seed=4),
}

SINGLE_QUERY = (0, 6 * 3600)  # s=0, t_s=06:00 (BASELINE.json configs[0], [1], [3])


@dataclasses.dataclass
class Timetable:
    num_vertices: int
    u: np.ndarray
    v: np.ndarray
    dep: np.ndarray
    dur: np.ndarray
    trip: Optional[np.ndarray] = None
    xy: Optional[np.ndarray] = None
    name: str = ""

    @property
    def num_connections(self) -> int:
        return int(self.u.shape[0])

    def arrays(self) -> Tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
        return self.u, self.v, self.dep, self.dur


def _knn(xy: np.ndarray, k: int):
    from scipy.spatial import cKDTree

    tree = cKDTree(xy)
    _, idx = tree.query(xy, k=k + 1)
    nbr = idx[:, 1:].astype(np.int64)
    n = xy.shape[0]
    # undirected adjacency: union of both kNN directions
    a = np.concatenate([np.repeat(np.arange(n), k), nbr.ravel()])
    b = np.concatenate([nbr.ravel(), np.repeat(np.arange(n), k)])
    key = np.unique(a * n + b)
    a, b = key // n, key % n
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(ptr, a + 1, 1)
    ptr = np.cumsum(ptr)
    return ptr, b


def _walk(rng, ptr, adj, start, length, n):
    line = [start]
    seen = {start}
    prev = -1
    cur = start
    for _ in range(length - 1):
        nb = adj[ptr[cur]:ptr[cur + 1]]
        cand = [int(x) for x in nb if x != prev and int(x) not in seen]
        if not cand:
            break
        nxt = cand[int(rng.integers(len(cand)))]
        line.append(nxt)
        seen.add(nxt)
        prev, cur = cur, nxt
    return line


def _lines(rng, xy, n_edges):
    n = xy.shape[0]
    ptr, adj = _knn(xy, 6)
    edges = set()
    served = np.zeros(n, dtype=bool)
    unserved = list(rng.permutation(n))
    lines = []
    cap = int(n_edges * 1.08) + 8
    while len(edges) < n_edges or (unserved and len(edges) < cap):
        while unserved and served[unserved[-1]]:
            unserved.pop()
        if not unserved and len(edges) >= n_edges:
            break
        if len(edges) < n_edges:
            start = int(unserved[-1]) if unserved else int(rng.integers(n))
            length = int(rng.integers(10, 41))
        else:  # feeder line from a still-unserved stop
            start = int(unserved[-1])
            length = 2
        line = _walk(rng, ptr, adj, start, length, n)
        if len(line) < 2:
            served[start] = True
            continue
        lines.append(np.array(line, dtype=np.int64))
        served[line] = True
        for a, b in zip(line[:-1], line[1:]):
            edges.add(a * n + b)
            edges.add(b * n + a)
    return lines


def _round60(x):
    return np.maximum(60, np.rint(x / 60.0).astype(np.int64) * 60)


def _in_peak(t):
    m = np.zeros(t.shape, dtype=bool)
    for a, b in PEAK_BANDS:
        m |= (t >= a) & (t < b)
    return m


def generate(name: str = "tiny", **override) -> Timetable:
    """Generate one of the BASELINE configs (``tiny``, ``city``, ``metro``,
    ``country``) or a custom one via keyword overrides
    (stops, edges, conns, irregular, seed)."""
    p = dict(CONFIGS.get(name, CONFIGS["tiny"]))
    p.update(override)
    n, n_edges, n_conns = int(p["stops"]), int(p["edges"]), int(p["conns"])
    rng = np.random.default_rng(int(p["seed"]))
    side = 400.0 * np.sqrt(n)
    xy = rng.uniform(0.0, side, size=(n, 2))
    lines = _lines(rng, xy, n_edges)

    # line directions (both) with per-segment durations and dwell
    dirs = []
    for ln in lines:
        for seq in (ln, ln[::-1]):
            d = np.hypot(*(xy[seq[1:]] - xy[seq[:-1]]).T)
            base = _round60(d / 8.0)
            peak = base + 60 * (rng.random(base.shape[0]) < 0.6)
            dwell = 60 * rng.integers(0, 2, size=seq.shape[0])
            dwell[0] = 0
            dirs.append((seq, base, peak, dwell))
    total_seg = sum(len(s) - 1 for s, *_ in dirs)
    trips_needed = max(1.0, n_conns / max(1, total_seg))
    # expected trips per direction for each headway (mean span 17 h, 5 peak
    # hours at double rate when the half headway is in the set)
    exp_trips = sorted(((61200.0 / h + 1.0 + (18000.0 / h if (h // 2) in HEADWAYS and h % 2 == 0 else 0.0)), h)
                       for h in HEADWAYS)

    U, V, D, L, T = [], [], [], [], []
    trip_id = 0
    for seq, base, peak, dwell in dirs:
        # pick between the two headways bracketing the target (mixture hits the mean)
        if trips_needed <= exp_trips[0][0]:
            h = exp_trips[0][1]
        elif trips_needed >= exp_trips[-1][0]:
            h = exp_trips[-1][1]
        else:
            j = next(i for i in range(len(exp_trips)) if exp_trips[i][0] >= trips_needed)
            (t_lo, h_lo), (t_hi, h_hi) = exp_trips[j - 1], exp_trips[j]
            w = (trips_needed - t_lo) / (t_hi - t_lo)
            h = h_hi if rng.random() < w else h_lo
        s0 = 3600 * int(rng.integers(5, 8))
        s1 = 3600 * int(rng.integers(22, 25))
        starts = np.arange(s0, s1 + 1, h, dtype=np.int64)
        if (h // 2) in HEADWAYS and h % 2 == 0:
            extra = starts + h // 2
            extra = extra[_in_peak(extra) & (extra <= s1)]
            starts = np.sort(np.concatenate([starts, extra]))
        nt = starts.shape[0]
        irr = rng.random(nt) < float(p["irregular"])
        jit = rng.integers(-120, 121, size=nt)
        starts = np.maximum(0, starts + np.where(irr, jit, 0))
        is_peak = _in_peak(starts)
        k = seq.shape[0] - 1
        # departure offsets along the line for the two duration variants
        off_b = np.concatenate([[0], np.cumsum(base + dwell[1:])[:-1]])
        off_p = np.concatenate([[0], np.cumsum(peak + dwell[1:])[:-1]])
        off = np.where(is_peak[:, None], off_p[None, :], off_b[None, :])
        dur = np.where(is_peak[:, None], peak[None, :], base[None, :])
        dep = starts[:, None] + off
        U.append(np.broadcast_to(seq[:-1], (nt, k)).ravel())
        V.append(np.broadcast_to(seq[1:], (nt, k)).ravel())
        D.append(dep.ravel())
        L.append(dur.ravel())
        T.append(np.repeat(np.arange(trip_id, trip_id + nt), k))
        trip_id += nt

    def cat(parts):
        return np.ascontiguousarray(np.concatenate(parts).astype(np.uint32))

    return Timetable(n, cat(U), cat(V), cat(D), cat(L), cat(T), xy.astype(np.float32), name)


def queries(tt: Timetable, sources: int = 1000, times: int = 10, seed: int = 7):
    """Paper protocol: random sources x uniformly random
    departure times in [0, 86400); returns (src, t_s) uint32 arrays of length
    sources*times, source-major."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, tt.num_vertices, size=sources)
    ts = rng.integers(0, 86400, size=(sources, times))
    return (np.repeat(src, times).astype(np.uint32), ts.ravel().astype(np.uint32))


def random_small(seed: int, nmax: int = 50, cmax: int = 2000, zero_dur: bool = True,
                 multi_day: bool = True) -> Timetable:
    """Small adversarial instances for parity sweeps: lambda = 0, duplicate
    connections, self-loops, multi-day departures, isolated vertices."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, nmax + 1))
    m = int(rng.integers(0, cmax + 1))
    horizon = int(rng.choice([86400, 2 * 86400])) if multi_day else 86400
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    mode = int(rng.integers(0, 3))
    if mode == 0:  # periodic-ish
        dep = (rng.integers(0, horizon // 600, m) * 600 + rng.choice([0, 0, 0, 7, 300], m))
    elif mode == 1:
        dep = rng.integers(0, horizon, m)
    else:  # few distinct times -> many ties
        dep = rng.choice(rng.integers(0, horizon, 16), m)
    durs = [0, 1, 60, 120, 300, 900, 3600] if zero_dur else [1, 60, 120, 300, 900, 3600]
    dur = rng.choice(durs, m)
    if m > 4:
        k = int(rng.integers(0, max(1, m // 10)))
        idx = rng.integers(0, m, k)
        u, v, dep, dur = (np.concatenate([a, a[idx]]) for a in (u, v, dep, dur))
    a = lambda x: np.ascontiguousarray(np.asarray(x, dtype=np.uint32))
    return Timetable(n, a(u), a(v), a(dep), a(dur), None, None, f"random_small[{seed}]")


def stats(tt: Timetable) -> dict:
    """Shape statistics (for DESIGN.md / bench reporting)."""
    n = tt.num_vertices
    key_e = tt.u.astype(np.uint64) * np.uint64(n) + tt.v.astype(np.uint64)
    ne = int(np.unique(key_e).shape[0])
    key_t = np.stack([tt.u, tt.v, tt.dur], axis=1)
    nt = int(np.unique(key_t, axis=0).shape[0]) if tt.num_connections < 5_000_000 else -1
    served = np.zeros(n, dtype=bool)
    served[tt.u] = True
    served[tt.v] = True
    return dict(stops=n, edges=ne, connections=tt.num_connections, types=nt,
                served=int(served.sum()), max_dep=int(tt.dep.max()) if tt.num_connections else 0,
                min_dur=int(tt.dur.min()) if tt.num_connections else 0)
