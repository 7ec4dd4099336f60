"""oracle/reference.py -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Plain, slow, obviously-correct CPU implementations of what the EAT hot path
computes, written from arXiv 1912.00966.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl
reference`` legs may import this module.  It shares no code with the CUDA
path (``paper_1912_00966_b200``) and never imports it.

Functions and the passage each follows:

* :func:`csa` / :class:`CSA`       -- Algorithm 1 Connection-Scan, PAPER.md:96-118,
  via the plain C in ``oracle/csa.c`` (reading R1: lambda=0 closure per
  equal-departure group; reading R2: uint32 seconds, INF = 0x7FFFFFFF).
* :func:`brute_force_eat`         -- the EAT definition itself, PAPER.md:57-59, 90:
  enumerate every time-respecting connection sequence from ``s``.
* :func:`td_dijkstra`             -- the label-setting variant named in PAPER.md:64,
  677 (prefix optimality of earliest-arrival paths), edge arrival function
  ``f_uv(t) = min{dep + lambda : dep >= t}``.
* :func:`get_connection`          -- getConnection of Sec. II-B, PAPER.md:226:
  ``t_c = min{t | (u,v,t,lambda) in C_uvl and t >= e[u]}`` by linear search.
* :func:`greedy_ap_cover`         -- the arithmetic-progression technique,
  PAPER.md:142 (smallest uncovered ``a``, longest AP from ``a`` covering the
  most uncovered numbers, repeat), tuples ``(first, last, difference)``.
* :func:`get_connection_from_aps` -- Algorithm 6, literally.
* :func:`cluster_ap_lookup`       -- the Cluster-AP hybrid rule
  (k = e[u]/3600, Alg. 6 on T[k]; if cluster k yields nothing, the first
  connection of the next non-empty cluster -- reading R4).
* :func:`witness_ok`              -- invariant check: a parent chain is a real
  time-respecting path.

Pins (tests/test_oracle_*.py, all ``-m "not gpu"``): paper-printed values
(SPEC examples), brute force on tiny inputs, the
time-dependent Dijkstra, a static shortest-path reduction through
``scipy.sparse.csgraph.dijkstra``, closed-form chains, invariants.
"""
from __future__ import annotations

import ctypes
import heapq
import os
import subprocess
from typing import Iterable, List, Optional, Sequence, Tuple

import numpy as np

INF = 0x7FFFFFFF  # reading R2: "maximum of the chosen width" under int32

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csa.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build_oracle(force: bool = False) -> str:
    """Compile oracle/csa.c with gcc -O3 into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build_oracle())
        P = ctypes.c_void_p
        u32p = ctypes.POINTER(ctypes.c_uint32)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.oracle_prepare.restype = P
        lib.oracle_prepare.argtypes = [ctypes.c_uint32, ctypes.c_uint64, u32p, u32p, u32p, u32p]
        lib.oracle_free.restype = None
        lib.oracle_free.argtypes = [P]
        lib.oracle_csa_query.restype = ctypes.c_int
        lib.oracle_csa_query.argtypes = [P, ctypes.c_uint32, ctypes.c_uint32, u32p, i64p]
        lib.oracle_csa_many.restype = ctypes.c_int
        lib.oracle_csa_many.argtypes = [P, u32p, u32p, ctypes.c_uint64, u32p]
        _lib = lib
    return _lib


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _ptr(a: np.ndarray, t=ctypes.c_uint32):
    return a.ctypes.data_as(ctypes.POINTER(t))


class CSA:
    """Algorithm 1 on a prepared, departure-sorted copy of
    the raw connection list.  ``query`` / ``query_many`` return uint32 arrays."""

    def __init__(self, n: int, u, v, dep, dur):
        self._lib = _load()
        self.n = int(n)
        self._arrays = [_u32(u), _u32(v), _u32(dep), _u32(dur)]
        m = len(self._arrays[0])
        for a in self._arrays:
            if len(a) != m:
                raise ValueError("u, v, dep, dur must have equal length")
        self.m = m
        self._h = self._lib.oracle_prepare(self.n, m, *[_ptr(a) for a in self._arrays])
        if not self._h:
            raise MemoryError("oracle_prepare failed")

    def close(self):
        if getattr(self, "_h", None):
            self._lib.oracle_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self, s: int, t_s: int, with_parent: bool = False):
        e = np.empty(self.n, dtype=np.uint32)
        par = np.empty(self.n, dtype=np.int64) if with_parent else None
        rc = self._lib.oracle_csa_query(self._h, int(s), int(t_s), _ptr(e),
                                        _ptr(par, ctypes.c_int64) if with_parent else None)
        if rc != 0:
            raise ValueError(f"invalid query (s={s}, t_s={t_s})")
        return (e, par) if with_parent else e

    def query_many(self, sources, times) -> np.ndarray:
        src, ts = _u32(sources), _u32(times)
        out = np.empty((len(src), self.n), dtype=np.uint32)
        rc = self._lib.oracle_csa_many(self._h, _ptr(src), _ptr(ts), len(src), _ptr(out))
        if rc != 0:
            raise ValueError("invalid query in batch")
        return out


def csa(n, u, v, dep, dur, s, t_s, with_parent=False):
    """One-shot Algorithm 1."""
    c = CSA(n, u, v, dep, dur)
    try:
        return c.query(s, t_s, with_parent)
    finally:
        c.close()


# ---------------------------------------------------------------------------
# Pure-Python pins (small inputs only)
# ---------------------------------------------------------------------------

Conn = Tuple[int, int, int, int]  # (u, v, t, lambda)


def brute_force_eat(n: int, conns: Sequence[Conn], s: int, t_s: int) -> List[int]:
    """The EAT definition by exhaustive enumeration of
    every time-respecting sequence of distinct connections leaving ``s`` at or
    after ``t_s``.  A path never needs to reuse a connection (reusing one at
    the same instant cannot lower any arrival), so distinct-connection
    sequences suffice.  Exponential: keep |C| <= ~10."""
    e = [INF] * n
    e[s] = t_s
    used = [False] * len(conns)

    def dfs(at: int, now: int):
        for i, (a, b, t, lam) in enumerate(conns):
            if used[i] or a != at or t < now:
                continue
            arr = t + lam
            if arr < e[b]:
                e[b] = arr
            used[i] = True
            dfs(b, arr)
            used[i] = False

    dfs(s, t_s)
    return e


def td_dijkstra(n: int, conns: Sequence[Conn], s: int, t_s: int) -> List[int]:
    """Time-dependent Dijkstra.  Edge (u,v) has arrival
    function f(t) = min{dep + lambda : (u,v,dep,lambda) in C, dep >= t}, which
    is non-decreasing in t (FIFO), so label setting is exact."""
    out = {}
    for (a, b, t, lam) in conns:
        out.setdefault(a, {}).setdefault(b, []).append((t, t + lam))
    e = [INF] * n
    e[s] = t_s
    done = [False] * n
    pq = [(t_s, s)]
    while pq:
        tu, u = heapq.heappop(pq)
        if done[u] or tu != e[u]:
            continue
        done[u] = True
        for v, lst in out.get(u, {}).items():
            best = INF
            for (t, arr) in lst:
                if t >= tu and arr < best:
                    best = arr
            if best < e[v]:
                e[v] = best
                heapq.heappush(pq, (best, v))
    return e


def get_connection(departures: Iterable[int], bound: int) -> Optional[int]:
    """getConnection: min{t : t >= e[u]} by linear search; None if empty."""
    best = None
    for t in departures:
        if t >= bound and (best is None or t < best):
            best = t
    return best


def greedy_ap_cover(values: Sequence[int]) -> List[Tuple[int, int, int]]:
    """AP technique: repeatedly take the smallest uncovered
    number a, find the longest arithmetic progression starting at a that
    covers the most uncovered numbers, emit (first, last, difference).
    Terms are drawn from the uncovered set (tuples are disjoint, so the
    expansion is exactly the input, "without any additional
    departure times").  Ties: smallest difference.  A single
    remaining number becomes (a, a, 1).  Duplicates are
    separate occurrences; each occurrence is covered once."""
    remaining = sorted(int(x) for x in values)
    out = []
    while remaining:
        a = remaining[0]
        pool = {}
        for x in remaining[1:]:
            pool[x] = pool.get(x, 0) + 1
        best_d, best_len = 1, 1
        for d in sorted({x - a for x in remaining[1:] if x > a}):
            k, x = 1, a + d
            while pool.get(x, 0) > 0:
                k += 1
                x += d
            if k > best_len:
                best_d, best_len = d, k
        terms = [a + i * best_d for i in range(best_len)]
        out.append((a, terms[-1], best_d))
        for t in terms:
            remaining.remove(t)
    return out


def expand_aps(aps: Iterable[Tuple[int, int, int]]) -> List[int]:
    """Expansion of AP tuples (first, last, difference), PAPER.md:259:
    t = startTime + i * difference, i in {0..k}, k = (end - start) / difference."""
    out = []
    for (f, l, d) in aps:
        k = 0 if l == f else (l - f) // d
        out.extend(f + i * d for i in range(k + 1))
    return out


def get_connection_from_aps(aps: Iterable[Tuple[int, int, int]], e_u: int) -> Optional[int]:
    """Algorithm 6 getConnectionFromAPs, line by line.
    Returns t_c, or None when it stays infinite."""
    t_c = INF
    for (start, end, diff) in aps:
        if start < e_u <= end:                       # line 3
            i = -(-(e_u - start) // diff)            # line 4: ceil((e[u]-start)/diff)
            t_c = min(t_c, start + i * diff)         # line 5
        if e_u <= start:                             # line 7
            t_c = min(t_c, start)                    # line 8
    return None if t_c == INF else t_c


def cluster_ap_lookup(departures: Sequence[int], bound: int, cluster_seconds: int = 3600) -> Optional[int]:
    """Cluster-AP hybrid rule, step by step:
    1. partition the type's departures into clusters C[i] by
       i = floor(t / cluster_seconds) ("[i:00:00, i:59:59]");
    2. cover each cluster with AP tuples T[i];
    3. k = e[u] / cluster_seconds; t_c = Alg. 6 on T[k];
    4. if cluster k yields no connection, "the first connection from the next
       non-empty part", read as: cluster k empty OR no departure >= e[u]
       in it (reading R4) -> the smallest departure of the next non-empty
       cluster; none if there is none."""
    clusters = {}
    for t in departures:
        clusters.setdefault(t // cluster_seconds, []).append(t)
    T = {i: greedy_ap_cover(ts) for i, ts in clusters.items()}
    k = bound // cluster_seconds
    if k in T:
        t_c = get_connection_from_aps(T[k], bound)
        if t_c is not None:
            return t_c
    later = [i for i in T if i > k]
    if not later:
        return None
    j = min(later)
    return min(f for (f, _l, _d) in T[j])


def witness_ok(n, u, v, dep, dur, s, t_s, e, parent) -> bool:
    """Each finite e[x] (x != s) is the arrival of parent connection p, whose
    own source has e[u_p] <= dep_p, recursively back to s: a time-respecting
    path ending exactly at e[x]."""
    for x in range(n):
        if x == s:
            if e[x] != t_s:
                return False
            continue
        if e[x] == INF:
            if parent[x] != -1:
                return False
            continue
        y, arrival, steps = x, int(e[x]), 0
        while y != s:
            p = int(parent[y])
            if p < 0:
                return False
            if int(v[p]) != y or int(dep[p]) + int(dur[p]) != int(e[y]):
                return False
            uu = int(u[p])
            if int(e[uu]) > int(dep[p]):
                return False
            y = uu
            steps += 1
            if steps > n + 1:
                return False
        if arrival != int(e[x]):
            return False
    return True
