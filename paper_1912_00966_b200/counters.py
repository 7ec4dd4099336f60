"""Algorithmic-byte accounting of the batched kernel (SURVEY
§8(d)).

Runs the instrumented variant of k_query_cta (EAT_BUILD_COUNTERS) on the
same queries and converts its work counters into the bytes the METHOD must
move per launch -- SURVEY §8(d)'s per-unit figures, independent of how our
layout packs them:

    per active source (vertex visit)    12 B  (e[u] + row_ptr pair)
    per edge evaluation                  8 B  (edge record) + 4 B (e[v] read-modify-write)
    per connection-type header read     16 B  ({v, lambda, first, last})
    per hour-cluster slot read          12 B + 8 B per AP run + 4 B per single departure it holds
    per next-cluster fallback            4 B
    per query                            8 B in (s, t_s) + 4*|V| B out (the e[] row)

Beside it, the bytes our device layout actually requests (``layout_bytes``):
8 B type_ptr pair per visit, 16 B header + 4 B cluster base per type, one
32-byte cluster record per slot, 4 B per spilled item, the query I/O.
e[] and the frontier bitmaps live in shared memory (no L2/HBM bytes).
"""
from __future__ import annotations

import numpy as np

KEYS = ("vertex_visits", "type_evals", "cluster_reads", "spill_items_read", "improvements", "sweeps_total",
        "edge_evals", "cluster_runs", "cluster_singles", "fallbacks", "select_bits")


def algorithmic_bytes(c: dict, nq: int, n: int) -> int:
    """SURVEY §8(d) bytes of one launch from its work counters."""
    return int(12 * c["vertex_visits"] + (8 + 4) * c["edge_evals"] + 16 * c["type_evals"]
               + 12 * c["cluster_reads"] + 8 * c["cluster_runs"] + 4 * c["cluster_singles"] + 4 * c["fallbacks"]
               + 8 * nq + 4 * n * nq)


def layout_bytes(c: dict, nq: int, n: int) -> int:
    """Bytes the packed device layout requests for the same work."""
    return int(8 * c["vertex_visits"] + (16 + 4) * c["type_evals"] + 32 * c["cluster_reads"]
               + 4 * c["spill_items_read"] + 8 * nq + 4 * n * nq)


def count_batch(tt, src, ts, device: int, **engine_kw) -> dict:
    import torch

    from .engine import Engine

    eng = Engine.from_timetable(tt, device=device, counters=True, **engine_kw)
    d_src = torch.tensor(np.asarray(src, np.uint32).astype(np.int32), device=device)
    d_ts = torch.tensor(np.asarray(ts, np.uint32).astype(np.int32), device=device)
    out = torch.empty((d_src.numel(), tt.num_vertices), dtype=torch.int32, device=device)
    eng.query_many_device(d_src, d_ts, out)
    torch.cuda.synchronize(device)
    st = eng.stats()
    eng.close()
    c = {k: int(st[k]) for k in KEYS}
    nq = int(d_src.numel())
    c["algorithmic_bytes"] = algorithmic_bytes(c, nq, tt.num_vertices)
    c["layout_bytes"] = layout_bytes(c, nq, tt.num_vertices)
    c["per_query"] = {k: c[k] / nq for k in KEYS}
    return c
