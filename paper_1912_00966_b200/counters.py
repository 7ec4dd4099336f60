"""Algorithmic-byte accounting of the batched kernel.

Runs the instrumented variant of k_query_cta (EAT_BUILD_COUNTERS) on the
same queries and converts its work counters to the bytes the method must
move per launch:
    8 B per active-vertex visit (type_ptr pair)
  + 32 B per connection-type record read (one sector)
  + 32 B per cluster record read (Cluster-AP lookup, one sector)
  + 4 B per out-of-line AP item read
  + 8 B per query (s, t_s) + 4*|V| B per query (output row write).
e[] and the frontier bitmaps live in shared memory and move no L2/HBM bytes.
"""
from __future__ import annotations

import numpy as np


def bytes_from_counts(c: dict, nq: int, n: int) -> int:
    return int(8 * c["vertex_visits"] + 32 * c["type_evals"] + 32 * c["cluster_reads"]
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
    keys = ("vertex_visits", "type_evals", "cluster_reads", "spill_items_read", "improvements", "sweeps_total")
    c = {k: int(st[k]) for k in keys}
    nq = int(d_src.numel())
    c["algorithmic_bytes"] = bytes_from_counts(c, nq, tt.num_vertices)
    c["per_query"] = {k: c[k] / nq for k in keys}
    return c
