#!/usr/bin/env python
"""compute-sanitizer driver.

Runs ONE case of the hot path on the tiny config (small enough for the
sanitizer's instrumentation) and checks its rows against the oracle, so a
sanitizer run also proves the instrumented kernels still compute the right
arrival times.  The shell loop in tools/sanitize.sh runs every case under
memcheck, racecheck and synccheck.

  python tools/sanitize.py CASE      (CASE in CASES, or "list")
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: parity of the sanitized run)
import synth  # noqa: E402
from paper_1912_00966_b200 import Engine  # noqa: E402

# case -> (kernel under test, engine kwargs, what to run)
CASES = {
    "cta_single": ("k_query_cta (1024 threads, one query)", dict(kernel="cta"), "single"),
    "cta_batch16": ("k_query_cta (uint16 e[] pass + uint32 recompute)", dict(arr_bits=16), "batch"),
    "cta_batch32": ("k_query_cta (uint32 e[])", dict(arr_bits=32), "batch"),
    "cta_targets": ("k_query_cta<TGT> (goal-directed)", dict(), "targets"),
    "cta_batch384": ("k_query_cta (384 threads, uint32 e[]: the batch default until r02 session 3)", dict(cta_threads=384, arr_bits=32),
                     "batch"),
    "cluster16": ("k_query_cluster<2> (16 CTAs, DSMEM e[], staged index)", dict(kernel="cluster", cluster_ctas=16),
                  "single"),
    "cluster2": ("k_query_cluster (2 CTAs)", dict(kernel="cluster", cluster_ctas=2, window=600), "single"),
    "cluster_sync": ("k_query_cluster<.., sync> (4 CTAs, cluster barrier per sweep)",
                     dict(kernel="cluster", cluster_ctas=4, cluster_sync=True), "single"),
    "grid_async": ("k_query_gasync (barrier-free grid, per-CTA counters)", dict(kernel="grid_async"), "single"),
    "grid_frontier": ("k_query_grid<32, frontier>", dict(kernel="frontier"), "single"),
    "grid_flat": ("k_query_grid<32, flat> (subwarp 64)", dict(kernel="frontier", subwarp=64), "single"),
    "grid_full": ("k_query_grid<1, full sweep>", dict(kernel="full_sweep"), "single"),
    "grid_bitmap": ("k_query_grid<32, bitmap>", dict(kernel="bitmap"), "single"),
    "groups": ("k_query_groups (CTA groups, invalid rows)", dict(kernel="frontier"), "batch_invalid"),
    "async": ("k_query_async", dict(kernel="async"), "single"),
    "part_loopback": ("k_part_round (loopback P=2, device min-merge)",
                      dict(mode="edge_partitioned", part_rank=0, part_count=2), "single"),
    "part_rounds": ("k_part_round (loopback P=2, one local sweep per round)",
                    dict(mode="edge_partitioned", part_rank=0, part_count=2, local_sweeps=1), "single"),
    "peer_loopback": ("k_peer_query (loopback P=2)",
                      dict(mode="edge_partitioned", part_rank=0, part_count=2, exchange="peer"), "single"),
}


def run(case: str) -> None:
    import torch

    what, kw, kind = CASES[case]
    tt = synth.generate("tiny")
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    try:
        eng = Engine.from_timetable(tt, **kw)
    except TypeError:  # option not in this build of the binding
        print(f"SKIP {case}: {kw} unsupported")
        return
    if kind == "single":
        for s, t_s in [synth.SINGLE_QUERY, (17, 40000)]:
            assert np.array_equal(eng.query(s, t_s), csa.query(s, t_s)), f"{case}: row differs from the oracle"
    elif kind in ("batch", "batch_invalid"):
        src, ts = synth.queries(tt, 12, 2)
        want = csa.query_many(src, ts)
        assert np.array_equal(eng.query_many(src, ts), want), f"{case}: rows differ"
        if kind == "batch_invalid":
            bad = src.astype(np.int64).copy()
            bad[::3] = tt.num_vertices + 1  # invalid queries interleaved with valid ones
            d_src = torch.tensor(bad.astype(np.int32), device="cuda")
            d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
            out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
            eng.query_many_device(d_src, d_ts, out)
            got = out.cpu().numpy().astype(np.uint32)
            keep = np.arange(src.size) % 3 != 0
            assert (got[~keep] == oracle.INF).all() and np.array_equal(got[keep], want[keep]), f"{case}: device rows"
    elif kind == "targets":
        src, ts = synth.queries(tt, 12, 2)
        dst = (np.arange(src.size) * 37 % tt.num_vertices).astype(np.uint32)
        want = csa.query_many(src, ts)[np.arange(src.size), dst]
        assert np.array_equal(eng.query_targets(src, ts, dst), want), f"{case}: targets differ"
    torch.cuda.synchronize()
    print(f"OK {case}: {what}")


if __name__ == "__main__":
    if sys.argv[1] == "list":
        print(" ".join(CASES))
    else:
        run(sys.argv[1])
