#!/usr/bin/env python
"""Parameter sweeps and same-box A/B of libeat builds (replaces round 1's
one-off sweep_* / ab_single / phase_time scripts).

  python tools/sweep.py WORKLOAD GRID [--lib ab/libeat_X.so] [--reps 5]

WORKLOAD  city_batch | metro_batch       -- 10k city / 1,024 metro queries (device API)
          single:CFG[:kernel]            -- s=0 06:00 + 4 seeded queries on CFG (L2 flushed)
GRID      JSON object of Engine keyword lists, e.g. '{"window": [600, 1200], "subtrips": [3]}'
          (every combination is run; '{}' = the defaults)

One JSON line per combination: median device ms (CUDA events), queries/s or
ms per query, sweeps, a checksum of the rows (equal across combinations: the
fixpoint is unique, R12) and, for the batched CTA kernel, the instrumented
work counters per query (counters=True build of the same combination).
Parity of single queries is checked against the oracle.
"""
import argparse
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("workload")
    ap.add_argument("grid", nargs="?", default="{}")
    ap.add_argument("--lib", default=None, help="libeat.so build to load (A/B)")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    from paper_1912_00966_b200 import _lib

    if args.lib:
        _lib.LIB_PATH = os.path.abspath(args.lib)
    import torch

    import synth
    from paper_1912_00966_b200 import Engine

    grid = json.loads(args.grid)
    keys = sorted(grid)
    combos = [dict(zip(keys, vals)) for vals in itertools.product(*(grid[k] for k in keys))] or [{}]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device="cuda")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    wl = args.workload
    if wl in ("city_batch", "metro_batch"):
        tt = synth.generate(wl.split("_")[0])
        src, ts = synth.queries(tt, *((1000, 10) if wl == "city_batch" else (256, 4)))
        d_src = torch.tensor(src.astype(np.int32), device="cuda")
        d_ts = torch.tensor(ts.astype(np.int32), device="cuda")
        out = torch.empty((src.size, tt.num_vertices), dtype=torch.int32, device="cuda")
        for kw in combos:
            kw = dict({"subtrips": 3}, **kw)
            eng = Engine.from_timetable(tt, **kw)
            eng.query_many_device(d_src, d_ts, out)
            ms = []
            for i in range(args.reps):
                flush.fill_(i)
                a.record()
                eng.query_many_device(d_src, d_ts, out)
                b.record()
                b.synchronize()
                ms.append(a.elapsed_time(b))
            rec = {"workload": wl, "lib": os.path.basename(_lib.LIB_PATH), **kw, "batch_ms_med": float(np.median(ms)),
                   "qps": src.size / float(np.median(ms)) * 1e3, "crc": int(out[::97].sum().item()),
                   "cta_grid": eng.stats()["cta_grid"]}
            if eng.stats()["cta_grid"] > 0:
                e2 = Engine.from_timetable(tt, counters=True, **kw)
                e2.query_many_device(d_src, d_ts, out)
                torch.cuda.synchronize()
                st = e2.stats()
                rec["per_query"] = {k: st[k] / src.size for k in (
                    "vertex_visits", "type_evals", "edge_evals", "cluster_reads", "improvements", "sweeps_total",
                    "select_bits")}
                sw = max(1, st["sweeps_total"])
                rec["cycles_per_sweep"] = {"phase": st["select_cycles"] / sw, "select_loop": st["select_loop_cycles"] / sw,
                                           "pair_loop": st["pair_loop_cycles"] / sw}
                e2.close()
            eng.close()
            print(json.dumps(rec), flush=True)
    elif wl.startswith("single:"):
        parts = wl.split(":")
        cfg, kernel = parts[1], (parts[2] if len(parts) > 2 else "auto")
        import oracle

        tt = synth.generate(cfg)
        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        s4, t4 = synth.queries(tt, 4, 1, seed=11)
        qs = [synth.SINGLE_QUERY] + list(zip(s4.tolist(), t4.tolist()))
        want = {q: csa.query(*q) for q in qs}
        o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
        for kw in combos:
            kw = dict({"subtrips": 3, "kernel": kernel}, **kw)
            eng = Engine.from_timetable(tt, **kw)
            res = {}
            for q in qs:
                eng.query_device(*q, o1)
                ms = []
                for i in range(args.reps):
                    flush.fill_(i)
                    a.record()
                    eng.query_device(*q, o1)
                    b.record()
                    b.synchronize()
                    ms.append(a.elapsed_time(b))
                ok = bool(np.array_equal(o1.cpu().numpy().view(np.uint32), want[q]))
                res[f"{q[0]}@{q[1]}"] = {"ms": float(np.median(ms)), "sweeps": eng.stats()["last_sweeps"],
                                         "rounds": eng.stats()["last_rounds"], "parity": ok}
            eng.close()
            print(json.dumps({"workload": wl, "lib": os.path.basename(_lib.LIB_PATH), **kw,
                              "mean_ms": float(np.mean([v["ms"] for v in res.values()])),
                              "parity": all(v["parity"] for v in res.values()), "queries": res}), flush=True)
    else:
        raise SystemExit(f"unknown workload {wl}")


if __name__ == "__main__":
    main()
