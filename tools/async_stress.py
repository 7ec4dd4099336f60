#!/usr/bin/env python
"""Stress the termination protocols of the asynchronous single-query kernels
(cluster / grid-async): many seeded single queries, every row
compared with the serial CSA oracle.  A false termination would leave some
vertex too late (a row differs); a hang would trip the gpurun timeout.

  python tools/async_stress.py [--city 2000] [--metro 200]

One JSON line per (config, kernel): queries, mismatching rows, wall seconds.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_1912_00966_b200 import Engine  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--city", type=int, default=2000)
    ap.add_argument("--metro", type=int, default=200)
    args = ap.parse_args()
    for cfg, nq, kernels in (("city", args.city, ("cluster", "grid_async")), ("metro", args.metro, ("grid_async",))):
        if nq <= 0:
            continue
        tt = synth.generate(cfg)
        rng = np.random.default_rng(11)
        src = rng.integers(0, tt.num_vertices, nq).astype(np.uint32)
        ts = rng.integers(0, 24 * 3600, nq).astype(np.uint32)
        want = oracle.CSA(tt.num_vertices, *tt.arrays()).query_many(src, ts)
        for kernel in kernels:
            eng = Engine.from_timetable(tt, subtrips=3, kernel=kernel)
            t0 = time.time()
            bad = 0
            for i in range(nq):
                if not np.array_equal(eng.query(int(src[i]), int(ts[i])), want[i]):
                    bad += 1
            print(json.dumps({"config": cfg, "kernel": kernel, "queries": nq, "mismatching_rows": bad,
                              "seconds": round(time.time() - t0, 1)}), flush=True)
            eng.close()


if __name__ == "__main__":
    main()
