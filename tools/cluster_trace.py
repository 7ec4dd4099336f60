#!/usr/bin/env python
"""Per-sweep timeline of one EAT_KERNEL_CLUSTER query (rank 0, thread 0,
globaltimer): select / barrier 1 / pairs / push + barrier 2, from a library
built with -DEAT_CL_TRACE (tools/build_variant.py cltrace -DEAT_CL_TRACE).

  python tools/cluster_trace.py ab/libeat_cltrace.so CFG [cluster_ctas] [window]
"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1912_00966_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.abspath(sys.argv[1])
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_00966_b200 import Engine  # noqa: E402

cfg = sys.argv[2]
ctas = int(sys.argv[3]) if len(sys.argv) > 3 else 0
window = int(sys.argv[4]) if len(sys.argv) > 4 else 0x7FFFFFFF
tt = synth.generate(cfg)
eng = Engine.from_timetable(tt, kernel="cluster", cluster_ctas=ctas, subtrips=3, window=window)
out = torch.empty(tt.num_vertices, dtype=torch.int32, device="cuda")
for _ in range(3):
    eng.query_device(*synth.SINGLE_QUERY, out)
torch.cuda.synchronize()
sw = eng.stats()["last_sweeps"]
buf = (ctypes.c_ulonglong * (1024 * 6))()
_lib.lib().eat_debug_cluster_trace(buf, 1024 * 6)
t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 6)[:min(sw, 1024)].astype(np.int64)
if os.environ.get("EAT_CLUSTER_ASYNC", "1") != "0":  # asynchronous loop: start, after select, after pairs, F
    busy = t[:, 5] > 0
    d = {"select": np.diff(t[:, [0, 1]]).ravel(), "pairs": np.diff(t[busy][:, [1, 3]]).ravel(),
         "F": t[busy, 5].astype(np.float64), "idle_iterations": np.array([float((~busy).sum())])}
else:
    d = {"select": np.diff(t[:, [0, 1]]).ravel(), "barrier1": np.diff(t[:, [1, 2]]).ravel(),
         "pairs": np.diff(t[:, [2, 3]]).ravel(), "push_barrier2": np.diff(t[:, [3, 4]]).ravel()}
d["sweep"] = np.diff(t[:, 0]) if sw > 1 else np.array([0])
print(json.dumps({"cfg": cfg, "cluster_ctas": eng.stats()["cluster_ctas"], "window": window, "sweeps": int(sw),
                  "ns_mean": {k: float(v.mean()) for k, v in d.items()},
                  "ns_p90": {k: float(np.percentile(v, 90)) for k, v in d.items()},
                  "first_sweeps_ns": t[:8, :6].tolist()}))
