#!/usr/bin/env python
"""Benchmark of the EAT hot path (BASELINE.json metric: EAT queries/s and
single-query ms at 1/2/4/8 B200; achieved bandwidth vs peak).

Default workload (BASELINE.json configs[2]): the batched city network -- ONE
fixed batch of 10,000 queries (1,000 random sources x 10 random departure
times, seed 7: the paper's protocol PAPER.md:458-460 scaled x10) on the
synthetic ~10k-stop / ~30k-edge / ~2M-connection city timetable.  One step =
the whole batch (every query runs the whole hot path: init, Cluster-AP
relaxation sweeps to the fixpoint, output of e[] for all stops).  With N
ranks the same 10k queries are split into N contiguous shards (strong
scaling, no data-path collective: queries are independent);
the line also carries a weak-scaling figure (every rank its own 10k).

Beside it, on the same line: single-query latency for configs[1] (city),
configs[3] (metro) and configs[4] (country; at N > 1 edge-partitioned over
the ranks, NCCL min-allreduce and in-kernel peer exchange), each with p50/p90
over 100 seeded queries and a parity flag against the oracle; the
roofline of the batched kernel against the L2 read bandwidth measured in the
same run; the oracle (serial CSA) on all host cores, whose rows are compared
with the device rows (parity over every row it solved).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Timing: CUDA events on the launching stream around each step's launch, L2
flushed (256 MiB write) between steps outside the events, barrier +
synchronize around the K steps, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EAT queries/s"
UNIT = "queries/s"
BATCH = (1000, 10)  # sources x times: BASELINE configs[2]'s 10k queries
BATCH_WORKLOADS = {
    # name: (synth config, (sources, times), description)
    "city_batch": ("city", BATCH, "city_batch_10k (BASELINE configs[2]: one 10k-query batch split over the GPUs)"),
    "metro_batch": ("metro", (256, 4), "metro_batch_1k (SURVEY 8(a) a12 with e[] in global memory: 1,024 "
                                       "metro queries split over the GPUs, CTA groups of one launch)"),
}
LATENCY_QUERIES = 100  # seeded (s, t_s) per config for p50/p90
PARITY_K = 10          # of which compared with the oracle


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _init_dist():
    """One process per GPU (torchrun env); rank r drives GPU LOCAL_RANK.
    EAT_BENCH_BACKEND=gloo (with more ranks than GPUs, ranks share devices
    round-robin) exercises the multi-rank logic on a one-GPU box."""
    import torch

    rank, world, local = _dist()
    ndev = max(1, torch.cuda.device_count())
    dev = local % ndev
    torch.cuda.set_device(dev)
    if world > 1:
        import torch.distributed as dist

        backend = os.environ.get("EAT_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines show the N ranks ...
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # ... on stderr: stdout is the JSON line
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    return rank, world, dev


def _reduce(x: float, dev: int, op: str = "max") -> float:
    """MAX / MIN / SUM of a host float over all ranks."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return x
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "min": dist.ReduceOp.MIN, "sum": dist.ReduceOp.SUM}[op])
    return float(t.item())


def _barrier():
    import torch.distributed as dist

    if dist.is_initialized():
        dist.barrier()


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _host_info() -> dict:
    """nproc, usable cores, CPU model, sockets, NUMA nodes of this host."""
    info = {"nproc": os.cpu_count()}
    try:
        info["usable_cores"] = len(os.sched_getaffinity(0))
    except Exception:
        info["usable_cores"] = os.cpu_count()
    try:
        txt = open("/proc/cpuinfo").read()
        models = [ln.split(":", 1)[1].strip() for ln in txt.splitlines() if ln.startswith("model name")]
        info["cpu_model"] = models[0] if models else None
        info["sockets"] = len({ln for ln in txt.splitlines() if ln.startswith("physical id")}) or None
    except Exception:
        info["cpu_model"] = None
    try:
        info["numa_nodes"] = len([d for d in os.listdir("/sys/devices/system/node") if d.startswith("node")])
    except Exception:
        info["numa_nodes"] = None
    return info


def _resolved(tt, ts):
    """connections-effectively-resolved: sum over queries of |{c : dep_c >= t_s}|
    (the set serial CSA must scan)."""
    d = np.sort(tt.dep)
    return int((d.size - np.searchsorted(d, ts, side="left")).sum())


def _oracle_rows(csa, src, ts, budget_s: float, threads: int, chunk: int = 16):
    """The oracle (serial CSA, oracle/csa.c, as it stands) over the queries
    in order on `threads` host threads (one query at a time per worker, each
    with its own output rows = private e[]; ctypes releases the GIL), until
    every query is done or the time budget is spent.  Returns (rows, done,
    seconds)."""
    nq = src.size
    rows = np.empty((nq, csa.n), dtype=np.uint32)
    t0 = time.perf_counter()

    def work(a):
        b = min(nq, a + chunk)
        rows[a:b] = csa.query_many(src[a:b], ts[a:b])
        return b - a

    done = 0
    with ThreadPoolExecutor(max_workers=threads) as ex:
        futs = []
        a = 0
        while a < nq:
            # keep ~2 chunks per worker in flight; stop submitting at the budget
            while a < nq and len(futs) < 2 * threads:
                futs.append(ex.submit(work, a))
                a += chunk
            done += futs.pop(0).result()
            if time.perf_counter() - t0 > budget_s:
                break
        for f in futs:
            done += f.result()
    dt = time.perf_counter() - t0
    return rows[:done], done, dt


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (this tier's
    reference arm), same workload/metric; rank 0 only."""
    rank, world, _ = _dist()
    if rank != 0:
        return
    import oracle
    import synth

    tt = synth.generate("city")
    src, ts = synth.queries(tt, *BATCH)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    host = _host_info()
    threads = host["usable_cores"] or 1
    per_step = int(args.ref_queries) if args.ref_queries else min(src.size, 128 * threads)
    for w in range(args.warmup):
        csa.query_many(src[:8], ts[:8])
    times = []
    for k in range(args.steps):
        a = (k * per_step) % src.size
        sl = np.arange(a, a + per_step) % src.size
        t0 = time.perf_counter()
        _, done, _ = _oracle_rows(csa, src[sl], ts[sl], 1e9, threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = per_step * args.steps / tot
    sample = (f"{per_step} of the 10,000 city-batch queries per step (cyclic), serial CSA (oracle/csa.c, gcc -O3), "
              f"{threads} host threads, one query per task, private e[] per query; queries/s extrapolates")
    cpu = {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": sample, **host}
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": BATCH_WORKLOADS["city_batch"][2], "stops": tt.num_vertices,
                       "connections": tt.num_connections, "queries_per_step": per_step},
            "cpu_baseline": cpu,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ latency legs
def _seeded_queries(tt, nq, seed=7):
    rng = np.random.default_rng(seed)
    return [(int(rng.integers(tt.num_vertices)), int(rng.integers(0, 86400))) for _ in range(nq)]


def _latency_dist(eng, tt, dev, stream, flush, csa, nq=LATENCY_QUERIES, parity_k=PARITY_K):
    """s=0 at 06:00 plus `nq` seeded (s, t_s): device ms per query (CUDA
    events on the launching stream, L2 flushed before each), sweeps; the first
    `parity_k` and the s=0 query compared with the oracle row by row."""
    import torch
    import synth

    out = torch.empty(tt.num_vertices, dtype=torch.int32, device=dev)
    qs = [synth.SINGLE_QUERY] + _seeded_queries(tt, nq)
    for q in qs[:3]:
        eng.query_device(*q, out, stream=stream)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms, sweeps, ok, checked = [], [], True, 0
    for i, q in enumerate(qs):
        with torch.cuda.stream(stream):
            flush.fill_(i)
            a.record(stream)
            eng.query_device(*q, out, stream=stream)
            b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
        sweeps.append(eng.stats()["last_sweeps"])
        if csa is not None and i <= parity_k:
            ok &= bool(np.array_equal(out.cpu().numpy().view(np.uint32), csa.query(*q)))
            checked += 1
    m = np.array(ms[1:])
    return {"s0_0600_ms": ms[0], "s0_0600_sweeps": sweeps[0], "p50_ms": float(np.percentile(m, 50)),
            "p90_ms": float(np.percentile(m, 90)), "mean_ms": float(m.mean()), "max_ms": float(m.max()),
            "queries": len(m), "seed": 7, "sweeps_p50": float(np.median(sweeps[1:])),
            "kernel": eng.stats()["kernel_name"], "l2": "flushed before each query",
            "parity": ok if checked else None, "parity_rows": checked}


def _latency_legs(args, rank, world, dev, stream, flush, city_tt):
    """Single-query latency for BASELINE configs[1], [3], [4]."""
    import torch
    import oracle
    import synth
    from paper_1912_00966_b200 import Engine

    res = {}
    cfgs = [c for c in args.latency.split(",") if c]
    for cfg in cfgs:
        if world > 1 and cfg != "country":
            continue  # replicated single-query latency: one GPU's figure (N = 1)
        t0 = time.perf_counter()
        tt = city_tt if cfg == "city" else synth.generate(cfg)
        gen_s = time.perf_counter() - t0
        if cfg == "country" and world > 1:
            res["country_part"] = _country_partitioned(args, rank, world, dev, stream, flush, tt)
            continue
        csa = oracle.CSA(tt.num_vertices, *tt.arrays()) if not args.no_cpu else None
        t0 = time.perf_counter()
        eng = Engine.from_timetable(tt, device=dev, subtrips=args.subtrips)
        build_s = time.perf_counter() - t0
        d = _latency_dist(eng, tt, dev, stream, flush, csa)
        d.update({"stops": tt.num_vertices, "connections": tt.num_connections, "generate_s": gen_s,
                  "build_s": build_s, "subtrips": args.subtrips})
        if cfg == "city":  # warm back-to-back figure of both single-query kernels (round-1 key)
            o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device=dev)
            d["warm_ms"] = {}
            for kname in ("cta", "frontier", "cluster"):
                e1 = Engine.from_timetable(tt, device=dev, kernel=kname, subtrips=args.subtrips)
                for _ in range(3):
                    e1.query_device(*synth.SINGLE_QUERY, o1, stream=stream)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                for _ in range(20):
                    e1.query_device(*synth.SINGLE_QUERY, o1, stream=stream)
                b.record(stream)
                b.synchronize()
                d["warm_ms"][kname] = a.elapsed_time(b) / 20
                e1.close()
        eng.close()
        if csa is not None:
            csa.close()
        res[cfg] = d
    return res


def _country_partitioned(args, rank, world, dev, stream, flush, tt):
    """configs[4] at N > 1: one query edge-partitioned over the ranks, with
    the NCCL min-allreduce exchange (to local quiescence, and one allreduce
    per sweep) and with the in-kernel peer exchange.  Rows are compared
    across the three schedules (the oracle's country parity runs in
    tests/test_gpu_parity.py::test_country_single_query)."""
    import torch
    import synth
    from paper_1912_00966_b200.parallel import edge_partitioned_engine, peer_partitioned_engine

    out = torch.empty(tt.num_vertices, dtype=torch.int32, device=dev)
    res, rows = {}, {}
    variants = (("allreduce", dict(local_sweeps=0)), ("allreduce_per_sweep", dict(local_sweeps=1)),
                ("peer", None))
    for name, kw in variants:
        try:
            eng = (peer_partitioned_engine(tt, device=dev, subtrips=args.subtrips) if kw is None else
                   edge_partitioned_engine(tt, device=dev, subtrips=args.subtrips, **kw))
        except Exception as exc:  # keep the line: report why this exchange did not run
            res[name] = {"error": repr(exc)[:300]}
            continue
        for _ in range(2):
            eng.query_device(*synth.SINGLE_QUERY, out, stream=stream)
        torch.cuda.synchronize()
        _barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms = []
        for i in range(5):
            with torch.cuda.stream(stream):
                flush.fill_(i)
                a.record(stream)
                eng.query_device(*synth.SINGLE_QUERY, out, stream=stream)
                b.record(stream)
            b.synchronize()
            ms.append(_reduce(a.elapsed_time(b), dev, "max"))
        st = eng.stats()
        rows[name] = out.cpu().numpy().copy()
        res[name] = {"ms_median": float(np.median(ms)), "rounds": st["last_rounds"], "sweeps": st["last_sweeps"],
                     "time": "device, max over ranks"}
        eng.close()
    names = list(rows)
    agree = all(np.array_equal(rows[names[0]], rows[k]) for k in names[1:]) if names else None
    res["rows_agree_across_exchanges"] = bool(_reduce(float(bool(agree)), dev, "min")) if names else None
    res["ranks"] = world
    return res


# ------------------------------------------------------------------ roofline
def _probe_l2_gbs(dev, stream) -> float:
    """L2-resident read bandwidth measured now (eat_probe_read: 32 MiB
    buffer, 128-bit loads, 148 x 8 CTAs), the peak of the L2-bound batch."""
    import torch
    from paper_1912_00966_b200 import _lib

    buf = torch.ones(8 * 1024 * 1024, dtype=torch.int32, device=dev)  # 32 MiB
    nbytes, reps = buf.numel() * 4, 64
    _lib.eat_probe_read(buf.data_ptr(), nbytes, 2, int(stream.cuda_stream))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0.0
    for _ in range(3):
        a.record(stream)
        _lib.eat_probe_read(buf.data_ptr(), nbytes, reps, int(stream.cuda_stream))
        b.record(stream)
        b.synchronize()
        best = max(best, nbytes * reps / (a.elapsed_time(b) / 1e3) / 1e9)
    return best


def _batch_roofline(tt, src, ts, dev, stream, args, step_ms, st0):
    """roofline of the batched CTA kernel: SURVEY 8(d) algorithmic bytes
    (instrumented run on the same queries) / mean launch time, against the
    L2 read bandwidth measured in this run (the index is L2-resident);
    the HBM fraction and the ncu-measured DRAM traffic beside it."""
    hbm, hbm_src = _hbm_peak()
    if st0["cta_grid"] == 0:
        # batches on CTA groups (e[] in global memory): no instrumented
        # variant; the DRAM traffic of the ncu capture against HBM peak
        traffic, src_ = None, None
        tp = os.path.join(ROOT, "profiles", "traffic_metro_batch.json")
        if os.path.exists(tp):
            with open(tp) as f:
                tj = json.load(f)
            traffic = tj["dram_bytes_per_launch"] * len(src) / tj["queries_per_launch"]
            src_ = tj["source"]
        mean_launch_s = (sum(step_ms) / len(step_ms)) / 1e3
        dram_gbs = traffic / mean_launch_s / 1e9 if traffic else None
        return {"bound": "hbm", "achieved": dram_gbs, "peak": hbm, "unit": "GB/s",
                "frac": dram_gbs / hbm if dram_gbs else None, "traffic": traffic, "kernel": "k_query_groups",
                "achieved_is": "measured DRAM bytes (ncu, scaled to this launch's queries) / mean launch time",
                "traffic_source": src_, "note": "random 32-byte gathers of a non-L2-resident index: latency-bound "
                                                "(DESIGN.md §6)"}
    try:
        from paper_1912_00966_b200 import counters

        cnt = counters.count_batch(tt, src, ts, dev, subtrips=args.subtrips)
        mean_launch_s = (sum(step_ms) / len(step_ms)) / 1e3
        achieved = cnt["algorithmic_bytes"] / mean_launch_s / 1e9
        l2 = _probe_l2_gbs(dev, stream)
        traffic, ncu_src, tj = None, None, {}
        tp = os.path.join(ROOT, "profiles", "traffic_city_batch.json")
        tp_ok = os.path.exists(tp)
        if tp_ok:
            with open(tp) as f:
                tj = json.load(f)
            traffic, ncu_src = tj.get("dram_bytes_per_launch"), tj.get("source")
        return {"bound": "l2", "achieved": achieved, "peak": l2, "unit": "GB/s", "frac": achieved / l2,
                "traffic": traffic, "kernel": f"k_query_cta<0,{st0['cta_threads']},512,0,0>",
                "peak_source": "measured in this run: eat_probe_read, 32 MiB L2-resident buffer, 128-bit loads",
                "algorithmic_bytes_per_launch": cnt["algorithmic_bytes"],
                "layout_bytes_per_launch": cnt["layout_bytes"],
                "bytes_rule": "SURVEY 8(d): 12 B/active source + 12 B/edge eval + 16 B/type header + "
                              "(12 + 8 runs + 4 singles) B/cluster slot + 4 B/fallback + 8 B + 4|V| B per query",
                "counters": cnt,
                "hbm": {"peak": hbm, "peak_source": hbm_src, "frac_of_algorithmic": achieved / hbm,
                        "dram_gbs": (traffic / mean_launch_s / 1e9) if traffic else None,
                        "dram_frac": (traffic / mean_launch_s / 1e9 / hbm) if traffic else None,
                        "traffic_source": ncu_src},
                # what actually bounds it: instruction issue -- the
                # committed ncu capture's issue-slot utilisation and IPC of 4
                "issue": {"issue_active_frac": (tj.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0) / 100.0)
                          if tp_ok else None,
                          "warp_instructions_per_query": (tj.get("warp_instructions", 0) / 1e4) if tp_ok else None,
                          "source": ncu_src}}
    except Exception as exc:  # keep the bench line even if accounting fails
        return {"bound": "l2", "achieved": None, "peak": None, "unit": "GB/s", "frac": None, "traffic": None,
                "error": repr(exc)}


# ------------------------------------------------------------------ main line
def _time_batch(eng, d_src, d_ts, d_out, stream, flush, steps):
    import torch

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        with torch.cuda.stream(stream):
            flush.fill_(k)
            ev[k][0].record(stream)
            eng.query_many_device(d_src, d_ts, d_out, stream=stream)
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


def run_gpu(args):
    import torch

    rank, world, dev = _init_dist()
    import synth
    from paper_1912_00966_b200 import Engine, pinned_empty

    cfg_name, (nsrc, ntime), wl_desc = BATCH_WORKLOADS[args.workload]
    city = cfg_name == "city"
    tt = synth.generate(cfg_name)
    all_src, all_ts = synth.queries(tt, nsrc, ntime)  # the same batch for every N (strong scaling)
    NQ = all_src.size
    lo, hi = NQ * rank // world, NQ * (rank + 1) // world
    src, ts = all_src[lo:hi], all_ts[lo:hi]
    nq = src.size
    eng = Engine.from_timetable(tt, device=dev, kernel="auto", subtrips=args.subtrips)
    st0 = eng.stats()
    stream = torch.cuda.Stream(device=dev)
    d_src = torch.tensor(src.astype(np.int32), device=dev)
    d_ts = torch.tensor(ts.astype(np.int32), device=dev)
    d_out = torch.empty((nq, tt.num_vertices), dtype=torch.int32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            eng.query_many_device(d_src, d_ts, d_out, stream=stream)
    torch.cuda.synchronize()
    _barrier()
    clocks = Clocks(dev)
    clocks.start()
    torch.cuda.synchronize()
    _barrier()
    step_ms = _time_batch(eng, d_src, d_ts, d_out, stream, flush, args.steps)
    _barrier()
    clk = clocks.stop()
    tot_ms = _reduce(float(sum(step_ms)), dev, "max")
    value = NQ * args.steps / (tot_ms / 1e3)

    # ---- weak scaling beside it: every rank its own full batch
    weak = None
    if world > 1:
        w_src, w_ts = synth.queries(tt, nsrc * world, ntime)
        per = nsrc * ntime
        wd_src = torch.tensor(w_src[rank * per:(rank + 1) * per].astype(np.int32), device=dev)
        wd_ts = torch.tensor(w_ts[rank * per:(rank + 1) * per].astype(np.int32), device=dev)
        wd_out = torch.empty((per, tt.num_vertices), dtype=torch.int32, device=dev)
        eng.query_many_device(wd_src, wd_ts, wd_out, stream=stream)
        torch.cuda.synchronize()
        _barrier()
        wms = _reduce(float(sum(_time_batch(eng, wd_src, wd_ts, wd_out, stream, flush, 3))), dev, "max")
        weak = {"value": world * per * 3 / (wms / 1e3), "unit": UNIT, "queries_per_gpu": per,
                "note": "every rank solves its own 10k queries (weak scaling)"}
        del wd_out

    # ---- the same batch with other sub-trip settings (N = 1): none (plain
    # Cluster-AP index) and the paper's scheme 2 (r = sqrt(avg trip))
    variants = {}
    if city and world == 1 and not args.fast:
        for st_alt, key in ((0, "no_subtrips_queries_per_s"), (2, "paper_scheme2_queries_per_s")):
            if st_alt == args.subtrips:
                continue
            eng0 = Engine.from_timetable(tt, device=dev, kernel="auto", subtrips=st_alt)
            eng0.query_many_device(d_src, d_ts, d_out, stream=stream)
            ms0 = _time_batch(eng0, d_src, d_ts, d_out, stream, flush, 3)
            variants[key] = nq * 3 / (sum(ms0) / 1e3)
            eng0.close()
        eng.query_many_device(d_src, d_ts, d_out, stream=stream)  # rows of the bench configuration again
        torch.cuda.synchronize()

    # ---- e2e through the public API with host buffers: pinned host queries
    # in, every step H2D of the queries + kernel + all result rows into pinned
    # host memory (eat_query_many "direct" mode: each CTA stores its finished
    # rows into the mapped host buffer over PCIe, overlapped with the other
    # queries' relaxation)
    h_out = pinned_empty((nq, tt.num_vertices))
    h_src, h_ts = pinned_empty((nq,)), pinned_empty((nq,))
    h_src[:] = src
    h_ts[:] = ts
    e2e_steps = max(1, min(args.steps, 5))
    eng.query_many(h_src, h_ts, out=h_out)  # warm-up (buffers)
    _barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.query_many(h_src, h_ts, out=h_out)
    e2e_s = _reduce(time.perf_counter() - t0, dev, "max")
    e2e_value = NQ * e2e_steps / e2e_s
    dev_rows = d_out.cpu().numpy().view(np.uint32)
    e2e_ok = bool(_reduce(float(np.array_equal(h_out, dev_rows)), dev, "min"))

    # ---- oracle beside it: all host cores at N = 1 (rank 0), whose rows are
    # compared with the device rows; at N > 1 every rank checks a sample of
    # its shard on one core
    import oracle

    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    host = _host_info()
    cpu, parity_rows, parity = None, 0, None
    if world == 1 and not args.no_cpu:
        threads = host["usable_cores"] or 1
        csa.query(int(src[0]), int(ts[0]))  # warm-up
        rows, done, dt = _oracle_rows(csa, src, ts, args.cpu_seconds, threads)
        parity_rows = done
        parity = bool(np.array_equal(rows, dev_rows[:done]))
        cpu = {"value": done / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"the first {done} of the {nq} batch queries, serial CSA (oracle/csa.c, gcc -O3) on "
                         f"{threads} host threads (one query per task, private e[]), {dt:.1f} s; "
                         f"its rows double as the parity reference", **host}
        del rows
    else:
        k = min(nq, 32)
        pick = np.linspace(0, nq - 1, k).astype(np.int64) if nq else np.zeros(0, np.int64)
        ok = bool(np.array_equal(csa.query_many(src[pick], ts[pick]), dev_rows[pick])) if k else True
        parity = bool(_reduce(float(ok), dev, "min"))
        parity_rows = int(_reduce(float(k), dev, "sum"))
    csa.close()
    del dev_rows

    # ---- roofline of the batched kernel (rank 0)
    roof = _batch_roofline(tt, src, ts, dev, stream, args, step_ms, st0) if rank == 0 else None

    line = None
    if rank == 0:
        resolved = _resolved(tt, all_ts) * args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": wl_desc,
                       "stops": tt.num_vertices, "edges": st0["num_edges"], "connections": tt.num_connections,
                       "types": st0["num_types"], "queries_per_step": NQ, "queries_per_gpu": nq,
                       "parallelism": f"query-sharded x{world} (contiguous shards, no collective)",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "kernel": "cta (batched)" if st0["cta_grid"] > 0 else
                       "CTA groups (k_query_groups, warp-flattened pairs + time window)",
                       "subtrips": args.subtrips, "window_s": 1500 if st0["cta_grid"] > 0 else 2400,
                       "cta_threads": st0["cta_threads"] if st0["cta_grid"] > 0 else None,
                       "shortcuts": st0["num_shortcuts"]},
            "parity": parity, "parity_rows": parity_rows,
            "parity_rule": "device rows == oracle rows (serial CSA on the raw timetable), every stop, bit-exact",
            "connections_resolved_per_s": resolved / (tot_ms / 1e3),
            "weak_scaling": weak,
            "variants": variants,
            "single_query_ms": None,
            "latency": None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(NQ * 8),
                    "d2h_bytes_per_step": int(NQ * tt.num_vertices * 4), "host_buffers": "pinned",
                    "rows_match_device_run": e2e_ok},
            # per step: the batched kernel, plus (more queries than resident
            # CTAs) the departure-time hand-out order -- our key kernel and the
            # 5 launches of cub's radix sort compiled into libeat
            "gpu_launches": args.steps * (2 if (st0["cta_grid"] > 0 and nq > st0["cta_grid"]) else 1),
            "library_launches": args.steps * (5 if (st0["cta_grid"] > 0 and nq > st0["cta_grid"]) else 0),
            "clocks": clk,
            "roofline": roof,
            "cpu_baseline": cpu,
        }

    # ---- single-query latency (configs[1], [3], [4]) under a watchdog: the
    # headline line above is complete, so a leg that fails or hangs (e.g. a
    # collective of the N > 1 edge partition) costs only its own keys
    emitted = threading.Lock()

    def emit(lat):
        if not emitted.acquire(blocking=False):
            return False
        if rank == 0:
            line["latency"] = lat
            line["single_query_ms"] = {k: v["s0_0600_ms"] for k, v in lat.items()
                                       if isinstance(v, dict) and "s0_0600_ms" in v}
            print(json.dumps(line), flush=True)
        return True

    def on_timeout():
        if emit({"error": f"latency legs did not finish within {args.leg_timeout} s"}):
            os._exit(0)

    wd = threading.Timer(args.leg_timeout, on_timeout)
    wd.daemon = True
    wd.start()
    try:
        latency = _latency_legs(args, rank, world, dev, stream, flush, tt) if city else {}
    except Exception as exc:  # noqa: BLE001 -- reported in the line
        latency = {"error": repr(exc)[:300]}
    wd.cancel()
    if not emit(latency):
        return
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


SINGLE_WORKLOADS = {
    # name: (synth config, engine kwargs, BASELINE configs[] it measures)
    "city_single": ("city", {}, "BASELINE configs[1]: city, 1 query s=0 t_s=06:00"),
    "metro_single": ("metro", {}, "BASELINE configs[3]: metro (30% irregular), 1 query s=0 t_s=06:00"),
    "country_part": ("country", {"mode": "edge_partitioned"},
                     "BASELINE configs[4]: country, 1 query s=0 t_s=06:00, edge-partitioned over the ranks "
                     "(NCCL min-allreduce of e[] per exchange round)"),
}


def run_single(args):
    """One single-query workload as its own line (metric: EAT single-query ms)."""
    import torch

    rank, world, dev = _init_dist()
    import synth
    from paper_1912_00966_b200 import Engine
    from paper_1912_00966_b200.parallel import nccl_unique_id

    cfg, kw, desc = SINGLE_WORKLOADS[args.workload]
    t0 = time.perf_counter()
    tt = synth.generate(cfg)
    gen_s = time.perf_counter() - t0
    kw = dict(kw, subtrips=args.subtrips)
    mode_label = kw.get("mode", "replicated")
    if mode_label == "edge_partitioned" and args.exchange == "peer":
        desc = desc.replace("NCCL min-allreduce of e[] per exchange round",
                            "in-kernel peer exchange: atomicMin on the owner's e[] over NVLink + inbox, NEXT-2")
    t0 = time.perf_counter()
    if kw.get("mode") == "edge_partitioned" and args.exchange == "peer":
        from paper_1912_00966_b200.parallel import peer_partitioned_engine

        kw.pop("mode")
        eng = peer_partitioned_engine(tt, device=dev, **kw) if world > 1 else Engine.from_timetable(
            tt, device=dev, mode="edge_partitioned", exchange="peer", **kw)
    else:
        if kw.get("mode") == "edge_partitioned":
            kw.update(part_rank=rank, part_count=world, nccl_unique_id=nccl_unique_id() if world > 1 else None,
                      local_sweeps=args.local_sweeps)
        eng = Engine.from_timetable(tt, device=dev, **kw)
    build_s = time.perf_counter() - t0
    st0 = eng.stats()
    s, t_s = synth.SINGLE_QUERY
    stream = torch.cuda.Stream(device=dev)
    out = torch.empty(tt.num_vertices, dtype=torch.int32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)
    for _ in range(args.warmup):
        eng.query_device(s, t_s, out, stream=stream)
    torch.cuda.synchronize()
    _barrier()
    clocks = Clocks(dev)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(k)
            ev[k][0].record(stream)
            eng.query_device(s, t_s, out, stream=stream)
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    _barrier()
    clk = clocks.stop()
    ms = [a.elapsed_time(b) for a, b in ev]
    tot = _reduce(float(sum(ms)), dev, "max")
    st = eng.stats()
    # e2e: public host API (D2H of e[] into a page-locked host buffer included)
    from paper_1912_00966_b200 import pinned_empty

    h = pinned_empty((tt.num_vertices,))
    eng.query(s, t_s, out=h)  # warm-up
    t0 = time.perf_counter()
    reps = max(1, min(args.steps, 5))
    for _ in range(reps):
        eng.query(s, t_s, out=h)
    e2e_ms = _reduce((time.perf_counter() - t0) * 1e3 / reps, dev, "max")
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        import oracle

        csa = oracle.CSA(tt.num_vertices, *tt.arrays())
        want = csa.query(s, t_s)
        t0 = time.perf_counter()
        k = 0
        while k < 5 and (k == 0 or time.perf_counter() - t0 < args.cpu_seconds):
            csa.query(s, t_s)
            k += 1
        cpu_ms = (time.perf_counter() - t0) * 1e3 / k
        cpu = {"value": cpu_ms, "unit": "ms", "cores": 1, "kind": "oracle",
               "sample": f"the same query (s={s}, t_s={t_s}) x{k}, serial CSA (oracle/csa.c), 1 host core",
               "parity": bool(np.array_equal(h, want)), **_host_info()}
        csa.close()
    if rank == 0:
        line = {"metric": "EAT single-query ms", "value": tot / args.steps, "unit": "ms", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot / args.steps,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
                "data": "synthetic",
                "config": {"workload": f"{args.workload} ({desc})", "stops": tt.num_vertices,
                           "connections": tt.num_connections, "edges": st0["num_edges"], "types": st0["num_types"],
                           "kernel": st0["kernel_name"], "mode": mode_label,
                           "exchange": args.exchange if mode_label == "edge_partitioned" else None,
                           "local_sweeps": args.local_sweeps if mode_label == "edge_partitioned" else None,
                           "l2": "flushed (256 MiB write) between timed steps", "index_bytes": st0["index_bytes"],
                           "generate_s": gen_s, "build_s": build_s, "subtrips": args.subtrips,
                           "shortcuts": st0["num_shortcuts"]},
                "sweeps": st["last_sweeps"], "rounds": st["last_rounds"],
                "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 8,
                        "d2h_bytes_per_step": tt.num_vertices * 4},
                "gpu_launches": args.steps * max(1, st["last_rounds"]),
                "clocks": clk, "roofline": None, "cpu_baseline": cpu}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="time budget of the all-cores oracle leg (its rows are the batch parity reference)")
    ap.add_argument("--ref-queries", type=int, default=0, help="--impl reference: queries per step (0: 128 x cores)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--leg-timeout", type=float, default=900.0,
                    help="seconds the single-query latency legs may take before the line is printed without them")
    ap.add_argument("--fast", action="store_true", help="skip the sub-trip variants")
    ap.add_argument("--latency", default="city,metro,country",
                    help="single-query latency legs of the batch line (configs[1], [3], [4]); '' = none")
    ap.add_argument("--subtrips", type=int, default=3,
                    help="sub-trip shortcuts (PAPER.md:342-354): 0 off, 1 r=sqrt(k) per trip, 2 r=sqrt(avg) "
                         "(the paper's scheme 2), >=3 fixed r (default 3: +3 %% q/s over scheme 2 on B200, "
                         "profiles/r01_sweep_subtrips_r.jsonl)")
    ap.add_argument("--workload", default="city_batch", choices=sorted(BATCH_WORKLOADS) + sorted(SINGLE_WORKLOADS))
    ap.add_argument("--exchange", default="allreduce", choices=["allreduce", "peer"],
                    help="country_part: per-round NCCL min-allreduce of e[] (BASELINE configs[4]) or the in-kernel "
                         "peer exchange over NVLink (NEXT-2, CUDA IPC between the ranks)")
    ap.add_argument("--local-sweeps", type=int, default=0,
                    help="country_part allreduce: local sweeps per exchange round (0 = to quiescence, 1 = one "
                         "allreduce per sweep)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.workload in BATCH_WORKLOADS:
        run_gpu(args)
    else:
        run_single(args)


if __name__ == "__main__":
    main()
