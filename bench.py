#!/usr/bin/env python
"""Benchmark of the EAT hot path (BASELINE.json metric: EAT queries/s and
single-query ms; achieved bandwidth vs peak).

Default workload (BASELINE.json configs[2], the batched city network): every
rank solves a batch of 10,000 queries (1,000 random sources x 10 random
departure times, the paper's protocol PAPER.md:458-460 scaled x10) on the
synthetic ~10k-stop / ~30k-edge / ~2M-connection city timetable.  One step =
one batch (every query runs the whole hot path: init, Cluster-AP relaxation
sweeps to the fixpoint, output of e[] for all stops).  Queries are
independent, so N ranks shard nothing: each rank gets its own 10k queries
(weak scaling, no data-path collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Timing: CUDA events on the launching stream around each step's single
kernel launch, L2 flushed (256 MiB write) between steps outside the events,
barrier + synchronize around the K steps, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "EAT queries/s"
UNIT = "queries/s"
QUERIES_PER_RANK = (1000, 10)  # sources x times
BATCH_WORKLOADS = {
    # name: (synth config, (sources, times) per rank, description)
    "city_batch": ("city", QUERIES_PER_RANK, "city_batch_10k (BASELINE configs[2]; 10k queries per GPU)"),
    "metro_batch": ("metro", (256, 4), "metro_batch_1k (SURVEY 8(a) a12 with e[] in global memory: 1,024 "
                                       "metro queries per GPU, CTA groups of one launch)"),
}
L2_READ_GBS = 17805.0  # measured L2-resident read bandwidth, 32 MiB working set (profiles/r01_ncu_summary.md)


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
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    return rank, world, dev


def _max_over_ranks(x: float, dev: int) -> float:
    """Max of a host float over all ranks (device tensor under NCCL)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        return x
    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([x], dtype=torch.float64, device=dev if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


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


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def _resolved(tt, ts):
    """connections-effectively-resolved: sum over queries of |{c : dep_c >= t_s}|
    (the set serial CSA must scan)."""
    d = np.sort(tt.dep)
    return int((d.size - np.searchsorted(d, ts, side="left")).sum())


def _cpu_baseline(tt, src, ts, budget_s: float):
    """Oracle (serial CSA, oracle/csa.c) as it stands, one host core, on a
    bounded prefix of the same query list."""
    import oracle

    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    csa.query(int(src[0]), int(ts[0]))  # warm-up
    t0 = time.perf_counter()
    done = 0
    while done < src.size and time.perf_counter() - t0 < budget_s:
        k = min(64, src.size - done)
        csa.query_many(src[done:done + k], ts[done:done + k])
        done += k
    dt = time.perf_counter() - t0
    csa.close()
    return {"value": done / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"first {done} of the {src.size} batch queries, serial CSA (oracle/csa.c, gcc -O3), "
                      f"{dt:.1f} s on 1 host core"}


def run_reference(args):
    """--impl reference: the oracle as it stands on the host cores (this tier's
    reference arm), same workload/metric; rank 0 only."""
    rank, world, _ = _dist()
    if rank != 0:
        return
    import synth
    import oracle

    tt = synth.generate("city")
    src, ts = synth.queries(tt, *QUERIES_PER_RANK)
    csa = oracle.CSA(tt.num_vertices, *tt.arrays())
    per_step = int(args.ref_queries)
    for w in range(args.warmup):
        csa.query_many(src[:8], ts[:8])
    times = []
    for k in range(args.steps):
        sl = slice((k * per_step) % src.size, (k * per_step) % src.size + per_step)
        t0 = time.perf_counter()
        csa.query_many(src[sl], ts[sl])
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = per_step * args.steps / tot
    sample = (f"{per_step} of the 10,000 city-batch queries per step, serial CSA (oracle/csa.c), 1 host core; "
              f"steps time the bounded sample, queries/s extrapolates")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": "city_batch_10k (BASELINE configs[2])", "stops": tt.num_vertices,
                       "connections": tt.num_connections, "queries_per_step": per_step},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


SINGLE_WORKLOADS = {
    # name: (synth config, engine kwargs, BASELINE configs[] it measures)
    "city_single": ("city", {}, "BASELINE configs[1]: city, 1 query s=0 t_s=06:00"),
    "metro_single": ("metro", {}, "BASELINE configs[3]: metro (30% irregular), 1 query s=0 t_s=06:00"),
    "country_part": ("country", {"mode": "edge_partitioned"},
                     "BASELINE configs[4]: country, 1 query s=0 t_s=06:00, edge-partitioned over the ranks "
                     "(NCCL min-allreduce of e[] per exchange round)"),
}


def run_single(args):
    """Single-query latency workloads (metric: EAT single-query ms)."""
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
            kw.update(part_rank=rank, part_count=world, nccl_unique_id=nccl_unique_id() if world > 1 else None)
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
    if world > 1:
        torch.distributed.barrier()
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
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    ms = [a.elapsed_time(b) for a, b in ev]
    tot = float(sum(ms))
    tot = _max_over_ranks(tot, dev)
    st = eng.stats()
    # e2e: public host API (D2H of e[] into a page-locked host buffer included)
    from paper_1912_00966_b200 import pinned_empty

    h = pinned_empty((tt.num_vertices,))
    eng.query(s, t_s, out=h)  # warm-up
    t0 = time.perf_counter()
    reps = max(1, min(args.steps, 5))
    for _ in range(reps):
        eng.query(s, t_s, out=h)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / reps
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
               "parity": bool(np.array_equal(h, want))}
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


def _batch_roofline(tt, src, ts, dev, args, step_ms, st0):
    """roofline object of the batched kernel: algorithmic bytes (instrumented
    CTA-kernel run on the same queries) / mean launch time vs the HBM peak."""
    if st0["cta_grid"] == 0:  # grouped grid kernel: no instrumented variant for byte accounting
        return {"bound": "hbm", "achieved": None, "peak": _peaks()[0], "unit": "GB/s", "frac": None, "traffic": None,
                "kernel": "k_query_groups", "note": "latency-bound frontier sweeps (DESIGN.md §9)"}
    try:
        from paper_1912_00966_b200 import counters

        cnt = counters.count_batch(tt, src, ts, dev, subtrips=args.subtrips)
        alg_bytes = cnt["algorithmic_bytes"]
        mean_launch_s = (sum(step_ms) / len(step_ms)) / 1e3
        peak, peak_src = _peaks()
        achieved = alg_bytes / mean_launch_s / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic_city_batch.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src, "kernel": "k_query_cta",
                "algorithmic_bytes_per_launch": alg_bytes, "counters": cnt,
                # the index is L2-resident: the same bytes against the measured
                # L2-resident read bandwidth (tools/l2_bw.py, profiles/r01_ncu_summary.md)
                "l2": {"peak": L2_READ_GBS, "frac": achieved / L2_READ_GBS,
                       "note": "kernel is issue-bound (ncu: IPC 2.44 of 4), not bandwidth-bound"}}
    except Exception as exc:  # keep the bench line even if accounting fails
        return {"bound": "hbm", "achieved": None, "peak": _peaks()[0], "unit": "GB/s", "frac": None,
                "traffic": None, "error": repr(exc)}


def run_gpu(args):
    import torch

    rank, world, dev = _init_dist()
    import synth
    from paper_1912_00966_b200 import Engine

    cfg_name, (nsrc, ntime), wl_desc = BATCH_WORKLOADS[args.workload]
    city = cfg_name == "city"
    tt = synth.generate(cfg_name)
    all_src, all_ts = synth.queries(tt, nsrc * world, ntime)
    per = nsrc * ntime
    src, ts = all_src[rank * per:(rank + 1) * per], all_ts[rank * per:(rank + 1) * per]
    nq = src.size
    eng = Engine.from_timetable(tt, device=dev, kernel="auto", subtrips=args.subtrips)
    st0 = eng.stats()
    stream = torch.cuda.Stream(device=dev)
    d_src = torch.tensor(src.astype(np.int32), device=dev)
    d_ts = torch.tensor(ts.astype(np.int32), device=dev)
    d_out = torch.empty((nq, tt.num_vertices), dtype=torch.int32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.int32, device=dev)  # 256 MiB > 126 MB L2

    def step():
        eng.query_many_device(d_src, d_ts, d_out, stream=stream)

    torch.cuda.synchronize()
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = Clocks(dev)
    clocks.start()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for k in range(args.steps):
        with torch.cuda.stream(stream):
            flush.fill_(k)
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = float(sum(step_ms))
    tot_ms = _max_over_ranks(tot_ms, dev)
    value = world * nq * args.steps / (tot_ms / 1e3)

    # ---- the same batch with other sub-trip settings: none (plain Cluster-AP
    # index) and the paper's scheme 2 (r = sqrt(average trip length))
    variants = {}
    for st_alt, key in ((0, "no_subtrips_queries_per_s_per_gpu"), (2, "paper_scheme2_queries_per_s_per_gpu")):
        if st_alt == args.subtrips or not city:
            continue
        eng0 = Engine.from_timetable(tt, device=dev, kernel="auto", subtrips=st_alt)
        for _ in range(2):
            eng0.query_many_device(d_src, d_ts, d_out, stream=stream)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ms0 = 0.0
        for k in range(3):
            with torch.cuda.stream(stream):
                flush.fill_(k)
                a.record(stream)
                eng0.query_many_device(d_src, d_ts, d_out, stream=stream)
                b.record(stream)
            b.synchronize()
            ms0 += a.elapsed_time(b)
        variants[key] = nq * 3 / (ms0 / 1e3)
        eng0.close()

    # ---- e2e through the public API with host buffers: pinned host queries
    # in, every step H2D of the queries + kernel + all result rows to pinned
    # host memory (eat_query_many "direct" mode: each CTA stores its finished
    # rows into the mapped host buffer over PCIe, overlapped with the other
    # queries' relaxation; pageable buffers go through a two-stream pipeline)
    from paper_1912_00966_b200 import pinned_empty

    h_out = pinned_empty((nq, tt.num_vertices))
    h_src, h_ts = pinned_empty((nq,)), pinned_empty((nq,))
    h_src[:] = src
    h_ts[:] = ts
    e2e_steps = max(1, min(args.steps, 5))
    eng.query_many(h_src, h_ts, out=h_out)  # warm-up (buffers)
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        eng.query_many(h_src, h_ts, out=h_out)
    e2e_s = time.perf_counter() - t0
    e2e_ok = bool(np.array_equal(h_out[:64].view(np.int32), d_out[:64].cpu().numpy()))
    e2e_s = _max_over_ranks(e2e_s, dev)
    e2e_value = world * nq * e2e_steps / e2e_s

    # ---- single-query latency (BASELINE configs[1]: s=0, t_s=06:00)
    s1, t1 = synth.SINGLE_QUERY
    o1 = torch.empty(tt.num_vertices, dtype=torch.int32, device=dev)
    single = {}
    for kname in (("cta", "frontier") if city else ()):
        e1 = Engine.from_timetable(tt, device=dev, kernel=kname, subtrips=args.subtrips)
        for _ in range(3):
            e1.query_device(s1, t1, o1, stream=stream)
        stream.synchronize()
        reps = 20
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            e1.query_device(s1, t1, o1, stream=stream)
        b.record(stream)
        b.synchronize()
        single[kname] = {"ms": a.elapsed_time(b) / reps, "sweeps": e1.stats()["last_sweeps"]}
        e1.close()

    # ---- algorithmic bytes of the batched kernel (counters from an instrumented run)
    roof = _batch_roofline(tt, src, ts, dev, args, step_ms, st0)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = _cpu_baseline(tt, src, ts, args.cpu_seconds)

    if rank == 0:
        resolved = _resolved(tt, ts) * world * args.steps
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": wl_desc,
                       "stops": tt.num_vertices, "edges": st0["num_edges"], "connections": tt.num_connections,
                       "types": st0["num_types"], "queries_per_gpu": nq, "parallelism": f"query-sharded x{world}",
                       "l2": "flushed (256 MiB write) between timed steps",
                       "kernel": "cta (batched)" if st0["cta_grid"] > 0 else "grid groups (k_query_groups, frontier)",
                       "subtrips": args.subtrips, "window_s": 1200 if st0["cta_grid"] > 0 else None,
                       "cta_threads": 256 if st0["cta_grid"] > 0 else None,
                       "shortcuts": st0["num_shortcuts"]},
            "connections_resolved_per_s": resolved / (tot_ms / 1e3),
            "variants": variants,
            "single_query_ms": {k: v["ms"] for k, v in single.items()},
            "single_query_sweeps": {k: v["sweeps"] for k, v in single.items()},
            "single_query_config": "city, s=0, t_s=06:00 (BASELINE configs[1]), device time per query" if city else None,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(nq * 8),
                    "d2h_bytes_per_step": int(nq * tt.num_vertices * 4), "host_buffers": "pinned",
                    "rows_match_device_run": e2e_ok},
            "gpu_launches": args.steps,
            "clocks": clk,
            "roofline": roof,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-queries", type=int, default=200)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--subtrips", type=int, default=3,
                    help="sub-trip shortcuts (PAPER.md:342-354): 0 off, 1 r=sqrt(k) per trip, 2 r=sqrt(avg) "
                         "(the paper's scheme 2), >=3 fixed r (default 3: +3 %% q/s over scheme 2 on B200, "
                         "profiles/r01_sweep_subtrips_r.jsonl)")
    ap.add_argument("--workload", default="city_batch", choices=sorted(BATCH_WORKLOADS) + sorted(SINGLE_WORKLOADS))
    ap.add_argument("--exchange", default="allreduce", choices=["allreduce", "peer"],
                    help="country_part: per-round NCCL min-allreduce of e[] (BASELINE configs[4]) or the in-kernel "
                         "peer exchange over NVLink (NEXT-2, CUDA IPC between the ranks)")
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
