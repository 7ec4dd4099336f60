"""Multi-GPU plumbing (one process per GPU, torch.distributed) for the two
partitionings of the north star:

* query-parallel (e1): independent queries are split into contiguous shards,
  one per rank, with no data-path collective (``shard_range``,
  ``query_many_sharded``);
* edge-partitioned single query (e2): every rank builds the index slice of
  its vertex range and libeat exchanges e[] with an NCCL min-allreduce per
  round; the NCCL unique id is created on rank 0 and broadcast over the
  torch.distributed group (``edge_partitioned_engine``);
* edge-partitioned with the in-kernel exchange (NEXT-2): the ranks' exchange
  blocks are mapped into each other's address space with CUDA IPC handles
  all-gathered over the torch.distributed group, and the query kernel lowers
  remote vertices with peer atomics (``peer_partitioned_engine``).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np


def shard_range(n: int, rank: int, world: int):
    """Contiguous, balanced shard [lo, hi) of n items for `rank` of `world`."""
    lo = n * rank // world
    hi = n * (rank + 1) // world
    return lo, hi


def query_many_sharded(solve: Callable[[np.ndarray, np.ndarray], np.ndarray], sources, times, group=None,
                       gather: bool = True) -> Optional[np.ndarray]:
    """Solve this rank's shard with ``solve(src, ts) -> [k, |V|]`` (e.g.
    ``Engine.query_many``); optionally all-gather the full [nq, |V|] result
    (row order = query order).  Works on any backend (gloo for CPU tests)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    src = np.asarray(sources, np.uint32)
    ts = np.asarray(times, np.uint32)
    lo, hi = shard_range(src.size, rank, world)
    part = solve(src[lo:hi], ts[lo:hi])
    if not gather or world == 1:
        return part if world == 1 or not gather else None
    nv = part.shape[1] if part.ndim == 2 and part.shape[0] else None
    # shards may be empty on some ranks: exchange |V| first
    t_nv = torch.tensor([nv if nv is not None else -1], dtype=torch.int64)
    all_nv = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(all_nv, t_nv, group=group)
    nv = max(int(x.item()) for x in all_nv)
    # all_gather needs equal shapes: pad every shard to the largest one
    sizes = [shard_range(src.size, r, world) for r in range(world)]
    most = max(b - a for a, b in sizes)
    rows = [torch.zeros((most, nv), dtype=torch.int64) for _ in range(world)]
    mine = torch.zeros((most, nv), dtype=torch.int64)
    mine[:hi - lo] = torch.from_numpy(part.astype(np.int64).reshape(hi - lo, nv))
    dist.all_gather(rows, mine, group=group)
    return torch.cat([rows[r][:b - a] for r, (a, b) in enumerate(sizes)]).numpy().astype(np.uint32)


def nccl_unique_id(group=None) -> bytes:
    """128-byte ncclUniqueId from rank 0, broadcast to all ranks."""
    import torch
    import torch.distributed as dist

    rank = dist.get_rank(group)
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        import ctypes

        nccl = ctypes.CDLL(_nccl_path())
        raw = ctypes.create_string_buffer(128)
        rc = nccl.ncclGetUniqueId(raw)
        if rc != 0:
            raise RuntimeError(f"ncclGetUniqueId failed: {rc}")
        buf = torch.frombuffer(bytearray(raw.raw), dtype=torch.uint8).clone()
    obj = [bytes(buf.numpy().tobytes())]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def _nccl_path() -> str:
    from .build_ext import nccl_dirs
    import os

    return os.path.join(nccl_dirs()[1], "libnccl.so.2")


def edge_partitioned_engine(tt, group=None, **kw):
    """Collective: every rank builds the slice of the index it owns and joins
    the NCCL communicator libeat uses for the per-round min-allreduce."""
    import torch.distributed as dist

    from .engine import Engine

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = nccl_unique_id(group) if world > 1 else None
    return Engine.from_timetable(tt, mode="edge_partitioned", part_rank=rank, part_count=world,
                                 nccl_unique_id=uid, **kw)


def exchange_peer_handles(mine: bytes, group=None) -> list:
    """All-gather every rank's exchange-block handle, in rank order."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, bytes(mine), group=group)
    return [bytes(x) for x in out]


def peer_partitioned_engine(tt, group=None, **kw):
    """Collective: every rank builds the slice it owns with the peer exchange
    (EAT_EXCHANGE_PEER), exports its block handle, all-gathers the handles
    and maps the other ranks' blocks.  Queries are collective afterwards."""
    import torch.distributed as dist

    from .engine import Engine

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    eng = Engine.from_timetable(tt, mode="edge_partitioned", part_rank=rank, part_count=world, exchange="peer",
                                multiprocess=True, **kw)
    if world > 1:
        eng.peer_connect(exchange_peer_handles(eng.peer_export(), group))
    return eng
