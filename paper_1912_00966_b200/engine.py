"""Thin Python front end of libeat.so (argument marshalling only).

``Engine(tt, ...)`` calls ``eat_build``; ``query`` / ``query_many`` call
``eat_query`` / ``eat_query_many`` with host NumPy buffers; the ``*_device``
methods take torch CUDA tensors (PyTorch is used for device memory and
streams only).  Nothing here computes any part of the EAT path.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from . import _lib
from ._lib import EAT_INF


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


def _p(a: Optional[np.ndarray], t=ctypes.c_uint32):
    return None if a is None else a.ctypes.data_as(ctypes.POINTER(t))


def _stream_ptr(stream) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _check_tensor(t, numel: int, name: str, device: int) -> None:
    """The C ABI cannot check device buffers: refuse a tensor that is not a
    contiguous 4-byte CUDA tensor of exactly `numel` elements on `device`
    (else the kernels would read or write past its end)."""
    import torch

    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name} must be a torch CUDA tensor")
    if not t.is_cuda or (device >= 0 and t.device.index != device):
        raise ValueError(f"{name} must live on cuda:{device} (got {t.device})")
    if t.element_size() != 4 or t.dtype.is_floating_point:
        raise ValueError(f"{name} must be int32/uint32 (got {t.dtype})")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements (got {t.numel()})")


def pinned_empty(shape, dtype=np.uint32) -> np.ndarray:
    """Page-locked host array (torch pinned storage viewed as NumPy)."""
    import torch

    t = torch.empty(int(np.prod(shape)) * np.dtype(dtype).itemsize, dtype=torch.uint8, pin_memory=True)
    arr = t.numpy().view(dtype).reshape(shape)
    return arr


class Engine:
    """A built EAT index on one device (or one edge partition of it)."""

    def __init__(self, num_vertices: int, u, v, dep, dur, xy=None, *, cluster_seconds: int = 3600,
                 renumber: str = "auto", kernel: str = "auto", subwarp: int = 0, device: int = -1,
                 host_only: bool = False, counters: bool = False, mode: str = "replicated", part_rank: int = 0, part_count: int = 1,
                 nccl_unique_id: Optional[bytes] = None, window: int = 0,
                 cta_threads: int = 0, subtrips: int = 0, trip=None, arr_bits: int = 0,
                 cluster_dir: str = "auto", lookup: str = "cluster_ap", continuation: Optional[int] = None,
                 exchange: str = "allreduce", multiprocess: bool = False, local_sweeps: int = 0,
                 devices=None, cluster_ctas: int = 0, cluster_sync: bool = False):
        self._h = None
        arrs = [_u32(u), _u32(v), _u32(dep), _u32(dur)]
        m = arrs[0].shape[0]
        if any(a.shape[0] != m for a in arrs):
            raise ValueError("u, v, dep, dur must have equal length")
        xy_a = None if xy is None else np.ascontiguousarray(np.asarray(xy, dtype=np.float32).reshape(-1))
        trip_a = None if trip is None else _u32(trip)
        if trip_a is not None and trip_a.shape[0] != m:
            raise ValueError("trip must have one id per connection")
        tt = _lib.eat_timetable(num_vertices=int(num_vertices), num_connections=int(m),
                                u=_p(arrs[0]), v=_p(arrs[1]), dep=_p(arrs[2]), dur=_p(arrs[3]), trip=_p(trip_a),
                                xy=_p(xy_a, ctypes.c_float))
        self._nccl_buf = None
        if nccl_unique_id is not None:
            self._nccl_buf = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        self._devs = None
        if devices is not None and len(devices) > 1:
            self._devs = (ctypes.c_int32 * len(devices))(*[int(d) for d in devices])
            device = int(devices[0])
        opts = _lib.eat_build_opts(cluster_seconds=int(cluster_seconds), renumber=_lib.EAT_RENUMBER[renumber],
                                   device=int(device), kernel=_lib.EAT_KERNEL[kernel],
                                   flags=(_lib.EAT_BUILD_HOST_ONLY if host_only else 0)
                                   | (_lib.EAT_BUILD_COUNTERS if counters else 0)
                                   | (_lib.EAT_BUILD_MULTIPROCESS if multiprocess else 0)
                                   | (_lib.EAT_BUILD_CLUSTER_SYNC if cluster_sync else 0), subwarp=int(subwarp),
                                   mode=_lib.EAT_MODE[mode], part_rank=int(part_rank), part_count=int(part_count),
                                   nccl_unique_id=ctypes.cast(self._nccl_buf, ctypes.c_void_p) if self._nccl_buf else None,
                                   window_seconds=int(window), cta_threads=int(cta_threads),
                                   subtrips=int(subtrips), arr_bits=int(arr_bits),
                                   cluster_dir={"auto": 0, "dense": 1, "compact": 2}[cluster_dir],
                                   lookup={"cluster_ap": 0, "ap": 1, "linear": 2}[lookup],
                                   continuation=0 if continuation is None else (int(continuation) or _lib.EAT_CONT_NONE),
                                   exchange=_lib.EAT_EXCHANGE[exchange], local_sweeps=int(local_sweeps),
                                   num_devices=len(self._devs) if self._devs is not None else 0,
                                   devices=ctypes.cast(self._devs, ctypes.POINTER(ctypes.c_int32))
                                   if self._devs is not None else None, cluster_ctas=int(cluster_ctas))
        self._h = _lib.eat_build(tt, opts)
        self.device = -1 if host_only else int(device)
        if self.device < 0 and not host_only:
            import torch

            self.device = torch.cuda.current_device()
        self.num_vertices = int(num_vertices)
        self.num_connections = int(m)

    @classmethod
    def from_timetable(cls, tt, **kw) -> "Engine":
        if kw.get("subtrips") and "trip" not in kw:
            kw["trip"] = tt.trip
        return cls(tt.num_vertices, tt.u, tt.v, tt.dep, tt.dur, getattr(tt, "xy", None), **kw)

    # ------------------------------------------------------------------ lifecycle
    def close(self):
        if self._h is not None:
            _lib.eat_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ queries
    def query(self, s: int, t_s: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """e[] of one query, uint32 [|V|] in caller ids.  `out` may be a
        preallocated C-contiguous uint32 array (``pinned_empty``: the device
        writes it directly)."""
        if out is None:
            out = np.empty(self.num_vertices, dtype=np.uint32)
        elif out.shape != (self.num_vertices,) or out.dtype != np.uint32 or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a C-contiguous uint32 array of shape ({self.num_vertices},)")
        _lib.eat_query(self._h, int(s), int(t_s), out.ctypes.data)
        return out

    def query_many(self, sources, times, out: Optional[np.ndarray] = None) -> np.ndarray:
        """[nq, |V|] uint32.  `out` may be a preallocated C-contiguous uint32
        array, e.g. from ``pinned_empty`` (page-locked: rows are copied
        straight from the device; pageable memory goes through pinned staging)."""
        src, ts = _u32(sources), _u32(times)
        if src.shape != ts.shape:
            raise ValueError("sources and times must have equal length")
        shape = (src.shape[0], self.num_vertices)
        if out is None:
            out = np.empty(shape, dtype=np.uint32)
        elif out.shape != shape or out.dtype != np.uint32 or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a C-contiguous uint32 array of shape {shape}")
        _lib.eat_query_many(self._h, src.ctypes.data, ts.ctypes.data, src.shape[0], out.ctypes.data)
        return out

    def query_targets(self, sources, times, dsts) -> np.ndarray:
        """Goal-directed EAT (eat_query_many_target): arrival at dsts[i] per query."""
        src, ts, dst = _u32(sources), _u32(times), _u32(dsts)
        if not (src.shape == ts.shape == dst.shape):
            raise ValueError("sources, times and dsts must have equal length")
        out = np.empty(src.shape[0], dtype=np.uint32)
        _lib.eat_query_many_target(self._h, src.ctypes.data, ts.ctypes.data, dst.ctypes.data, src.shape[0],
                                   out.ctypes.data)
        return out

    def query_targets_device(self, sources, times, dsts, out, stream=None):
        """int32 CUDA tensors [nq]; out [nq] receives the arrival at each target."""
        nq = int(sources.numel())
        for t, nm in ((sources, "sources"), (times, "times"), (dsts, "dsts"), (out, "out")):
            _check_tensor(t, nq, nm, self.device)
        _lib.eat_query_many_target_device(self._h, sources.data_ptr(), times.data_ptr(), dsts.data_ptr(),
                                          int(sources.numel()), out.data_ptr(), _stream_ptr(stream))
        return out

    def query_device(self, s: int, t_s: int, out, stream=None):
        """out: int32/uint32 CUDA tensor [num_vertices] on this engine's device."""
        _check_tensor(out, self.num_vertices, "out", self.device)
        _lib.eat_query_device(self._h, int(s), int(t_s), out.data_ptr(), _stream_ptr(stream))
        return out

    def query_many_device(self, sources, times, out, stream=None):
        """sources, times: int32 CUDA tensors [nq]; out: int32 CUDA tensor [nq, num_vertices]."""
        nq = int(sources.numel())
        _check_tensor(sources, nq, "sources", self.device)
        _check_tensor(times, nq, "times", self.device)
        _check_tensor(out, nq * self.num_vertices, "out", self.device)
        _lib.eat_query_many_device(self._h, sources.data_ptr(), times.data_ptr(), nq, out.data_ptr(),
                                   _stream_ptr(stream))
        return out

    def lookup_device(self, types, bounds, out, stream=None):
        for t, nm in ((types, "types"), (bounds, "bounds"), (out, "out")):
            _check_tensor(t, int(types.numel()), nm, self.device)
        _lib.eat_lookup_device(self._h, types.data_ptr(), bounds.data_ptr(), int(types.numel()), out.data_ptr(),
                               _stream_ptr(stream))
        return out

    def selftest(self):
        """(ceil-div mismatches, cluster-index mismatches) on this device (eat_selftest; 0, 0 expected)."""
        return _lib.eat_selftest(self._h)

    def peer_export(self) -> bytes:
        """This rank's exchange-block handle (EAT_EXCHANGE_PEER, multiprocess)."""
        return _lib.eat_peer_export(self._h)

    def peer_connect(self, handles) -> None:
        """Map every rank's block (handles in rank order; collective)."""
        _lib.eat_peer_connect(self._h, handles)

    def partition_range(self, rank: int, count: int):
        """Internal-vertex range [lo, hi) owned by edge partition `rank` of `count`."""
        return _lib.eat_partition_range(self._h, int(rank), int(count))

    # ------------------------------------------------------------------ introspection
    def stats(self) -> dict:
        d = _lib.eat_get_stats(self._h).as_dict()
        d["kernel_name"] = _lib.EAT_KERNEL_NAMES.get(d["kernel"], "?")
        return d

    def export(self) -> dict:
        """Host copy of the packed index (layout documented in include/eat.h)."""
        n = self.num_vertices
        nt, nr, npool = _lib.eat_index_sizes(self._h)
        perm = np.empty(n, dtype=np.uint32)
        tptr = np.empty(n + 1, dtype=np.uint32)
        trec = np.empty((max(nt, 1), 8), dtype=np.uint32)
        crec = np.empty((max(nr, 1), 8), dtype=np.uint32)
        pool = np.empty(max(npool, 1), dtype=np.uint32)
        _lib.eat_index_export(self._h, perm.ctypes.data, tptr.ctypes.data, trec.ctypes.data, crec.ctypes.data,
                              pool.ctypes.data)
        return dict(perm=perm, type_ptr=tptr, type_rec=trec[:nt], crec=crec[:nr], pool=pool[:npool])
