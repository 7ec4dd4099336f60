"""ctypes binding of libeat.so (include/eat.h): argument marshalling only.

Every function here has the name of the C entry point it wraps; every step
of the EAT path runs inside libeat.so (host compressor + sm_100a kernels).
If libeat.so is missing the import fails loudly -- there is no fallback.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libeat.so")

EAT_INF = 0x7FFFFFFF
EAT_CONT_NONE = 0xFFFFFFFF  # eat_build_opts.continuation: no continuation (one hop per sweep)

EAT_OK, EAT_EINVAL, EAT_ERANGE, EAT_ENOMEM, EAT_ECUDA, EAT_ENCCL, EAT_EUNSUPPORTED, EAT_ESTATE = range(8)
STATUS_NAMES = ["EAT_OK", "EAT_EINVAL", "EAT_ERANGE", "EAT_ENOMEM", "EAT_ECUDA", "EAT_ENCCL",
                "EAT_EUNSUPPORTED", "EAT_ESTATE"]

EAT_RENUMBER = {"auto": 0, "none": 1, "bfs": 2, "morton": 3}
EAT_KERNEL = {"auto": 0, "frontier": 1, "full_sweep": 2, "cta": 3, "async": 4, "connection": 5, "bitmap": 6,
              "cluster": 7, "grid_async": 8}
EAT_KERNEL_NAMES = {v: k for k, v in EAT_KERNEL.items()}
EAT_MODE = {"replicated": 0, "edge_partitioned": 1}
EAT_BUILD_HOST_ONLY = 0x1
EAT_BUILD_COUNTERS = 0x2
EAT_BUILD_MULTIPROCESS = 0x4
EAT_BUILD_CLUSTER_SYNC = 0x8
EAT_EXCHANGE = {"allreduce": 0, "peer": 1}
EAT_PEER_HANDLE_BYTES = 64

# symbols include/eat.h declares (checked by tests/test_index_host.py::test_abi_symbols_exported)
EXPORTED = ["eat_build", "eat_query", "eat_query_device", "eat_query_many", "eat_query_many_device",
            "eat_query_many_target", "eat_query_many_target_device",
            "eat_lookup_device", "eat_get_stats", "eat_index_export", "eat_index_sizes", "eat_partition_range", "eat_peer_export", "eat_peer_connect", "eat_free", "eat_last_error",
            "eat_abi_version", "eat_probe_read", "eat_selftest"]

u32p = ctypes.POINTER(ctypes.c_uint32)


class eat_timetable(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_uint32), ("num_connections", ctypes.c_uint64),
                ("u", u32p), ("v", u32p), ("dep", u32p), ("dur", u32p), ("trip", u32p),
                ("xy", ctypes.POINTER(ctypes.c_float))]


class eat_build_opts(ctypes.Structure):
    _fields_ = [("cluster_seconds", ctypes.c_uint32), ("renumber", ctypes.c_uint32), ("device", ctypes.c_int32),
                ("kernel", ctypes.c_uint32), ("flags", ctypes.c_uint32), ("subwarp", ctypes.c_uint32),
                ("mode", ctypes.c_uint32), ("part_rank", ctypes.c_uint32), ("part_count", ctypes.c_uint32),
                ("nccl_unique_id", ctypes.c_void_p), ("window_seconds", ctypes.c_uint32),
                ("cta_threads", ctypes.c_uint32), ("subtrips", ctypes.c_uint32),
                ("arr_bits", ctypes.c_uint32), ("lookup", ctypes.c_uint32), ("cluster_dir", ctypes.c_uint32),
                ("continuation", ctypes.c_uint32), ("exchange", ctypes.c_uint32),
                ("local_sweeps", ctypes.c_uint32), ("num_devices", ctypes.c_uint32),
                ("devices", ctypes.POINTER(ctypes.c_int32)), ("cluster_ctas", ctypes.c_uint32)]


class eat_stats(ctypes.Structure):
    _fields_ = [("num_vertices", ctypes.c_uint32), ("num_clusters", ctypes.c_uint32),
                ("num_connections", ctypes.c_uint64), ("num_types", ctypes.c_uint64),
                ("num_edges", ctypes.c_uint64), ("num_cluster_records", ctypes.c_uint64),
                ("num_items", ctypes.c_uint64), ("num_spill_items", ctypes.c_uint64),
                ("index_bytes", ctypes.c_uint64), ("build_ms", ctypes.c_double),
                ("last_sweeps", ctypes.c_uint32), ("last_rounds", ctypes.c_uint32),
                ("invalid_queries", ctypes.c_uint64), ("kernel", ctypes.c_uint32),
                ("smem_vertices_max", ctypes.c_uint32), ("vertex_visits", ctypes.c_uint64),
                ("type_evals", ctypes.c_uint64), ("cluster_reads", ctypes.c_uint64),
                ("spill_items_read", ctypes.c_uint64), ("improvements", ctypes.c_uint64),
                ("sweeps_total", ctypes.c_uint64), ("num_shortcuts", ctypes.c_uint64),
                ("select_cycles", ctypes.c_uint64), ("pair_cycles", ctypes.c_uint64),
                ("select_loop_cycles", ctypes.c_uint64), ("pair_loop_cycles", ctypes.c_uint64),
                ("cta_grid", ctypes.c_uint32), ("num_devices", ctypes.c_uint32),
                ("edge_evals", ctypes.c_uint64), ("cluster_runs", ctypes.c_uint64),
                ("cluster_singles", ctypes.c_uint64), ("fallbacks", ctypes.c_uint64),
                ("select_bits", ctypes.c_uint64), ("cta_threads", ctypes.c_uint32),
                ("cluster_ctas", ctypes.c_uint32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class EatError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")


_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                              "(libeat has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        H = ctypes.c_void_p
        S = ctypes.c_int
        L.eat_build.argtypes = [ctypes.POINTER(eat_timetable), ctypes.POINTER(eat_build_opts), ctypes.POINTER(H)]
        L.eat_build.restype = S
        L.eat_query.argtypes = [H, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p]
        L.eat_query.restype = S
        L.eat_query_device.argtypes = [H, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
        L.eat_query_device.restype = S
        L.eat_query_many.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        L.eat_query_many.restype = S
        L.eat_query_many_device.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                            ctypes.c_void_p]
        L.eat_query_many_device.restype = S
        L.eat_query_many_target.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                            ctypes.c_void_p]
        L.eat_query_many_target.restype = S
        L.eat_query_many_target_device.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                                   ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
        L.eat_query_many_target_device.restype = S
        L.eat_lookup_device.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.c_void_p]
        L.eat_lookup_device.restype = S
        L.eat_get_stats.argtypes = [H, ctypes.POINTER(eat_stats)]
        L.eat_get_stats.restype = S
        L.eat_index_export.argtypes = [H] + [ctypes.c_void_p] * 5
        L.eat_index_export.restype = S
        L.eat_index_sizes.argtypes = [H] + [ctypes.POINTER(ctypes.c_uint64)] * 3
        L.eat_index_sizes.restype = S
        L.eat_partition_range.argtypes = [H, ctypes.c_uint32, ctypes.c_uint32, u32p, u32p]
        L.eat_partition_range.restype = S
        L.eat_peer_export.argtypes = [H, ctypes.c_void_p]
        L.eat_peer_export.restype = S
        L.eat_peer_connect.argtypes = [H, ctypes.c_void_p, ctypes.c_uint32]
        L.eat_peer_connect.restype = S
        L.eat_free.argtypes = [H]
        L.eat_free.restype = None
        L.eat_last_error.argtypes = []
        L.eat_last_error.restype = ctypes.c_char_p
        if hasattr(L, "eat_probe_read"):  # (older builds under A/B lack the ABI-3 utilities)
            L.eat_probe_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p]
            L.eat_probe_read.restype = S
        if hasattr(L, "eat_selftest"):
            L.eat_selftest.argtypes = [H, ctypes.POINTER(ctypes.c_uint64)]
            L.eat_selftest.restype = S
        L.eat_abi_version.argtypes = []
        L.eat_abi_version.restype = ctypes.c_uint32
        _lib = L
    return _lib


def check(status: int):
    if status != EAT_OK:
        raise EatError(status, (lib().eat_last_error() or b"").decode(errors="replace"))


# ---------------------------------------------------------------- same-name wrappers
def eat_build(tt: eat_timetable, opts: eat_build_opts | None) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    check(lib().eat_build(ctypes.byref(tt), ctypes.byref(opts) if opts is not None else None, ctypes.byref(h)))
    return h


def eat_query(h, s: int, t_s: int, out_ptr: int):
    check(lib().eat_query(h, s, t_s, out_ptr))


def eat_query_device(h, s: int, t_s: int, d_out: int, stream: int):
    check(lib().eat_query_device(h, s, t_s, d_out, stream))


def eat_query_many(h, src_ptr: int, ts_ptr: int, nq: int, out_ptr: int):
    check(lib().eat_query_many(h, src_ptr, ts_ptr, nq, out_ptr))


def eat_query_many_device(h, d_src: int, d_ts: int, nq: int, d_out: int, stream: int):
    check(lib().eat_query_many_device(h, d_src, d_ts, nq, d_out, stream))


def eat_query_many_target(h, src_ptr: int, ts_ptr: int, dst_ptr: int, nq: int, out_ptr: int):
    check(lib().eat_query_many_target(h, src_ptr, ts_ptr, dst_ptr, nq, out_ptr))


def eat_query_many_target_device(h, d_src: int, d_ts: int, d_dst: int, nq: int, d_out: int, stream: int):
    check(lib().eat_query_many_target_device(h, d_src, d_ts, d_dst, nq, d_out, stream))


def eat_lookup_device(h, d_type: int, d_bound: int, n: int, d_out: int, stream: int):
    check(lib().eat_lookup_device(h, d_type, d_bound, n, d_out, stream))


def eat_get_stats(h) -> eat_stats:
    st = eat_stats()
    check(lib().eat_get_stats(h, ctypes.byref(st)))
    return st


def eat_index_export(h, perm, type_ptr, type_rec, crec, pool):
    check(lib().eat_index_export(h, perm, type_ptr, type_rec, crec, pool))


def eat_index_sizes(h):
    a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    check(lib().eat_index_sizes(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def eat_partition_range(h, rank: int, count: int):
    lo, hi = ctypes.c_uint32(), ctypes.c_uint32()
    check(lib().eat_partition_range(h, rank, count, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def eat_peer_export(h) -> bytes:
    buf = ctypes.create_string_buffer(EAT_PEER_HANDLE_BYTES)
    check(lib().eat_peer_export(h, buf))
    return buf.raw


def eat_peer_connect(h, handles) -> None:
    blob = b"".join(bytes(x) for x in handles)
    if len(blob) != EAT_PEER_HANDLE_BYTES * len(handles):
        raise ValueError("every peer handle must be EAT_PEER_HANDLE_BYTES long")
    buf = ctypes.create_string_buffer(blob, len(blob))
    check(lib().eat_peer_connect(h, buf, len(handles)))


def eat_free(h):
    lib().eat_free(h)


def eat_last_error() -> str:
    return (lib().eat_last_error() or b"").decode(errors="replace")


def eat_probe_read(d_buf: int, nbytes: int, reps: int, stream: int):
    check(lib().eat_probe_read(d_buf, nbytes, reps, stream))


def eat_selftest(h):
    f = (ctypes.c_uint64 * 2)()
    check(lib().eat_selftest(h, f))
    return int(f[0]), int(f[1])


def eat_abi_version() -> int:
    return int(lib().eat_abi_version())
