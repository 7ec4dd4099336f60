/*
 * eat.h -- C ABI of libeat.so, the B200 earliest-arrival-time (EAT) engine.
 *
 * Method: arXiv 1912.00966, Haryan et al., "GPU Algorithm for Earliest
 * Arrival Time Problem in Public Transport Networks".
 *   - Problem: given connections (u, v, t, lambda), a
 *     source s and a start time t_s, the earliest arrival time e[v] at every
 *     vertex over time-respecting paths that leave s at or after t_s.
 *   - Method: topology-driven relaxation sweeps.
 *     Each sweep takes, for every connection type C_{u,v,lambda}
 *     whose source u is active, the first departure >= e[u] through the
 *     Cluster-AP hybrid rule (hour clusters + arithmetic progressions +
 *     "first connection of the next non-empty cluster", PAPER.md:300-306,
 *     Algorithm 6) and applies atomicMin to e[v]
 *     (PAPER.md:403-409); double-buffered frontiers;
 *     sweeps repeat until no vertex improves.
 *
 * Conventions (all entry points):
 *   - Times are uint32 seconds; EAT_INF = 0x7FFFFFFF marks
 *     "unreachable" (reading R2 in DESIGN.md).  Every finite time < EAT_INF.
 *   - Vertex ids are the CALLER's ids 0..num_vertices-1 on input and output
 *     (the engine renumbers internally for locality and maps back).
 *   - Ownership: eat_build copies everything it needs; the caller may free its
 *     arrays on return.  The handle owns all host and device memory it
 *     allocates; outputs are caller-allocated.  eat_free(NULL) is a no-op.
 *   - Errors: every call returns an eat_status; no C++ exception crosses the
 *     ABI; on error outputs are left untouched (host variants) or unspecified
 *     (device variants) and eat_last_error() returns a thread-local message.
 *   - Threading: a handle is immutable after eat_build; calls on one handle
 *     are serialised by an internal mutex, and their device work too: a
 *     *_device call's stream first waits for the previous call's work on the
 *     handle (whatever its stream), host calls wait for it; distinct handles
 *     are independent.
 *   - There is no CPU fallback: every query runs in the CUDA kernels of
 *     libeat.so; without a usable CUDA device the query calls return
 *     EAT_ECUDA.
 */
#ifndef EAT_H
#define EAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EAT_INF 0x7FFFFFFFu
#define EAT_ABI_VERSION 4u

typedef enum eat_status {
    EAT_OK = 0,
    EAT_EINVAL = 1,        /* bad argument: NULL pointer, id out of range, bad option */
    EAT_ERANGE = 2,        /* a time >= EAT_INF (dep + dur, or t_s) */
    EAT_ENOMEM = 3,        /* host or device allocation failed */
    EAT_ECUDA = 4,         /* CUDA runtime error, or no CUDA device */
    EAT_ENCCL = 5,         /* NCCL error (edge-partitioned mode) */
    EAT_EUNSUPPORTED = 6,  /* option combination not supported by this build */
    EAT_ESTATE = 7         /* call not valid for this handle (e.g. host-only handle) */
} eat_status;

/* Raw timetable, structure of arrays, one entry per connection
 * (u, v, t=dep, lambda=dur).  Loops (u == v), lambda = 0
 * and duplicate connections are accepted.  Arrays are read only during
 * eat_build. */
typedef struct eat_timetable {
    uint32_t num_vertices;        /* |V| >= 1 */
    uint64_t num_connections;     /* |C| >= 0 */
    const uint32_t *u;            /* [num_connections] source vertex  (< num_vertices) */
    const uint32_t *v;            /* [num_connections] target vertex  (< num_vertices) */
    const uint32_t *dep;          /* [num_connections] departure t at u, seconds */
    const uint32_t *dur;          /* [num_connections] duration lambda, seconds; dep+dur < EAT_INF */
    const uint32_t *trip;         /* optional (NULL): trip id per connection (needed by opts.subtrips) */
    const float *xy;              /* optional (NULL): [2*num_vertices] stop coordinates */
} eat_timetable;

/* eat_build_opts.renumber: internal vertex order (a locality choice only;
 * results are returned in caller ids either way). */
enum {
    EAT_RENUMBER_AUTO = 0,        /* MORTON if xy given, else BFS */
    EAT_RENUMBER_NONE = 1,
    EAT_RENUMBER_BFS = 2,
    EAT_RENUMBER_MORTON = 3
};

/* eat_build_opts.kernel: relaxation schedule for single queries. */
enum {
    EAT_KERNEL_AUTO = 0,          /* single queries: CTA kernel for graphs of <= 2048 stops, CLUSTER when e[]
                                     and the type ranges fit the shared memory of a 16-CTA cluster (city,
                                     metro), else FRONTIER; batches: CTA when e[] fits shared memory */
    EAT_KERNEL_FRONTIER = 1,      /* grid-wide persistent kernel, worklist frontier, global arr; requested
                                     explicitly, batches also run this schedule (CTA groups, e[] in global) */
    EAT_KERNEL_FULL_SWEEP = 2,    /* grid-wide persistent kernel, every type every sweep, active bitmap */
    EAT_KERNEL_CTA = 3,           /* one CTA per query, arr in shared memory */
    EAT_KERNEL_ASYNC = 4,         /* CTA-partitioned: each CTA owns a vertex range (e[] slice in shared
                                     memory), sweeps locally to quiescence, exchanges via global atomicMin
                                     + inboxes; one grid barrier per exchange round */
    EAT_KERNEL_CONNECTION = 5,    /* ablation (NEXT-3): the paper's Connection-version, a thread per raw
                                     connection every sweep (Algorithm 4) */
    EAT_KERNEL_BITMAP = 6,        /* grid-wide persistent kernel, global arr, active-vertex bitmap scanned
                                     by warps (warp per 32-vertex word, lanes over types); no worklist */
    EAT_KERNEL_CLUSTER = 7,       /* one thread-block cluster of cluster_ctas CTAs (one per SM) per query,
                                     e[] and the frontier bitmaps distributed over the CTAs' shared memory
                                     (DSMEM: ld / atom.min / atom.or on the owner CTA), the owned sources'
                                     index staged in shared memory; asynchronous: every CTA relaxes its
                                     marked vertices on its own, termination by a pending-vertex counter
                                     (no per-sweep barrier).  Needs e[] + ranges of |V| to fit 16 CTAs */
    EAT_KERNEL_GRID_ASYNC = 8     /* the asynchronous schedule on the whole GPU: persistent cooperative grid,
                                     global e[] and marked bitmap (word w owned by CTA w mod grid), every CTA
                                     relaxes its marked vertices on its own; termination by per-CTA mark /
                                     done counters and a two-wave detector; no barrier between relaxations */
};

/* eat_build_opts.mode */
enum {
    EAT_MODE_REPLICATED = 0,      /* whole index on this device (query-parallel sharding is the caller's) */
    EAT_MODE_EDGE_PARTITIONED = 1 /* this process owns the out-edges of a vertex range; NCCL min-allreduce */
};

/* eat_build_opts.flags */
#define EAT_BUILD_HOST_ONLY 0x1u   /* compress only, no device upload: introspection (eat_index_*) */
#define EAT_BUILD_COUNTERS 0x2u    /* batched kernel runs its instrumented variant (work counters in eat_stats) */
#define EAT_BUILD_CLUSTER_SYNC 0x8u /* EAT_KERNEL_CLUSTER: synchronous sweeps (one cluster barrier per sweep, the
                                      time window) instead of the asynchronous default (results identical) */
#define EAT_BUILD_MULTIPROCESS 0x4u /* EDGE_PARTITIONED + EAT_EXCHANGE_PEER: this process is rank part_rank of
                                       part_count processes (blocks joined with eat_peer_export/connect);
                                       without it all part_count partitions run in this process (loopback) */

/* eat_build_opts.exchange (EDGE_PARTITIONED): how partitions share e[] */
#define EAT_EXCHANGE_ALLREDUCE 0u  /* host-driven rounds: local sweeps, then ncclAllReduce(min) of e[] ++ flag */
#define EAT_EXCHANGE_PEER 1u       /* in-kernel (NEXT-2): a lowered vertex owned elsewhere gets a system-scope
                                      atomicMin on its owner's e[] through a peer pointer plus an inbox entry;
                                      cross-partition barrier in device memory; no host round trip, no dense
                                      collective.  Loopback: all partitions as CTA groups of one launch. */
#define EAT_PEER_HANDLE_BYTES 64u  /* one rank's exported exchange-block handle (cudaIpcMemHandle_t) */

typedef struct eat_build_opts {
    uint32_t cluster_seconds;     /* hour-cluster width; 0 -> 3600; valid 1..4096 */
    uint32_t renumber;            /* EAT_RENUMBER_* */
    int32_t device;               /* CUDA device ordinal; -1 -> current device */
    uint32_t kernel;              /* EAT_KERNEL_* */
    uint32_t flags;               /* EAT_BUILD_* */
    uint32_t subwarp;             /* grid kernels (FRONTIER, edge partition): lanes per active vertex, 1,2,4,8,16,32
                                     (virtual warps; 0 -> 32 = the Warps-version);
                                     64 = warp-flattened (vertex, type) pairs with the time window */
    uint32_t mode;                /* EAT_MODE_* */
    uint32_t part_rank;           /* EDGE_PARTITIONED: this process's rank */
    uint32_t part_count;          /* EDGE_PARTITIONED: number of ranks (1 = single partition) */
    const void *nccl_unique_id;   /* EDGE_PARTITIONED with part_count > 1: 128-byte ncclUniqueId, same on every rank */
    uint32_t window_seconds;      /* CTA-kernel schedule (and grid kernel with subwarp 64): a sweep relaxes the active vertices with
                                     e[u] <= min_active(e) + window (others stay active); EAT_INF = every
                                     active vertex (the paper's schedule); 0 -> EAT_DEFAULT_WINDOW.
                                     Results are identical for every value (same fixpoint). */
    uint32_t cta_threads;         /* batched CTA kernel threads per query: 0 -> 320; 512, 384, 320, 256, 192 or 128
                                     (occupancy knob, tools/sweep.py; 320: 5 CTAs x 10 warps per SM at 40 registers,
                                     1.4 % over 384 threads at 32, profiles/r02_ab_cta_threads_s3.jsonl) */
    uint32_t subtrips;            /* sub-trip shortcuts (needs tt->trip): 0 off;
                                     1 = r = round(sqrt(k)) per trip of k connections;
                                     2 = r = round(sqrt(average trip length)); >= 3: r itself;
                                     EAT_SUBTRIPS_HIER + r (r >= 2): blocks of r, r^2, ... (ours).
                                     Arrival times are unchanged; sweeps (hops) drop. */
    uint32_t arr_bits;            /* batched CTA kernel e[] in shared memory: 0 or 32 -> uint32 (default);
                                     16 -> uint16 offsets from t_s (twice the queries per SM; a query whose
                                     arrivals pass t_s + 65534 s is recomputed with uint32; measured slower on
                                     the city batch).  Results identical. */
    uint32_t lookup;              /* grid kernels, ablation (NEXT-3): 0 Cluster-AP;
                                     1 Connection-type-AP, Algorithm 6 over all AP tuples;
                                     2 Connection-type, linear getConnection */
    uint32_t cluster_dir;         /* cluster-record addressing: 0 auto (dense for |V| > 52k when it costs <= 3x),
                                     1 dense (record of type t, cluster k at t*y + k -- the paper's CL[y*i+j],
                                     PAPER.md:386-390: fetched in parallel with the type record),
                                     2 compact (records only for [c_first, c_last] of each type) */
    uint32_t continuation;        /* grid frontier kernel (single queries whose e[] does not fit one CTA):
                                     after a sub-warp lowers e[v] it relaxes v's types itself in the same
                                     sweep, up to this many extra vertices per frontier vertex, so a chain
                                     advances several hops per sweep (measured: metro -11 %, country -15 %
                                     at 1; deeper chains lengthen the slowest sweep).  0 = default (1),
                                     EAT_CONT_NONE = off (one hop per sweep, the paper's schedule),
                                     1..64 explicit; else EAT_EINVAL. */
    uint32_t exchange;            /* EDGE_PARTITIONED: EAT_EXCHANGE_ALLREDUCE (default) or EAT_EXCHANGE_PEER */
    uint32_t local_sweeps;        /* EDGE_PARTITIONED + ALLREDUCE: at most this many local relaxation sweeps
                                     per exchange round.  0 = sweep to local quiescence (default; fewest
                                     rounds); 1 = the north star's literal schedule, one ncclAllReduce(min) of
                                     e[] per sweep.  Results identical for every value. */
    uint32_t num_devices;         /* REPLICATED: entries in `devices` (0 or 1: the single device `device`) */
    const int32_t *devices;       /* REPLICATED with num_devices > 1: one index replica per listed CUDA device
                                     (SURVEY 8(e) e1).  eat_query_many / eat_query_many_target shard the
                                     queries in contiguous chunks, one host thread per device, each device
                                     writing its own rows (no communication).  devices[0] is the primary:
                                     every other call (single queries, *_device variants, stats) runs there.
                                     Copied at build; caller may free it after eat_build returns. */
    uint32_t cluster_ctas;        /* EAT_KERNEL_CLUSTER: CTAs per cluster, 2, 4, 8 or 16 (non-portable);
                                     0 -> the largest that the device schedules for this graph */
} eat_build_opts;

#define EAT_CONT_NONE 0xFFFFFFFFu
#define EAT_SUBTRIPS_HIER 1000u  /* eat_build_opts.subtrips: hierarchical sub-trips, base r = value - 1000 */
#define EAT_DEFAULT_WINDOW 1500u   /* seconds; city batch with sub-trips r = 3, 320-thread CTAs: 1.231M q/s vs 1.219M at 1200 s,
                                      1.229M at 1800 s, 1.195M at 900 s (profiles/r02_sweep_window_320.jsonl) */

typedef struct eat_handle eat_handle;

/* Build the compressed index (host) and upload it (device).  Steps:
 * validate; renumber; CSR of connection types by source vertex (relation R,
 * PAPER.md:225); per type, hour clusters covered by
 * greedy arithmetic progressions packed as 32-byte cluster
 * records; upload.  Untimed preprocessing, like the paper's.
 * opts may be NULL (all defaults).  EDGE_PARTITIONED with part_count > 1 is
 * collective: every rank must call it (it creates the NCCL communicator).
 * Errors: EAT_EINVAL (NULL tt/out, num_vertices == 0, id >= num_vertices,
 * bad option), EAT_ERANGE (dep + dur >= EAT_INF), EAT_ENOMEM, EAT_ECUDA,
 * EAT_ENCCL. */
eat_status eat_build(const eat_timetable *tt, const eat_build_opts *opts, eat_handle **out);

/* One query (s, t_s) -> out_arr[num_vertices] (host memory), caller ids.
 * out_arr[s] = t_s; unreachable vertices get EAT_INF (PAPER.md:58-59,
 * Algorithm 2).  Copies the result device->host.
 * Errors: EAT_EINVAL (s >= num_vertices, NULL out), EAT_ERANGE
 * (t_s >= EAT_INF), EAT_ESTATE (host-only handle), EAT_ECUDA, EAT_ENCCL. */
eat_status eat_query(eat_handle *h, uint32_t s, uint32_t t_s, uint32_t *out_arr);

/* Same, device output: d_out is a device pointer [num_vertices] on the
 * handle's device; work is enqueued on `cuda_stream` (a cudaStream_t, NULL =
 * legacy default stream).  Returns after enqueue (the query's sweep count
 * becomes available in eat_get_stats after the stream completes). */
eat_status eat_query_device(eat_handle *h, uint32_t s, uint32_t t_s, uint32_t *d_out, void *cuda_stream);

/* Batched independent queries (the paper's protocol):
 * sources[i], times[i] for i < nq; out is row-major [nq][num_vertices] in
 * host memory.  Each query is solved by one CTA of the batched kernel.
 * Errors as eat_query (checked for every i before any work). */
eat_status eat_query_many(eat_handle *h, const uint32_t *sources, const uint32_t *times, uint64_t nq,
                          uint32_t *out);

/* Same, all pointers device pointers on the handle's device, enqueued on
 * cuda_stream.  Query validity (s < num_vertices, t_s < EAT_INF) is checked
 * on the device: an invalid query yields a row of EAT_INF and sets the
 * stats field `invalid_queries`. */
eat_status eat_query_many_device(eat_handle *h, const uint32_t *d_sources, const uint32_t *d_times, uint64_t nq,
                                 uint32_t *d_out, void *cuda_stream);

/* Goal-directed EAT (NEXT-4; the goal-directed variant named in PAPER.md:60,
 * 679): for i < nq, out[i] = earliest arrival time at dsts[i] for the query
 * (sources[i], times[i]), EAT_INF if unreachable.  The search is the same
 * relaxation, pruned: a vertex whose arrival is already >= the best known
 * arrival at the target is dropped (every path through it arrives later).
 * Host arrays; out has nq entries.  Errors as eat_query_many, plus EAT_EINVAL
 * for dsts[i] >= num_vertices. */
eat_status eat_query_many_target(eat_handle *h, const uint32_t *sources, const uint32_t *times,
                                 const uint32_t *dsts, uint64_t nq, uint32_t *out);

/* Same, device pointers on the handle's device, enqueued on cuda_stream;
 * invalid (s, t_s, dst) triples yield EAT_INF and count in invalid_queries. */
eat_status eat_query_many_target_device(eat_handle *h, const uint32_t *d_sources, const uint32_t *d_times,
                                        const uint32_t *d_dsts, uint64_t nq, uint32_t *d_out, void *cuda_stream);

/* Test/introspection entry point: the Cluster-AP lookup kernel alone
 * (PAPER.md:305-306 with Algorithm 6).  For i < n: d_out[i] = the smallest
 * departure >= d_bound[i] of internal connection type d_type[i], or EAT_INF.
 * Device pointers, enqueued on cuda_stream.  EAT_EINVAL if any type id is
 * out of range is NOT checked on the device: ids must be < num_types. */
eat_status eat_lookup_device(eat_handle *h, const uint32_t *d_type, const uint32_t *d_bound, uint64_t n,
                             uint32_t *d_out, void *cuda_stream);

typedef struct eat_stats {
    /* build */
    uint32_t num_vertices;
    uint32_t num_clusters;        /* max(24, ceil((max_dep+1)/cluster_seconds)) */
    uint64_t num_connections;
    uint64_t num_types;           /* connection types owned by this handle */
    uint64_t num_edges;           /* distinct (u,v) owned by this handle */
    uint64_t num_cluster_records; /* 32-byte cluster records */
    uint64_t num_items;           /* AP items (runs + singletons) */
    uint64_t num_spill_items;     /* items stored out of line */
    uint64_t index_bytes;         /* device bytes of the packed index */
    double build_ms;              /* host build wall time */
    /* last single query (valid after its stream completed) */
    uint32_t last_sweeps;         /* relaxation sweeps (incl. the final empty one) */
    uint32_t last_rounds;         /* EDGE_PARTITIONED: exchange rounds */
    uint64_t invalid_queries;     /* batched device variant: invalid (s, t_s) seen */
    uint32_t kernel;              /* EAT_KERNEL_* actually used for single queries */
    uint32_t smem_vertices_max;   /* largest |V| the CTA kernel keeps in shared memory */
    /* EAT_BUILD_COUNTERS only: cumulative work of the batched kernel since build */
    uint64_t vertex_visits;       /* active vertices processed (type_ptr pair read) */
    uint64_t type_evals;          /* 32-byte type records read */
    uint64_t cluster_reads;       /* 32-byte cluster records read (Cluster-AP lookups) */
    uint64_t spill_items_read;    /* out-of-line AP items read */
    uint64_t improvements;        /* successful atomicMin relaxations */
    uint64_t sweeps_total;        /* relaxation sweeps summed over queries */
    uint64_t num_shortcuts;       /* sub-trip shortcut connections added at build (indexed with the rest) */
    uint64_t select_cycles;       /* EAT_BUILD_COUNTERS: SM clock cycles of the CTA kernel's select phases */
    uint64_t pair_cycles;         /*   ... and of its relaxation (pair) phases, summed over queries */
    uint64_t select_loop_cycles;  /*   ... slowest warp's own work inside the select phases (rest = barrier) */
    uint64_t pair_loop_cycles;    /*   ... slowest warp's own work inside the pair phases */
    uint32_t cta_grid;            /* resident CTAs (= queries in flight) of the batched CTA kernel; 0 if e[] does not fit */
    uint32_t num_devices;         /* devices holding a replica of this handle's index (1 unless eat_build_opts.devices) */
    /* EAT_BUILD_COUNTERS only, for SURVEY 8(d)'s algorithmic bytes: */
    uint64_t edge_evals;          /* (u,v) edges evaluated: first type of each distinct target in a vertex's type list */
    uint64_t cluster_runs;        /* AP runs (count >= 2) held by the hour-cluster slots read */
    uint64_t cluster_singles;     /* single departures (leftovers) held by the hour-cluster slots read */
    uint64_t fallbacks;           /* lookups answered by the next non-empty cluster */
    uint64_t select_bits;         /* active (deferred or new) vertices examined by the CTA kernel's select phases */
    uint32_t cta_threads;         /* threads per CTA (= per query in flight) of the batched CTA kernel */
    uint32_t cluster_ctas;        /* EAT_KERNEL_CLUSTER: CTAs per cluster (0 for other kernels) */
} eat_stats;

eat_status eat_get_stats(const eat_handle *h, eat_stats *out);

/* Device self-test of the exactness assumptions behind two integer shortcuts
 * of the kernels: (1) Algorithm 6's ceil-division ceil((e - start) / diff)
 * computed in fp32 without integer fix-up, for every pair of
 * 12-bit operands (and 0 for a zero numerator), with the branch-free item
 * lookup of the single-query kernels checked against the branching one
 * (every first-term/difference pair, four run lengths, the boundary bounds);
 * (2) the hour cluster k = floor(e / cluster_seconds)
 * computed by reciprocal multiplication with this handle's
 * cluster width, for every e < 2^31.  failures[0], failures[1] receive the
 * mismatch counts (0 on a correct device).  Errors: EAT_EINVAL (NULL),
 * EAT_ESTATE (host-only handle), EAT_ECUDA. */
eat_status eat_selftest(const eat_handle *h, uint64_t *failures);

/* Measurement utility (not a step of the EAT method): read d_buf (device
 * memory, `bytes` a multiple of 16) `reps` times with 128-bit loads from a
 * grid of (SM count x 8) CTAs of 256 threads, enqueued on cuda_stream.
 * bench.py times it with CUDA events on a buffer that fits the L2 -- the
 * measured L2-resident read bandwidth is the roofline peak of the batched
 * kernel, whose index is L2-resident.  Errors: EAT_EINVAL
 * (NULL / misaligned buffer), EAT_ECUDA. */
eat_status eat_probe_read(const void *d_buf, uint64_t bytes, uint32_t reps, void *cuda_stream);

/* Introspection of the packed index (host copy), for tests and tools.
 * Layout: vertices are internal ids; perm[c] is
 * the internal id of caller vertex c.  Types of internal vertex x are
 * type_ptr[x] .. type_ptr[x+1]-1.  type_rec is [num_types][8] uint32:
 * {v, lambda, first_dep, last_dep, crec_base, c_first, u, 0}.  crec is
 * [num_cluster_records][8] uint32: {next_min, item0..item6} or a spill
 * record {next_min, 0xFFFFFFFE, pool_offset, pool_count, ...}.  Items are
 * uint32: bits 0-11 first offset in the cluster, 12-23 stride, 24-31
 * count-1; 0xFFFFFFFF = empty slot.  Any pointer may be NULL to skip it.
 * Sizes in elements are given by eat_index_sizes (type_ptr has
 * num_vertices+1 entries). */
eat_status eat_index_export(const eat_handle *h, uint32_t *perm, uint32_t *type_ptr, uint32_t *type_rec,
                            uint32_t *crec, uint32_t *pool);

/* Element counts of the (whole, unpartitioned) host index copy that
 * eat_index_export writes: types, cluster records, spilled items.  Any
 * pointer may be NULL.  Errors: EAT_EINVAL for a NULL handle. */
eat_status eat_index_sizes(const eat_handle *h, uint64_t *num_types, uint64_t *num_cluster_records,
                           uint64_t *num_pool_items);

/* EAT_EXCHANGE_PEER across processes (one per GPU), collective in this order:
 * every rank builds with EAT_BUILD_MULTIPROCESS, exports its exchange-block
 * handle (EAT_PEER_HANDLE_BYTES into handle_out), the caller all-gathers the
 * handles in rank order (e.g. torch.distributed), every rank connects with
 * the part_count handles (its own entry is ignored).  The blocks are mapped
 * with cudaIpcOpenMemHandle (NVLink peer access between GPUs; also works for
 * two processes on one device).  Queries are then collective like NCCL's:
 * every rank calls eat_query/eat_query_device with the same (s, t_s) and gets
 * the full e[].  Errors: EAT_ESTATE on a handle of another kind or a second
 * connect, EAT_EINVAL on count != part_count, EAT_ECUDA on IPC failures. */
eat_status eat_peer_export(eat_handle *h, void *handle_out);
eat_status eat_peer_connect(eat_handle *h, const void *handles, uint32_t count);

/* Internal-vertex range [*lo, *hi) whose out-types partition `rank` of
 * `count` owns in EAT_MODE_EDGE_PARTITIONED (contiguous after renumbering,
 * balanced by connection-type count).  Host-only; any handle.
 * Errors: EAT_EINVAL (NULL handle/outputs, count == 0, rank >= count). */
eat_status eat_partition_range(const eat_handle *h, uint32_t rank, uint32_t count, uint32_t *lo, uint32_t *hi);

void eat_free(eat_handle *h);
const char *eat_last_error(void);
uint32_t eat_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* EAT_H */
