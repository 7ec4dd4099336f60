// kernels.cuh -- launch interface of the sm_100a relaxation kernels (kernels.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace eat {

// Device view of the packed index (layout: eat_internal.h).
struct DevIndex {
    uint32_t n;                 // |V| (all vertices; a partition owns a sub-range of sources)
    uint32_t cs;                // cluster seconds
    uint32_t window;            // CTA schedule: process frontier vertices with e[u] <= min + window (kInf = all)
    uint32_t cta_threads;       // CTA-kernel variant: 512 (default), 384 or 256 threads per query
    uint32_t cs_magic;          // floor(2^(31+l) / cs) + 1, l = ceil(log2 cs): e / cs == (e * cs_magic) >> (31 + l)
    uint32_t cs_shift;          // 31 + l   (exact for every e < 2^31)
    uint32_t dense_nc;          // > 0: dense cluster directory, record (t, k) at t*dense_nc + k
    uint32_t lookup_mode;       // 0 Cluster-AP; ablations (grid kernels): 1 Connection-type-AP, 2 Connection-type linear
    uint32_t cont_budget;       // grid frontier kernel: extra vertices a sub-warp relaxes in the same sweep (continuation)
    uint32_t zero;              // always 0 (a value the compiler cannot fold: pins a load's issue point)
    uint64_t num_conns;         // connection-version schedule: raw connections on the device
    const uint4 *conns;         // [num_conns] {u, v, dep, arr} internal ids (EAT_KERNEL_CONNECTION only)
    uint64_t num_types;
    const uint32_t *type_ptr;   // [n+1]
    const uint4 *type_hdr;      // [T] 16-byte type headers {v, lambda, first_dep, last_dep}
    const uint32_t *type_cb;    // [T] crec_base - c_first (mod 2^32): record of cluster k is type_cb[t] + k
    const uint4 *crec;          // [2*R]  (32 B per cluster record)
    const uint32_t *pool;       // spilled items
    const uint32_t *type_src;   // [T] internal source vertex per type (full-sweep schedule)
    const uint32_t *perm;       // [n] caller id -> internal id
};

// Work counters of the instrumented (EAT_BUILD_COUNTERS) batched kernel:
// [0] vertex visits, [1] type headers read, [2] cluster slots read, [3]
// spilled items read, [4] improvements, [5] sweeps, [6]-[9] select / pair
// phase cycles (CTA kernel), [10] edge evaluations, [11] AP runs and [12]
// single departures held by the slots read, [13] next-cluster fallbacks,
// [14] active vertices examined by the select phases.
constexpr int kWorkCounters = 15;

// Control-word blocks (ctl) of the persistent kernels: kCtlWords words; the
// grid-barrier counter sits alone on the second 128-byte line (kBarWord) so
// its polling does not contend with the frontier counters' atomics.
constexpr uint32_t kCtlWords = 64;
constexpr uint32_t kBarWord = 32;

// Scratch of the grid-wide persistent single-query kernel.
struct GridWork {
    uint32_t *arr;       // [n] arrival times, internal ids
    uint32_t *q0, *q1;   // [n] frontier worklists (ping-pong)
    uint2 *r0, *r1;      // [n] type range [type_ptr[x], type_ptr[x+1]) of each queued x (frontier schedule)
    uint32_t *stamp;     // [n] "queued for sweep k" stamps (dedup)
    uint32_t *bm;        // [3*W] rotating active bitmaps (full-sweep schedule)
    uint32_t *ctl;       // [kCtlWords]: 0-2 rotating counters, 8 sweeps, 11-13 window base, kBarWord grid barrier
};

enum { kSchedFrontier = 0, kSchedFull = 1, kSchedFlat = 2, kSchedConn = 3, kSchedBitmap = 4 };

// Dynamic shared memory of the CTA kernel for n vertices (uint16 or uint32 e[]).
size_t cta_smem_bytes(uint32_t n, bool a16);

// Exactness self-test of ceil_div12 and cluster_of (eat_selftest): d_fail[0..1] mismatch counts.
cudaError_t launch_selftest(const DevIndex &ix, unsigned long long *d_fail, cudaStream_t st);

// Read-bandwidth probe (eat_probe_read): n 16-byte words, reps times.
cudaError_t launch_read_probe(const uint4 *p, uint64_t n, uint32_t reps, cudaStream_t st);

// Cluster-AP lookup for (type, bound) pairs (test entry point).
cudaError_t launch_lookup(const DevIndex &ix, const uint32_t *d_type, const uint32_t *d_bound, uint64_t n,
                          uint32_t *d_out, cudaStream_t st);

// Arguments of the CTA (one query per CTA, e[] in shared memory) kernel.
struct CtaArgs {
    const uint32_t *src = nullptr, *ts = nullptr;  // [nq] queries (caller ids / seconds)
    uint64_t nq = 0;
    uint32_t *out = nullptr;        // [nq][n] rows, or [nq] arrivals when dst != NULL
    uint32_t *sweeps = nullptr;     // optional [nq] sweep counts
    unsigned long long *qcounter = nullptr;  // 1 word, zeroed per launch (dynamic query scheduling)
    unsigned long long *invalid = nullptr;   // invalid-query counter
    unsigned long long *counters = nullptr;  // EAT_BUILD_COUNTERS work counters (instrumented variant) or NULL
    const uint32_t *dst = nullptr;  // goal-directed targets or NULL
    uint32_t *ovf_list = nullptr;   // [nq] + 1 count word (ovf_cnt): uint16-pass overflow queries
    uint32_t *ovf_cnt = nullptr;
    unsigned int *done = nullptr;   // streamed e2e: [nq] finished-row flags (mapped host memory) or NULL
    const uint32_t *qorder = nullptr;  // optional [nq]: the order in which CTAs take the queries
    int threads = 256;              // 1024, 512, 384, 320, 256, 192 or 128
    bool arr16 = false;             // uint16 pass (+ uint32 recompute of overflowing queries)
    uint64_t grid_cap = 0;
};

// One CTA per query, e[] in shared memory (kernels.cu).
cudaError_t launch_query_cta(const DevIndex &ix, const CtaArgs &a, cudaStream_t st);

// Grid-wide persistent kernel for one query with global arr (cooperative launch).
// subwarp 0: warp-flattened pairs + time window (default); 1..32: virtual warps of that width.
cudaError_t launch_query_grid(const DevIndex &ix, int subwarp, int sched, const GridWork &w, uint32_t s,
                              uint32_t t_s, uint32_t *d_out, cudaStream_t st);

// Batched queries with e[] in global memory: `groups` CTA groups of one
// cooperative launch, each with its own scratch (h_ws host copy / d_ws device
// array of GridWork), solve the nq queries (frontier schedule); row q of out,
// or out[q] = e[dst[q]] when dst != NULL (goal-directed).
// qorder (optional, [nq]): the order in which groups take the queries.
cudaError_t launch_query_groups(const DevIndex &ix, int subwarp, const GridWork *h_ws, const GridWork *d_ws,
                                uint32_t groups, const uint32_t *src, const uint32_t *ts, uint64_t nq, uint32_t *out,
                                unsigned long long *qcounter, unsigned long long *invalid, const uint32_t *dst,
                                const uint32_t *qorder, cudaStream_t st);

// Query order by source locality (k_query_groups): v1[i] = the i-th query
// when sorted by the internal id of its source (locality renumbering puts
// nearby stops at nearby ids), so the CTA groups in flight at any time
// explore overlapping parts of the index and share its L2 lines.
struct SortScratch {
    uint32_t *k0 = nullptr, *k1 = nullptr, *v0 = nullptr, *v1 = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    uint64_t cap = 0;
};
cudaError_t sort_queries_by_source(const DevIndex &ix, const uint32_t *src, uint64_t nq, SortScratch &sc,
                                   cudaStream_t st);
void sort_scratch_free(SortScratch &sc);
// Query order by departure time (batched CTA kernel): v1[i] = the i-th query
// when sorted by t_s ascending -- a later departure reaches less of the day's
// service and is cheaper (city: 21-24 h 3x cheaper), so expensive queries go
// first and the last wave of the persistent grid is short.
// shift: sort by t_s >> shift (stable: caller order inside each bucket).
cudaError_t sort_queries_by_time(const uint32_t *ts, uint64_t nq, uint32_t shift, SortScratch &sc, cudaStream_t st);

// Arguments of the cluster kernel (cluster.cu: one query per thread-block
// cluster, e[] distributed over the CTAs' shared memory).
struct ClusterArgs {
    const uint32_t *src = nullptr, *ts = nullptr;  // [nq] queries (caller ids / seconds), or NULL:
    uint32_t s1 = 0, ts1 = 0;                      // ... the single query (s1, ts1) passed by value
    uint64_t nq = 0;
    uint32_t *out = nullptr;                 // [nq][n] rows
    uint32_t *sweeps = nullptr;              // optional [nq] sweep counts
    unsigned long long *qcounter = nullptr;  // 1 word (zeroed by the launch)
    unsigned long long *invalid = nullptr;   // invalid-query counter
    int cs = 16;                             // CTAs per cluster (power of two, <= 16)
    int stage = 0;                           // index staged in shared memory: 0 none, 1 type ranges, 2 + headers
    uint32_t tl_cap = 0;                     // stage 2: most types owned by one CTA
    bool async = false;                      // no per-sweep cluster barrier (pending-vertex counter)
    uint64_t max_clusters = 0;               // 0: as many as fit
};
cudaError_t launch_query_cluster(const DevIndex &ix, const ClusterArgs &a, cudaStream_t st);

// Co-resident clusters of cs CTAs for n vertices at a staging level (0: does not fit / not schedulable).
int cluster_max_active(uint32_t n, int cs, int stage, uint32_t tl_cap, bool async);

// Scratch of the barrier-free grid kernel (gasync.cu, EAT_KERNEL_GRID_ASYNC).
constexpr uint32_t kGaCntWordsPerCta = 288;  // gasync.cu: 32 per-warp S sectors + R
struct GAsyncWork {
    uint32_t *arr;   // [n] arrival times, internal ids
    uint32_t *bm;    // [W] marked-vertex bitmap
    uint32_t *cnt;   // [kGaCntWordsPerCta * grid] per-CTA counters: S per warp (marks set), R (vertices done)
    uint32_t *ctl;   // [kCtlWords]: 0 done flag, 8 iterations of CTA 0, kBarWord grid barrier
};
// CTAs of the launch for n vertices (one per SM; 0 if the per-CTA slices do not fit shared memory).
int gasync_grid(uint32_t n);
cudaError_t launch_query_gasync(const DevIndex &ix, const GAsyncWork &w, uint32_t s, uint32_t t_s, uint32_t *d_out,
                                cudaStream_t st);

// CTAs per SM of the persistent grid kernels (env EAT_GRID_CTAS_PER_SM, default 1).
int grid_ctas_per_sm();

// Occupancy-derived grid size of the CTA kernel variant for n vertices (0 if e[] does not fit).
int cta_grid_size(uint32_t n, int threads, bool a16);

// Static shared memory of the CTA kernel (bytes).
size_t cta_static_smem();

}  // namespace eat
