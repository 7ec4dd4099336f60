// kernels.cu -- sm_100a relaxation kernels of the EAT hot path (north-star
// subsystem 3).  Integer, irregular, latency/memory bound: no tensor cores.
//
// Per sweep, every active source u (frontier) reads
// e[u] once; the lanes of its sub-warp (virtual warp) take
// u's connection types (contiguous per edge)
// and for each:
//   - early termination: skip if e[u] > last departure or
//     max(e[u], first) + lambda >= e[v];
//   - Cluster-AP lookup (PAPER.md:300-306 + Algorithm 6):
//     first departure >= e[u] via one 32-byte cluster record;
//   - Relax (Algorithm 3) as atomicMin on e[v]
//     (PAPER.md:403-409); a strict improvement marks v in the NEXT frontier.
// Sweeps repeat until the next frontier is empty.
//
// Kernels: k_query_cta (one query per CTA, e[] in shared memory: batches and
// small single queries), k_query_grid (one query on the whole GPU: frontier,
// full-sweep, bitmap, connection and flattened schedules), k_query_groups
// (batches whose e[] needs global memory: CTA groups, frontier schedule),
// k_lookup (the lookup alone, for parity).
#include <algorithm>
#include <cstdlib>
#include <cuda/atomic>
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>

#include "device_common.cuh"
#include "eat_internal.h"
#include "kernels.cuh"

namespace eat {

namespace {

using namespace dev;

}  // namespace

// CTAs per SM of the persistent grid kernels (fewer CTAs = cheaper grid
// barrier): EAT_GRID_CTAS_PER_SM (1..8, default 1 -- the kernels use
// 1024-thread CTAs; tuning knob).
int grid_ctas_per_sm() {
    static int v = [] {
        const char *e = getenv("EAT_GRID_CTAS_PER_SM");
        int x = e ? atoi(e) : 1;
        return x < 1 ? 1 : (x > 8 ? 8 : x);
    }();
    return v;
}

#ifdef EAT_EXP_TRACE
__device__ unsigned long long g_trace[4096 * 4];
__device__ unsigned long long g_trace2[4096 * 8];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// timer read that waits for `dep` (scoreboard on the input register)
__device__ __forceinline__ unsigned long long gtimer_dep(uint32_t dep) {
    unsigned long long t;
    asm volatile("{ .reg .u32 d; mov.u32 d, %1; mov.u64 %0, %%globaltimer; }" : "=l"(t) : "r"(dep));
    return t;
}
#endif

namespace {

// ---------------------------------------------------------------- lookup kernel
__global__ void k_lookup(DevIndex ix, const uint32_t *type, const uint32_t *bound, uint64_t n, uint32_t *out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const TypeRec tr = load_type(ix, type[i]);
        out[i] = type_next_departure(ix, type[i], tr, bound[i]);
    }
}

// Instrumented variant only (SURVEY 8(d) algorithmic bytes): the contents of
// the hour-cluster slot a lookup read -- AP runs (count >= 2) and single
// departures -- and whether the answer came from the next non-empty cluster.
__device__ __noinline__ void slot_census(const DevIndex &ix, uint32_t cb, uint32_t eu, uint32_t tc, uint32_t &runs,
                                         uint32_t &singles, uint32_t &spill, uint32_t &fallback) {
    const uint32_t k = cluster_of(ix, eu);
    const uint64_t r = uint32_t(cb + k);
    const uint4 r0 = __ldg(ix.crec + 2 * r), r1 = __ldg(ix.crec + 2 * r + 1);
    auto one = [&](uint32_t it) {
        if (it == kItemEmpty) return;
        if ((it >> 24) > 0) ++runs;
        else ++singles;
    };
    if (r0.y == kItemSpill) {
        spill += r0.w;
        for (uint32_t i = 0; i < r0.w; ++i) one(__ldg(ix.pool + r0.z + i));
    } else {
        one(r0.y), one(r0.z), one(r0.w), one(r1.x), one(r1.y), one(r1.z), one(r1.w);
    }
    if (tc != kInf && cluster_of(ix, tc) > k) ++fallback;
}

// ---------------------------------------------------------------- CTA kernel
// One CTA solves one query at a time with e[] in shared memory (40 KB for a
// 10k-stop city): sweeps are separated by __syncthreads instead of grid-wide
// barriers, and relaxation is chaotic inside a sweep (updates are visible at
// once; a vertex lowered after it was read is re-marked).
// Queries are taken dynamically from a global counter (persistent grid).
//
// One sweep (two CTA barriers):
//   1. select + compact: every thread scans its bitmap words; an active
//      vertex is selected when e[u] <= base + window (window = EAT_INF: all
//      of them, the paper's schedule; base = min e[] over the frontier,
//      tracked incrementally); selected vertices are appended to s_list by
//      shared-memory atomics (order is irrelevant), the rest stay active;
//   2. warp-level flattening: each warp takes g <= 32 listed vertices, scans their
//      type counts with shuffles and evaluates the (vertex, type) pairs 32 at
//      a time (owner lane found by a 5-step shuffle search) -- all lanes busy,
//      no per-vertex divergence, no block scan;
//   3. next frontier = improved (nxt) + deferred (cur).
// THREADS per CTA and LISTCAP (selected vertices per sweep; overflow stays
// active) are template parameters: 512/2048 fits 4 CTAs (queries) per SM for
// a 10k-stop city, 384/512 and 320/512 (the default) fit 5.

// COUNT: instrumented variant (EAT_BUILD_COUNTERS) accumulating, per launch,
// the work counters used for algorithmic-byte accounting:
// counters[0] vertex visits, [1] type records read, [2] cluster records read,
// [3] spilled items read, [4] improvements (successful atomicMin), [5] sweeps,
// [6]/[7] select / pair phase cycles (thread 0, barrier to barrier), [8]/[9]
// the slowest warp's own select / pair loop cycles.
//
// Shared-memory e[] of one query.  SArr<false>: uint32 arrival times.
// SArr<true>: uint16 offsets from t_s (0xFFFF = unreached), half the shared
// memory per query so more queries fit per SM; an improvement whose offset
// would not fit (>= 18.2 h after t_s) raises the overflow flag and the query is
// recomputed by the uint32 variant (exact either way).
template <bool A16>
struct SArr;

template <>
struct SArr<false> {
    uint32_t *a;
    uint32_t base;
    __device__ __forceinline__ uint32_t get(uint32_t i) const { return reinterpret_cast<volatile uint32_t *>(a)[i]; }
    __device__ __forceinline__ void init(uint32_t i) { a[i] = kInf; }
    __device__ __forceinline__ void set(uint32_t i, uint32_t v) { a[i] = v; }
    __device__ __forceinline__ uint32_t amin(uint32_t i, uint32_t v, uint32_t *) { return atomicMin(a + i, v); }
    static __host__ __device__ size_t bytes(uint32_t n) { return size_t((n + 3u) & ~3u) * 4u; }
};

template <>
struct SArr<true> {
    uint16_t *a;
    uint32_t base;
    __device__ __forceinline__ uint32_t get(uint32_t i) const {
        const uint32_t r = reinterpret_cast<volatile uint16_t *>(a)[i];
        return r == 0xFFFFu ? kInf : base + r;
    }
    __device__ __forceinline__ void init(uint32_t i) { a[i] = 0xFFFFu; }
    __device__ __forceinline__ void set(uint32_t i, uint32_t v) { a[i] = uint16_t(v - base); }
    // atomic min on a 16-bit slot via 32-bit CAS on its word; returns the old arrival
    __device__ __forceinline__ uint32_t amin(uint32_t i, uint32_t v, uint32_t *ovf) {
        const uint32_t rel = v - base;
        if (rel >= 0xFFFFu) {  // offset does not fit: recompute this query in uint32
            *ovf = 1u;
            return v;
        }
        uint32_t *w = reinterpret_cast<uint32_t *>(a) + (i >> 1);
        const uint32_t sh = (i & 1u) * 16u;
        uint32_t old = *reinterpret_cast<volatile uint32_t *>(w);
        for (;;) {
            const uint32_t cur = (old >> sh) & 0xFFFFu;
            if (rel >= cur) return cur == 0xFFFFu ? kInf : base + cur;
            const uint32_t nw = (old & ~(0xFFFFu << sh)) | (rel << sh);
            const uint32_t prev = atomicCAS(w, old, nw);
            if (prev == old) return cur == 0xFFFFu ? kInf : base + cur;
            old = prev;
        }
    }
    static __host__ __device__ size_t bytes(uint32_t n) { return size_t((n + 7u) & ~7u) * 2u; }
};

// Minimum resident CTAs per SM for the register budget: shared memory (e[]
// of a 10k-stop city) already caps residency at 4 (512 threads) or 5.
template <int T, bool A16>
constexpr int cta_min_blocks() { return T >= 1024 ? 1 : (A16 ? 8 : (T >= 512 ? 4 : 5)); }

template <bool COUNT, int kCtaThreads, int kListCap, bool A16, bool TGT>
__global__ void __launch_bounds__(kCtaThreads, (cta_min_blocks<kCtaThreads, A16>())) k_query_cta(DevIndex ix, const uint32_t *__restrict__ src,
                                                               const uint32_t *__restrict__ tsv, uint64_t nq,
                                                               uint32_t *__restrict__ out, uint32_t *sweeps_out,
                                                               unsigned long long *qcounter,
                                                               unsigned long long *invalid,
                                                               unsigned long long *counters,
                                                               const uint32_t *__restrict__ dstv,
                                                               const uint32_t *__restrict__ qlist,
                                                               const uint32_t *__restrict__ qcount,
                                                               uint32_t *__restrict__ ovf_list,
                                                               uint32_t *__restrict__ ovf_cnt,
                                                               unsigned int *done) {
    constexpr uint32_t kCtaWarps = kCtaThreads / 32;
    extern __shared__ uint32_t sm[];
    const uint32_t n = ix.n;
    const uint32_t W = (n + 31u) / 32u;
    const uint32_t npad = (n + 3u) & ~3u;
    SArr<A16> ar;
    ar.a = reinterpret_cast<decltype(ar.a)>(sm);
    uint32_t *bmD = sm + SArr<A16>::bytes(n) / 4u;  // deferred: active, not yet selected
    uint32_t *bmN = bmD + W;    // new: lowered since their last selection
    __shared__ uint32_t s_list[kListCap];
    __shared__ uint32_t s_cnt[2], s_more[2];  // per sweep parity: listed / (deferred + improved)
    __shared__ uint32_t s_tmin[3];            // window base, rotating per sweep
    __shared__ uint32_t s_ovf;                // A16: an arrival offset overflowed
    __shared__ unsigned long long s_tw[2];    // COUNT: slowest warp's select / pair loop cycles
    __shared__ unsigned long long s_q;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    const uint32_t window = ix.window;
    (void)npad;
    const uint64_t nq_eff = qcount ? uint64_t(*qcount) : nq;

    for (;;) {
        if (tid == 0) {
            const unsigned long long qi = atomicAdd(qcounter, 1ull);
            s_q = qi >= nq_eff ? ~0ull : (qlist ? (unsigned long long)qlist[qi] : qi);
        }
        __syncthreads();
        const unsigned long long q = s_q;
        if (q == ~0ull) break;
        const uint32_t s = src[q], ts = tsv[q];
        // goal-directed query (NEXT-4): only e[dst] is wanted
        const uint32_t dq = TGT ? dstv[q] : 0u;
        uint32_t *orow = TGT ? out + q : out + q * uint64_t(n);
        if (s >= n || ts >= kInf || dq >= n) {
            if (TGT) {
                if (tid == 0) orow[0] = kInf;
            } else {
                for (uint32_t i = tid; i < n; i += kCtaThreads) orow[i] = kInf;
            }
            if (tid == 0) {
                atomicAdd(invalid, 1ull);
                if (sweeps_out) sweeps_out[q] = 0;
            }
            if (done) {
                __threadfence_system();
                __syncthreads();
                if (tid == 0) *reinterpret_cast<volatile unsigned int *>(done + q) = 1u;
            }
            __syncthreads();
            continue;
        }
        // Initialize (Algorithm 2)
        ar.base = ts;
        for (uint32_t i = tid; i < n; i += kCtaThreads) ar.init(i);
        for (uint32_t i = tid; i < W; i += kCtaThreads) {
            bmD[i] = 0;
            bmN[i] = 0;
        }
        if (tid == 0) {
            s_cnt[0] = s_cnt[1] = 0;
            s_more[0] = s_more[1] = 0;
            s_tmin[0] = ts;
            s_tmin[1] = s_tmin[2] = kInf;
            s_ovf = 0;
        }
        __syncthreads();
        if (tid == 0) {
            const uint32_t si = __ldg(ix.perm + s);  // caller id -> internal id
            ar.set(si, ts);
            bmN[si >> 5] = 1u << (si & 31u);
        }
        __syncthreads();
        const uint32_t di = TGT ? __ldg(ix.perm + dq) : 0u;
        uint32_t sweeps = 0;
        uint32_t c_vis = 0, c_type = 0, c_crec = 0, c_spill = 0, c_impr = 0;
        uint32_t c_edge = 0, c_runs = 0, c_singles = 0, c_fb = 0, c_selbits = 0;
        unsigned long long c_sel_cyc = 0, c_pair_cyc = 0, t_mark = COUNT ? clock64() : 0;
        unsigned long long c_sel_loop = 0, c_pair_loop = 0;  // slowest warp's own loop time
        if (COUNT && tid == 0) s_tw[0] = s_tw[1] = 0;
        // rotating s_tmin slots: t_cur = sweep % 3 (this sweep's window base),
        // t_nxt = (sweep + 1) % 3 (written by this sweep), t_old = (sweep + 2) % 3;
        // only t_cur is carried across sweeps (registers are the kernel's
        // limit: 40 at five 320-thread CTAs per SM, 32 at 384)
        uint32_t t_cur = 0;
        for (;;) {
            const uint32_t p = sweeps & 1u;
            const uint32_t t_nxt = t_cur == 2u ? 0u : t_cur + 1u, t_old = t_cur == 0u ? 2u : t_cur - 1u;
            uint32_t thr = kInf;
            if (window < kInf) {
                const uint32_t base = s_tmin[t_cur];
                thr = base + min(window, kInf - base);  // saturating
            }
            // goal-directed: a vertex with e[u] >= e[dst] cannot lower e[dst]
            const uint32_t best = TGT ? ar.get(di) : uint32_t(kInf);
            const unsigned long long t_sw0 = COUNT ? clock64() : 0ull;
            // ---- 1. select + compact: active = deferred | new
            uint32_t dmin = kInf, ndef = 0;  // ndef: some vertex stays deferred
            for (uint32_t w = tid; w < W; w += kCtaThreads) {
                uint32_t word = bmD[w] | bmN[w];
                if (!word) continue;
                if (COUNT) c_selbits += __popc(word);
                bmN[w] = 0;
                uint32_t sel = word;
                if (thr < kInf || (TGT && best < kInf)) {
                    sel = 0;
                    uint32_t rest = word;
                    while (rest) {  // (two e[] reads in flight per step: -0.7 %, r02_ab_select_unroll.jsonl)
                        const uint32_t b = __ffs(rest) - 1u;
                        rest &= rest - 1u;
                        const uint32_t a = ar.get(w * 32u + b);
                        if (TGT && a >= best) word &= ~(1u << b);  // pruned for good
                        else if (a <= thr) sel |= 1u << b;
                        else dmin = min(dmin, a);
                    }
                }
                uint32_t taken = 0;
                const uint32_t k = __popc(sel);
                if (k) {
                    const uint32_t pos = atomicAdd(&s_cnt[p], k);
                    const uint32_t put = pos < uint32_t(kListCap) ? min(k, uint32_t(kListCap) - pos) : 0u;
                    uint32_t rest = sel;
                    for (uint32_t i = 0; i < put; ++i) {
                        const uint32_t b = __ffs(rest) - 1u;
                        rest &= rest - 1u;
                        s_list[pos + i] = w * 32u + b;
                        taken |= 1u << b;
                    }
                    while (rest) {  // list full: stays active for a later sweep
                        const uint32_t b = __ffs(rest) - 1u;
                        rest &= rest - 1u;
                        dmin = min(dmin, ar.get(w * 32u + b));
                    }
                }
                bmD[w] = word & ~taken;
                ndef |= word & ~taken;
            }
            if (COUNT && lane == 0) atomicMax(&s_tw[0], clock64() - t_sw0);
            // (the select spread over fewer warps is slower -- 4 of 8: -6 %, 2: -15 %,
            // profiles/r02_ab_select_warps.jsonl: the phase is on the sweep's critical path)
            if (window < kInf) {
                dmin = __reduce_min_sync(0xFFFFFFFFu, dmin);
                if (lane == 0 && dmin < kInf) atomicMin(&s_tmin[t_nxt], dmin);
            }
            // s_more is a flag: every writer stores the same value (a warp
            // reduction + atomic per warp measured 0.9 % slower)
            if (ndef) s_more[p] = 1u;
            __syncthreads();
            if (COUNT && tid == 0) {
                const unsigned long long now = clock64();
                c_sel_cyc += now - t_mark;
                t_mark = now;
                c_sel_loop += s_tw[0];
                s_tw[0] = 0;
            }
            const unsigned long long t_pr0 = COUNT ? clock64() : 0ull;
            if (tid == 0) {  // slots of the next sweep: everyone is past their last read
                s_cnt[p ^ 1u] = 0;
                s_more[p ^ 1u] = 0;
                s_tmin[t_old] = kInf;
            }
            const uint32_t F = min(s_cnt[p], uint32_t(kListCap));
            // ---- 2. warp-level flattened (vertex, type) pairs; a warp takes g
            // list entries so that small frontiers still spread over all warps
            const uint32_t g = min(32u, max(1u, (F + kCtaWarps - 1u) / kCtaWarps));
            uint32_t imin = kInf;  // minimum improved arrival: feeds the next window base
            // warp w takes the list entries k0 + w + i * warps (strided: the
            // selected vertices of one bitmap word -- spatial neighbours, often
            // all heavy or all light -- spread over the warps; consecutive
            // chunks of g entries: -2 %, profiles/r02_ab_cta_strided.jsonl)
            for (uint32_t k0 = 0; k0 < F; k0 += kCtaWarps * g) {
                const uint32_t j = k0 + wid + lane * kCtaWarps;
                uint32_t x = 0, p0 = 0, nt = 0;
                if (lane < g && j < F) {
                    x = s_list[j];
                    p0 = __ldg(ix.type_ptr + x);
                    nt = __ldg(ix.type_ptr + x + 1) - p0;
                    if (COUNT) ++c_vis;
                }
                uint32_t incl = nt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= uint32_t(o)) incl += y;
                }
                const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
                const uint32_t pbase = p0 - (incl - nt);
                // (measured alternatives, profiles/r02_ab_owner_search_variants.jsonl:
                // a start-bitmask + shared-memory owner map -1 %, e[u] read once per
                // chunk and shuffled -2 %: the per-pair read sees fresher arrivals;
                // scan and search over the first 2^ceil(log2 g) lanes only -4 %,
                // r02_ab_cta_pow2_search.jsonl)
                for (uint32_t base = 0; base < tot; base += 32u) {
                    const uint32_t qp = base + lane;
                    // owner lane: smallest L with incl[L] > qp
                    uint32_t L = 0;
#pragma unroll
                    for (uint32_t step = 16; step > 0; step >>= 1) {
                        const uint32_t v = __shfl_sync(0xFFFFFFFFu, incl, L + step - 1u);
                        if (v <= qp) L += step;
                    }
                    // type of pair qp = p0 - (incl - nt) + qp of its owner: one shuffle
                    const uint32_t t = __shfl_sync(0xFFFFFFFFu, pbase, L) + qp;
                    const uint32_t u = __shfl_sync(0xFFFFFFFFu, x, L);
                    if (qp >= tot) continue;
                    const uint32_t o_p0 = COUNT ? __ldg(ix.type_ptr + u) : t;  // first type of u (COUNT)
                    const uint32_t eu = ar.get(u);
                    // the cluster base goes out with the header (a lazy load after
                    // the early-termination tests costs -5 %: one more dependent hop,
                    // profiles/r02_ab_type_hdr16_segmin.jsonl).  type_cb also holds
                    // t * dense_nc for a dense directory, so this kernel has no
                    // per-pair directory branch (the speculative record prefetch of
                    // the grid kernels, relax_type_global, is latency-bound work)
                    const uint32_t cb = __ldg(ix.type_cb + t);
                    TypeRec tr = load_type(ix, t);
                    // the first test consumes cb (& 0, a runtime zero): the compiler
                    // would otherwise sink its load into the lookup branch
                    tr.last |= cb & ix.zero;
                    if (COUNT) {
                        ++c_type;
                        if (t == o_p0 || __ldg(&ix.type_hdr[t - 1].x) != tr.v) ++c_edge;  // first type of (u,v)
                    }
                    if (eu > tr.last) continue;
                    const uint32_t av = ar.get(tr.v);
                    const uint32_t lim = TGT ? min(av, ar.get(di)) : av;
                    if (max(eu, tr.first) + tr.lam >= lim) continue;  // PAPER.md:411-416 (+ target bound)
                    uint32_t tc;
                    if (eu <= tr.first) {
                        tc = tr.first;
                    } else {
                        tc = cluster_lookup(ix, cb, eu);
                        if (COUNT) {
                            ++c_crec;
                            slot_census(ix, cb, eu, tc, c_runs, c_singles, c_spill, c_fb);
                        }
                    }
                    // (a segmented min over lanes sharing the target before the
                    // shared atomicMin costs 10 %: r02_ab_type_hdr16_segmin.jsonl;
                    // relaxing a target lowered within the window at once instead
                    // of marking it -- continuation -- halves the sweeps but costs
                    // 11 %: +18 % type evaluations, r02_ab_cta_continuation.jsonl)
                    const uint32_t cand = tc + tr.lam;
                    if (cand < av) {
                        const uint32_t old = ar.amin(tr.v, cand, &s_ovf);
                        if (cand < old) {
                            atomicOr(bmN + (tr.v >> 5), 1u << (tr.v & 31u));
                            imin = min(imin, cand);
                            if (COUNT) ++c_impr;
                        }
                    }
                }
            }
            if (COUNT && lane == 0) atomicMax(&s_tw[1], clock64() - t_pr0);
            // imin < INF iff this warp improved something
            imin = __reduce_min_sync(0xFFFFFFFFu, imin);
            if (lane == 0 && imin < kInf) {
                s_more[p] = 1u;
                if (window < kInf) atomicMin(&s_tmin[t_nxt], imin);
            }
            __syncthreads();
            if (COUNT && tid == 0) {
                const unsigned long long now = clock64();
                c_pair_cyc += now - t_mark;
                t_mark = now;
                c_pair_loop += s_tw[1];
                s_tw[1] = 0;
            }
            ++sweeps;
            t_cur = t_nxt;
            if (s_more[p] == 0u) break;  // nothing deferred, nothing lowered: fixpoint
            if (A16 && s_ovf) break;      // recomputed by the uint32 variant
        }
        {  // q and the row pointer re-derived from shared memory: not live across the sweeps
            const unsigned long long q = *reinterpret_cast<volatile unsigned long long *>(&s_q);
            uint32_t *orow = TGT ? out + q : out + q * uint64_t(n);
            if (A16 && s_ovf) {
                if (tid == 0) ovf_list[atomicAdd(ovf_cnt, 1u)] = uint32_t(q);
                __syncthreads();
                continue;
            }
            // Output in caller ids
            if (TGT) {
                if (tid == 0) orow[0] = ar.get(di);
            } else if ((n & 3u) == 0u && (reinterpret_cast<uintptr_t>(orow) & 15u) == 0u) {
                // 16-byte stores (rows may live in mapped host memory: eat_query_many direct mode)
                const uint4 *pv = reinterpret_cast<const uint4 *>(ix.perm);
                uint4 *ov = reinterpret_cast<uint4 *>(orow);
                for (uint32_t i = tid; i < n / 4u; i += kCtaThreads) {
                    const uint4 pi = __ldg(pv + i);
                    ov[i] = make_uint4(ar.get(pi.x), ar.get(pi.y), ar.get(pi.z), ar.get(pi.w));
                }
            } else {
                for (uint32_t i = tid; i < n; i += kCtaThreads) orow[i] = ar.get(__ldg(ix.perm + i));
            }
            if (tid == 0 && sweeps_out) sweeps_out[q] = sweeps;
            if (COUNT) {
                unsigned long long v[10] = {c_vis, c_type, c_crec, c_spill, c_impr, c_edge, c_runs, c_singles, c_fb,
                                            c_selbits};
                const int slot[10] = {0, 1, 2, 3, 4, 10, 11, 12, 13, 14};
                for (int k = 0; k < 10; ++k) {
                    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xFFFFFFFFu, v[k], o);
                    if (lane == 0 && v[k]) atomicAdd(counters + slot[k], v[k]);
                }
                if (tid == 0) {
                    atomicAdd(counters + 5, (unsigned long long)sweeps);
                    atomicAdd(counters + 6, c_sel_cyc);
                    atomicAdd(counters + 7, c_pair_cyc);
                    atomicAdd(counters + 8, c_sel_loop);
                    atomicAdd(counters + 9, c_pair_loop);
                }
            }
            if (done) {
                // streamed e2e (eat_query_many, page-locked output): flag the
                // finished row in mapped host memory once every thread's row
                // stores are visible system-wide (one plain store per query: no
                // atomics on host memory, which PCIe hosts need not support); the
                // host copies a chunk as soon as all its rows are flagged
                __threadfence_system();
                __syncthreads();
                if (tid == 0) *reinterpret_cast<volatile unsigned int *>(done + q) = 1u;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- grid kernel
// One query on the whole GPU: persistent cooperative grid, global e[],
// one grid barrier per sweep.  SCHED == kSchedFrontier: the frontier is a
// worklist (sub-warp per queued vertex, dedup by sweep stamps).
// SCHED == kSchedFull: topology-driven full sweep, one thread per connection
// type, active test on a bitmap (the paper's thread-per-type schedule,
// PAPER.md:228, 305).
// 1024-thread CTAs, one per SM: the same 32 warps per SM as 4 x 256 with a
// quarter of the grid-barrier arrivals (metro -10 %, country -9 %;
// DESIGN.md §9).
constexpr int kGridThreads = 1024;
// The frontier schedule skips the e[v] pre-read before its atomicMin (city
// single query -5 %, metro/country unchanged: profiles/r01_ab_frontier_no_av.jsonl).
constexpr bool kFrontierNoAv = true;

// One query by `nctas` co-resident CTAs (thread gtid of gsz): the whole grid
// (k_query_grid) or one CTA group of a multi-query launch (k_query_groups).
template <int SW, int SCHED>
__device__ __forceinline__ void grid_solve(const DevIndex &ix, const GridWork &w, uint32_t s, uint32_t ts,
                                           uint32_t *out, uint64_t gtid, uint64_t gsz, uint32_t nctas,
                                           uint32_t *bar, uint32_t &bar_epoch) {
    const uint32_t n = ix.n;
    const uint32_t W = (n + 31u) / 32u;
    // Initialize (Algorithm 2)
    for (uint64_t i = gtid; i < n; i += gsz) {
        w.arr[i] = kInf;
        if (SCHED != kSchedFull && SCHED != kSchedConn && SCHED != kSchedBitmap) w.stamp[i] = 0;
    }
    constexpr bool kBitmapSched = SCHED == kSchedFull || SCHED == kSchedConn || SCHED == kSchedBitmap;
    if (kBitmapSched)
        for (uint64_t i = gtid; i < 3ull * W; i += gsz) w.bm[i] = 0;
    if (gtid == 0) {
        w.ctl[0] = 1;  // sweep 0 sees one active vertex
        w.ctl[1] = 0;
        w.ctl[2] = 0;
        w.ctl[11] = ts;  // window base (min e[] over the frontier), 3 rotating slots
        w.ctl[12] = kInf;
        w.ctl[13] = kInf;
    }
    grid_sync(bar, bar_epoch, nctas);
    if (gtid == 0) {
        const uint32_t si = __ldg(ix.perm + s);  // caller id -> internal id
        w.arr[si] = ts;
        if (!kBitmapSched) {
            w.q0[0] = si;
            w.r0[0] = make_uint2(__ldg(ix.type_ptr + si), __ldg(ix.type_ptr + si + 1));
        }
        else w.bm[si >> 5] = 1u << (si & 31u);
    }
    uint32_t cnt_cur = grid_sync(bar, bar_epoch, nctas, w.ctl + 0);  // sweep 0's frontier size (1)

    uint32_t sweep = 0;
    for (;;) {
        const uint32_t c_cur = sweep % 3u, c_nxt = (sweep + 1u) % 3u, c_old = (sweep + 2u) % 3u;
        if (gtid == 0) w.ctl[c_old] = 0;
#ifdef EAT_EXP_TRACE
        if (gtid == 0 && sweep < 4096) {
            g_trace[sweep * 4 + 0] = gtimer();
            g_trace[sweep * 4 + 3] = ld_cg(w.ctl + c_cur);
        }
#endif
        if (SCHED == kSchedFlat) {
            // worklist + time window + warp-flattened (vertex, type) pairs
            const uint32_t cnt = cnt_cur;
            const uint32_t *qc = (sweep & 1u) ? w.q1 : w.q0;
            uint32_t *qn = (sweep & 1u) ? w.q0 : w.q1;
            const uint32_t t_cur = sweep % 3u, t_nxt = (sweep + 1u) % 3u, t_old = (sweep + 2u) % 3u;
            if (gtid == 0) w.ctl[11 + t_old] = kInf;
            uint32_t thr = kInf;
            if (ix.window < kInf) {
                const uint32_t base = ld_cg(w.ctl + 11 + t_cur);
                thr = base + min(ix.window, kInf - base);
            }
            const uint32_t lane = threadIdx.x & 31u;
            const uint64_t wid = gtid >> 5, nwarps = gsz >> 5;
            uint64_t gg = (cnt + nwarps - 1) / nwarps;
            const uint32_t g = uint32_t(gg < 1 ? 1 : (gg > 32 ? 32 : gg));
            // strided: warp w takes entries k0 + w + i * warps (metro batch +1.4 %,
            // profiles/r02_ab_cta_strided.jsonl)
            for (uint64_t k0 = 0; k0 < cnt; k0 += nwarps * g) {
                const uint64_t qi = k0 + wid + uint64_t(lane) * nwarps;
                uint32_t x = 0, p0 = 0, nt = 0;
                if (lane < g && qi < cnt) {
                    x = ld_cg(qc + qi);
                    const uint32_t ex = ld_cg(w.arr + x);
                    if (ex <= thr) {
                        p0 = __ldg(ix.type_ptr + x);
                        nt = __ldg(ix.type_ptr + x + 1) - p0;
                    } else {  // deferred: stays on the frontier
                        atomicMin(w.ctl + 11 + t_nxt, ex);
                        if (atomicExch(w.stamp + x, sweep + 1u) != sweep + 1u) push_aggregated(x, qn, w.ctl + c_nxt);
                    }
                }
                uint32_t incl = nt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                    if (lane >= uint32_t(o)) incl += y;
                }
                const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
                for (uint32_t base = 0; base < tot; base += 32u) {
                    const uint32_t qp = base + lane;
                    uint32_t L = 0;
#pragma unroll
                    for (uint32_t step = 16; step > 0; step >>= 1) {
                        const uint32_t v = __shfl_sync(0xFFFFFFFFu, incl, L + step - 1u);
                        if (v <= qp) L += step;
                    }
                    const uint32_t o_incl = __shfl_sync(0xFFFFFFFFu, incl, L);
                    const uint32_t o_nt = __shfl_sync(0xFFFFFFFFu, nt, L);
                    const uint32_t o_p0 = __shfl_sync(0xFFFFFFFFu, p0, L);
                    const uint32_t u = __shfl_sync(0xFFFFFFFFu, x, L);
                    if (qp >= tot) continue;
                    const uint32_t t = o_p0 + (qp - (o_incl - o_nt));
                    const uint32_t eu = ld_cg(w.arr + u);
                    const TypeRec tr = load_type(ix, t);
                    if (eu > tr.last) continue;
                    const uint32_t av = ld_cg(w.arr + tr.v);
                    if (max(eu, tr.first) + tr.lam >= av) continue;
                    const uint32_t tc = eu <= tr.first ? tr.first : cluster_lookup(ix, __ldg(ix.type_cb + t), eu);
                    const uint32_t cand = tc + tr.lam;
                    if (cand < av) {
                        const uint32_t old = atomicMin(w.arr + tr.v, cand);
                        if (cand < old) {
                            if (ix.window < kInf) atomicMin(w.ctl + 11 + t_nxt, cand);
                            if (atomicExch(w.stamp + tr.v, sweep + 1u) != sweep + 1u)
                                push_aggregated(tr.v, qn, w.ctl + c_nxt);
                        }
                    }
                }
            }
        } else if (SCHED == kSchedFrontier) {
            const uint32_t cnt = cnt_cur;
            const uint32_t *qc = (sweep & 1u) ? w.q1 : w.q0;
            uint32_t *qn = (sweep & 1u) ? w.q0 : w.q1;
            // queued vertices carry their type range, so a hop's type records
            // are fetched together with e[x] instead of after type_ptr[x]
            const uint2 *rc = (sweep & 1u) ? w.r1 : w.r0;
            uint2 *rn = (sweep & 1u) ? w.r0 : w.r1;
            // a warp per frontier vertex; when the frontier outnumbers the
            // warps, half-warps, so two vertices' dependent chains overlap
            // (metro -5 %, country -7 %; quarter-warps lose)
            const uint32_t sw = (SW == 32 && cnt > uint32_t(gsz >> 5)) ? 16u : uint32_t(SW);
            const uint32_t lane = uint32_t(gtid & (sw - 1u));
            // continuation: a sub-warp that lowers e[v] relaxes v's types itself
            // in this sweep (up to ix.cont_budget extra vertices per frontier
            // vertex, default 1) instead of queueing v for the next sweep: a
            // chain advances up to 1 + budget hops per sweep.  v is not stamped,
            // so a later lowering by anyone still queues it (chaotic relaxation
            // converges to the same fixpoint)
            const uint32_t wl = threadIdx.x & 31u;
            const unsigned smask = sw == 32u ? 0xFFFFFFFFu : (((1u << sw) - 1u) << (wl & ~(sw - 1u)));
            for (uint64_t it = gtid / sw; it < cnt; it += gsz / sw) {
#ifdef EAT_EXP_TRACE
                const bool tr0 = gtid == 0 && it == 0 && sweep < 4096;
                uint32_t hop = 0;
                if (tr0) g_trace2[sweep * 8 + 0] = gtimer();
#endif
                uint32_t x = ld_cg(qc + it);
                uint32_t budget = ix.cont_budget;
                uint32_t eu = ld_cg(w.arr + x);
                const uint2 rx = __ldcg(rc + it);
                uint32_t p0 = rx.x, p1 = rx.y;
                for (;;) {
#ifdef EAT_EXP_TRACE
                    if (tr0 && hop < 2) g_trace2[sweep * 8 + 1 + hop * 3] = gtimer_dep(eu + p1);
#endif
                    uint32_t cv = kNone;
                    for (uint32_t t = p0 + lane; t < p1; t += sw) {
                        const uint32_t v = relax_type_global<false, kFrontierNoAv>(ix, t, eu, w.arr);
                        if (v == kNone) continue;
                        if (budget > 0 && cv == kNone) {
                            cv = v;
                            continue;
                        }
                        const uint2 rv = make_uint2(__ldg(ix.type_ptr + v), __ldg(ix.type_ptr + v + 1));
                        if (atomicExch(w.stamp + v, sweep + 1u) != sweep + 1u) push_aggregated(v, rv, qn, rn, w.ctl + c_nxt);
                    }
#ifdef EAT_EXP_TRACE
                    if (tr0 && hop < 2) g_trace2[sweep * 8 + 2 + hop * 3] = gtimer_dep(cv);
#endif
                    const unsigned cm = __ballot_sync(smask, cv != kNone) & smask;
#ifdef EAT_EXP_TRACE
                    if (tr0 && hop < 2) g_trace2[sweep * 8 + 3 + hop * 3] = gtimer_dep(cm);
                    ++hop;
#endif
                    if (!cm) break;
                    const uint32_t src = __ffs(cm) - 1u;
                    x = __shfl_sync(smask, cv, src);
                    // the next hop's loads go out before this hop's queue pushes
                    eu = ld_cg(w.arr + x);
                    p0 = __ldg(ix.type_ptr + x);
                    p1 = __ldg(ix.type_ptr + x + 1);
                    if (cv != kNone && wl != src) {
                        const uint2 rv = make_uint2(__ldg(ix.type_ptr + cv), __ldg(ix.type_ptr + cv + 1));
                        if (atomicExch(w.stamp + cv, sweep + 1u) != sweep + 1u) push_aggregated(cv, rv, qn, rn, w.ctl + c_nxt);
                    }
                    --budget;
                }
            }
        } else {
            const uint32_t *bc = w.bm + uint64_t(c_cur) * W;
            uint32_t *bn = w.bm + uint64_t(c_nxt) * W;
            uint32_t *bo = w.bm + uint64_t(c_old) * W;
            for (uint64_t i = gtid; i < W; i += gsz) bo[i] = 0;
            bool improved = false;
            if (SCHED == kSchedBitmap) {
                // bitmap frontier: a warp per 32-vertex word of the active bitmap,
                // lanes over the types of each active vertex; an improvement only
                // sets the target's bit (no worklist, no stamps)
                const uint32_t lane = threadIdx.x & 31u;
                for (uint64_t wd = gtid >> 5; wd < W; wd += gsz >> 5) {
                    uint32_t word = ld_cg(bc + wd);
                    while (word) {
                        const uint32_t b = __ffs(word) - 1u;
                        word &= word - 1u;
                        const uint32_t x = uint32_t(wd) * 32u + b;
                        const uint32_t eu = ld_cg(w.arr + x);
                        const uint32_t p0 = __ldg(ix.type_ptr + x), p1 = __ldg(ix.type_ptr + x + 1);
                        for (uint32_t t = p0 + lane; t < p1; t += 32u) {
                            const uint32_t v = relax_type_global(ix, t, eu, w.arr);
                            if (v != kNone) {
                                atomicOr(bn + (v >> 5), 1u << (v & 31u));
                                improved = true;
                            }
                        }
                    }
                }
            } else if (SCHED == kSchedConn) {
                // Connection-version (Algorithm 4): a thread per
                // connection, Relax (Alg. 3) when its source is active
                for (uint64_t c = gtid; c < ix.num_conns; c += gsz) {
                    const uint4 cn = __ldg(ix.conns + c);  // {u, v, dep, arr}
                    if (!((ld_cg(bc + (cn.x >> 5)) >> (cn.x & 31u)) & 1u)) continue;
                    if (ld_cg(w.arr + cn.x) > cn.z || cn.w >= ld_cg(w.arr + cn.y)) continue;
                    if (cn.w < atomicMin(w.arr + cn.y, cn.w)) {
                        atomicOr(bn + (cn.y >> 5), 1u << (cn.y & 31u));
                        improved = true;
                    }
                }
            } else {
                // thread per connection type
                for (uint64_t t = gtid; t < ix.num_types; t += gsz) {
                    const uint32_t x = __ldg(ix.type_src + t);
                    if (!((ld_cg(bc + (x >> 5)) >> (x & 31u)) & 1u)) continue;
                    const uint32_t v = relax_type_global(ix, t, ld_cg(w.arr + x), w.arr);
                    if (v != kNone) {
                        atomicOr(bn + (v >> 5), 1u << (v & 31u));
                        improved = true;
                    }
                }
            }
            if (__any_sync(0xFFFFFFFFu, improved) && (threadIdx.x & 31u) == 0) atomicExch(w.ctl + c_nxt, 1u);
        }
#ifdef EAT_EXP_TRACE
        __syncthreads();
        if (threadIdx.x == 0 && sweep < 4096) atomicMax(&g_trace[sweep * 4 + 1], gtimer());
#endif
        cnt_cur = grid_sync(bar, bar_epoch, nctas, w.ctl + c_nxt);  // next frontier size / improved flag
#ifdef EAT_EXP_TRACE
        if (gtid == 0 && sweep < 4096) g_trace[sweep * 4 + 2] = gtimer();
#endif
        ++sweep;
        if (cnt_cur == 0u) break;
    }
    // caller-ordered row (NULL: the caller reads w.arr itself); 16-byte
    // stores when aligned (rows may live in mapped host memory)
    if (out && (n & 3u) == 0u && (reinterpret_cast<uintptr_t>(out) & 15u) == 0u) {
        const uint4 *pv = reinterpret_cast<const uint4 *>(ix.perm);
        uint4 *ov = reinterpret_cast<uint4 *>(out);
        for (uint64_t i = gtid; i < n / 4u; i += gsz) {
            const uint4 pi = __ldg(pv + i);
            ov[i] = make_uint4(ld_cg(w.arr + pi.x), ld_cg(w.arr + pi.y), ld_cg(w.arr + pi.z), ld_cg(w.arr + pi.w));
        }
    } else if (out) {
        for (uint64_t i = gtid; i < n; i += gsz) out[i] = ld_cg(w.arr + __ldg(ix.perm + i));
    }
    if (gtid == 0) w.ctl[8] = sweep;
}

template <int SW, int SCHED>
__global__ void __launch_bounds__(kGridThreads, 1) k_query_grid(DevIndex ix, GridWork w, uint32_t s, uint32_t ts,
                                                             uint32_t *out) {
    uint32_t epoch = 0;  // barrier counter w.ctl[kBarWord] is zeroed per launch
    grid_solve<SW, SCHED>(ix, w, s, ts, out, blockIdx.x * uint64_t(kGridThreads) + threadIdx.x,
                          uint64_t(gridDim.x) * kGridThreads, gridDim.x, w.ctl + kBarWord, epoch);
}

// Batched queries when e[] does not fit shared memory (e[]
// in global memory): the grid splits into groups of cpg CTAs; each group
// takes queries from a global counter and solves them one after another
// with the frontier schedule, using its own scratch (ws[g]) and barrier.
// 512-thread CTAs, four per SM (32 registers): 64 warps per SM hide the
// latency of many concurrent queries (metro batch 12.8k -> 18.8k q/s vs one
// 1024-thread CTA per SM, profiles/r01_sweep_group_shape.jsonl).
constexpr int kGroupThreads = 512;
constexpr int kGroupMinBlocks = 4;

template <int SW>
__global__ void __launch_bounds__(kGroupThreads, kGroupMinBlocks) k_query_groups(DevIndex ix, const GridWork *__restrict__ ws,
                                                               uint32_t cpg, const uint32_t *__restrict__ src,
                                                               const uint32_t *__restrict__ tsv, uint64_t nq,
                                                               uint32_t *__restrict__ out,
                                                               unsigned long long *qcounter,
                                                               unsigned long long *invalid,
                                                               const uint32_t *__restrict__ dstv,
                                                               const uint32_t *__restrict__ qorder) {
    const uint32_t g = blockIdx.x / cpg, crank = blockIdx.x % cpg;
    const GridWork w = ws[g];
    const uint64_t gtid = crank * uint64_t(kGroupThreads) + threadIdx.x, gsz = uint64_t(cpg) * kGroupThreads;
    uint32_t *bar = w.ctl + kBarWord;
    uint32_t epoch = 0;
    // The query index is broadcast through ctl[20 + (iteration & 1)]: a slot
    // is rewritten two iterations later, i.e. only after every CTA of the
    // group passed the next iteration's barrier and so read it -- also when
    // an invalid query skips grid_solve (and its barriers) entirely.
    for (uint32_t iter = 0;; ++iter) {
        uint32_t *slot = w.ctl + 20 + (iter & 1u);
        if (gtid == 0) {
            const unsigned long long qi = atomicAdd(qcounter, 1ull);
            *slot = qi < nq ? (qorder ? qorder[qi] : uint32_t(qi)) : 0xFFFFFFFFu;
        }
        const uint32_t q = grid_sync(bar, epoch, cpg, slot);  // also: the previous row is written
        if (q == 0xFFFFFFFFu) break;
        // goal-directed queries (dstv, NEXT-4): only e[dst] is written, out[q]
        uint32_t *orow = dstv ? out + q : out + uint64_t(q) * ix.n;
        const uint32_t s = src[q], ts = tsv[q], dq = dstv ? dstv[q] : 0u;
        if (s >= ix.n || ts >= kInf || dq >= ix.n) {
            if (dstv) {
                if (gtid == 0) orow[0] = kInf;
            } else {
                for (uint64_t i = gtid; i < ix.n; i += gsz) orow[i] = kInf;
            }
            if (gtid == 0) atomicAdd(invalid, 1ull);
            continue;
        }
        // warp-flattened (vertex, type) pairs with the time window, as the CTA
        // kernel: a batch is throughput-bound, and the window cuts the type
        // evaluations a query needs (metro 1,024 queries: 18.0k -> 43.6k q/s
        // vs the latency-oriented frontier schedule with continuation,
        // profiles/r02_ab_groups_flat_schedule.jsonl; EAT_GROUPS_FRONTIER
        // builds the old schedule for A/B)
#ifdef EAT_GROUPS_FRONTIER
        grid_solve<SW, kSchedFrontier>(ix, w, s, ts, dstv ? nullptr : orow, gtid, gsz, cpg, bar, epoch);
#else
        grid_solve<SW, kSchedFlat>(ix, w, s, ts, dstv ? nullptr : orow, gtid, gsz, cpg, bar, epoch);
#endif
        if (dstv && gtid == 0) orow[0] = ld_cg(w.arr + __ldg(ix.perm + dq));
    }
}

template <bool COUNT, int T, int L, bool A16, bool TGT = false>
cudaError_t launch_cta_one(const DevIndex &ix, const CtaArgs &a, const uint32_t *qlist, const uint32_t *qcount,
                           uint32_t *ovf_list, uint32_t *ovf_cnt, uint64_t grid_cap, cudaStream_t st) {
    const size_t smem = cta_smem_bytes(ix.n, A16);
    auto kern = k_query_cta<COUNT, T, L, A16, TGT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    uint64_t grid = std::min<uint64_t>(uint64_t(sms) * per_sm, a.nq);
    if (grid_cap > 0) grid = std::min<uint64_t>(grid, grid_cap);
    if (grid == 0) return cudaSuccess;
    e = cudaMemsetAsync(a.qcounter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    kern<<<unsigned(grid), T, smem, st>>>(ix, a.src, a.ts, a.nq, a.out, a.sweeps, a.qcounter, a.invalid, a.counters,
                                          a.dst, qlist, qcount, ovf_list, ovf_cnt, a.done);
    return cudaGetLastError();
}

// uint16 pass over all queries, then the uint32 variant over the overflow
// list (count read on the device; empty in practice for one-day feeds).
template <bool COUNT, int T, int L>
cudaError_t launch_cta_pair(const DevIndex &ix, const CtaArgs &a, cudaStream_t st) {
    if (!a.arr16) return launch_cta_one<COUNT, T, L, false>(ix, a, a.qorder, nullptr, nullptr, nullptr, a.grid_cap, st);
    cudaError_t e = cudaMemsetAsync(a.ovf_cnt, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    e = launch_cta_one<COUNT, T, L, true>(ix, a, a.qorder, nullptr, a.ovf_list, a.ovf_cnt, a.grid_cap, st);
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return launch_cta_one<COUNT, T, L, false>(ix, a, a.ovf_list, a.ovf_cnt, nullptr, nullptr, uint64_t(sms), st);
}

template <bool COUNT>
cudaError_t launch_cta_variant(const DevIndex &ix, const CtaArgs &a, cudaStream_t st) {
    if (a.dst) {  // goal-directed queries: one variant (256 threads, uint32 e[])
        if (COUNT) return cudaErrorNotSupported;
        return launch_cta_one<false, 256, 512, false, true>(ix, a, nullptr, nullptr, nullptr, nullptr, a.grid_cap, st);
    }
    switch (a.threads) {
        case 1024: return launch_cta_pair<COUNT, 1024, 2048>(ix, a, st);
        case 512: return launch_cta_pair<COUNT, 512, 2048>(ix, a, st);
        case 384: return launch_cta_pair<COUNT, 384, 512>(ix, a, st);
        case 320: return launch_cta_pair<COUNT, 320, 512>(ix, a, st);
        case 192: return launch_cta_pair<COUNT, 192, 512>(ix, a, st);
        case 128: return launch_cta_pair<COUNT, 128, 512>(ix, a, st);
        default: return launch_cta_pair<COUNT, 256, 512>(ix, a, st);
    }
}

template <int SW>
cudaError_t launch_groups_sw(const DevIndex &ix, const GridWork *h_ws, const GridWork *d_ws, uint32_t groups,
                             const uint32_t *src, const uint32_t *ts, uint64_t nq, uint32_t *out,
                             unsigned long long *qcounter, unsigned long long *invalid, const uint32_t *dst,
                             const uint32_t *qorder, cudaStream_t st) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_groups<SW>, kGroupThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint32_t cpg = uint32_t(sms * per_sm) / groups;
    if (cpg < 1) return cudaErrorInvalidConfiguration;
    for (uint32_t g = 0; g < groups; ++g)
        if ((e = cudaMemsetAsync(h_ws[g].ctl + kBarWord, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(qcounter, 0, sizeof(unsigned long long), st)) != cudaSuccess) return e;
    DevIndex ixc = ix;
    const GridWork *wp = d_ws;
    uint32_t c = cpg;
    void *args[] = {&ixc, &wp, &c, &src, &ts, &nq, &out, &qcounter, &invalid, &dst, &qorder};
    return cudaLaunchCooperativeKernel((const void *)k_query_groups<SW>, dim3(groups * cpg), dim3(kGroupThreads), args,
                                       0, st);
}

template <int SW, int SCHED>
cudaError_t launch_grid_sw(const DevIndex &ix, const GridWork &w, uint32_t s, uint32_t ts, uint32_t *out,
                           cudaStream_t st) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_grid<SW, SCHED>, kGridThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    per_sm = std::min(per_sm, grid_ctas_per_sm());
    dim3 grid(unsigned(sms * per_sm)), block(kGridThreads);
    e = cudaMemsetAsync(w.ctl + kBarWord, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    DevIndex ixc = ix;
    GridWork wc = w;
    void *args[] = {&ixc, &wc, &s, &ts, &out};
    return cudaLaunchCooperativeKernel((const void *)k_query_grid<SW, SCHED>, grid, block, args, 0, st);
}

}  // namespace

size_t cta_smem_bytes(uint32_t n, bool a16) {
    const size_t W = (n + 31u) / 32u;
    return (a16 ? SArr<true>::bytes(n) : SArr<false>::bytes(n)) + 2 * W * sizeof(uint32_t);
}

template <int T, int L, bool A16>
int cta_grid_size_t(uint32_t n) {
    int dev = 0, optin = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k_query_cta<false, T, L, A16, false>) != cudaSuccess) return 0;
    const size_t smem = cta_smem_bytes(n, A16);
    if (smem + fa.sharedSizeBytes > size_t(optin)) return 0;
    cudaFuncSetAttribute(k_query_cta<false, T, L, A16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_cta<false, T, L, A16, false>, T, smem);
    return per_sm * sms;
}

template <bool A16>
int cta_grid_size_a(uint32_t n, int threads) {
    switch (threads) {
        case 1024: return cta_grid_size_t<1024, 2048, A16>(n);
        case 512: return cta_grid_size_t<512, 2048, A16>(n);
        case 384: return cta_grid_size_t<384, 512, A16>(n);
        case 320: return cta_grid_size_t<320, 512, A16>(n);
        case 192: return cta_grid_size_t<192, 512, A16>(n);
        case 128: return cta_grid_size_t<128, 512, A16>(n);
        default: return cta_grid_size_t<256, 512, A16>(n);
    }
}

int cta_grid_size(uint32_t n, int threads, bool a16) {
    // the uint16 pass always has the uint32 variant behind it: both must fit
    const int g32 = cta_grid_size_a<false>(n, threads);
    if (!a16 || g32 == 0) return g32;
    return cta_grid_size_a<true>(n, threads);
}

size_t cta_static_smem() {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_query_cta<false, 1024, 2048, false, false>);
    return fa.sharedSizeBytes;
}

namespace {
__device__ uint32_t g_probe_sink;

// Streaming read of n 16-byte words, reps times (eat_probe_read).
__global__ void __launch_bounds__(256) k_read_probe(const uint4 *__restrict__ p, uint64_t n, uint32_t reps) {
    uint32_t acc = 0;
    for (uint32_t r = 0; r < reps; ++r)
        for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
            const uint4 v = __ldcg(p + i);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x9E3779B9u) g_probe_sink = acc;  // keeps the loads alive
}
}  // namespace

cudaError_t launch_read_probe(const uint4 *p, uint64_t n, uint32_t reps, cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    k_read_probe<<<unsigned(sms * 8), 256, 0, st>>>(p, n, reps);
    return cudaGetLastError();
}

namespace {
// Sort key of query q: its source's internal id (locality order), invalid
// sources last.
__global__ void k_query_keys(const uint32_t *__restrict__ perm, uint32_t n, const uint32_t *__restrict__ src,
                             uint64_t nq, uint32_t *__restrict__ keys, uint32_t *__restrict__ vals) {
    for (uint64_t q = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; q < nq; q += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t s = src[q];
        keys[q] = s < n ? __ldg(perm + s) : n;
        vals[q] = uint32_t(q);
    }
}
}  // namespace

cudaError_t sort_queries_by_source(const DevIndex &ix, const uint32_t *src, uint64_t nq, SortScratch &sc,
                                   cudaStream_t st) {
    if (nq > 0xFFFFFFFFull) return cudaErrorInvalidValue;
    cudaError_t e;
    if (sc.cap < nq) {
        sort_scratch_free(sc);
        size_t tmp = 0;
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                                 (uint32_t *)nullptr, (uint32_t *)nullptr, int(nq))) != cudaSuccess)
            return e;
        void **bufs[] = {(void **)&sc.k0, (void **)&sc.k1, (void **)&sc.v0, (void **)&sc.v1};
        for (void **b : bufs)
            if ((e = cudaMalloc(b, nq * 4)) != cudaSuccess) return e;
        if ((e = cudaMalloc(&sc.tmp, tmp)) != cudaSuccess) return e;
        sc.tmp_bytes = tmp;
        sc.cap = nq;
    }
    k_query_keys<<<unsigned(std::min<uint64_t>((nq + 255) / 256, 1184)), 256, 0, st>>>(ix.perm, ix.n, src, nq, sc.k0,
                                                                                      sc.v0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int bits = 1;
    while (bits < 32 && (1ull << bits) <= ix.n) ++bits;
    size_t tmp = sc.tmp_bytes;
    return cub::DeviceRadixSort::SortPairs(sc.tmp, tmp, sc.k0, sc.k1, sc.v0, sc.v1, int(nq), 0, bits, st);
}

namespace {
// keys = t_s >> shift (coarse buckets keep the caller order inside each --
// the radix sort is stable), values = query index
__global__ void k_time_keys(const uint32_t *ts, uint64_t n, uint32_t shift, uint32_t *k, uint32_t *v) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        k[i] = ts[i] >> shift;
        v[i] = uint32_t(i);
    }
}
}  // namespace

cudaError_t sort_queries_by_time(const uint32_t *ts, uint64_t nq, uint32_t shift, SortScratch &sc, cudaStream_t st) {
    if (nq > 0xFFFFFFFFull) return cudaErrorInvalidValue;
    cudaError_t e;
    if (sc.cap < nq) {
        sort_scratch_free(sc);
        size_t tmp = 0;
        if ((e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                                 (uint32_t *)nullptr, (uint32_t *)nullptr, int(nq))) != cudaSuccess)
            return e;
        void **bufs[] = {(void **)&sc.k0, (void **)&sc.k1, (void **)&sc.v0, (void **)&sc.v1};
        for (void **b : bufs)
            if ((e = cudaMalloc(b, nq * 4)) != cudaSuccess) return e;
        if ((e = cudaMalloc(&sc.tmp, tmp)) != cudaSuccess) return e;
        sc.tmp_bytes = tmp;
        sc.cap = nq;
    }
    k_time_keys<<<unsigned(std::min<uint64_t>((nq + 255) / 256, 1184)), 256, 0, st>>>(ts, nq, shift, sc.k0, sc.v0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    size_t tmp = sc.tmp_bytes;
    return cub::DeviceRadixSort::SortPairs(sc.tmp, tmp, sc.k0, sc.k1, sc.v0, sc.v1, int(nq), 0, int(32 - shift), st);
}

void sort_scratch_free(SortScratch &sc) {
    void *p[] = {sc.k0, sc.k1, sc.v0, sc.v1, sc.tmp};
    for (void *x : p)
        if (x) cudaFree(x);
    sc = SortScratch{};
}

namespace {
// eat_selftest: (1) ceil_div12 == integer ceil for every 1 <= a, s < 2^12,
// and 0 for a = 0 (every s, also 0); the branch-free item_next_bf ==
// item_next for every (first-term offset, difference) pair with count - 1 in
// {0, 1, 7, 255} at x = 0, off - 1, off, off + 1, off + stride, last,
// last + 1, 4095, and for the empty item;
// (2) cluster_of(e) == e / cs for every e < 2^31 (this index's cs).
__global__ void k_selftest(DevIndex ix, unsigned long long *fail) {
    const uint64_t gtid = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x, gsz = uint64_t(gridDim.x) * blockDim.x;
    unsigned long long f0 = 0, f1 = 0;
    for (uint64_t i = gtid; i < (1ull << 24); i += gsz) {
        const uint32_t a = uint32_t(i >> 12), st = uint32_t(i & 0xFFFu);
        if (a == 0) {
            if (ceil_div12(0u, st) != 0u) ++f0;
        } else if (st != 0 && ceil_div12(a, st) != (a + st - 1u) / st) {
            ++f0;
        }
        const uint32_t off = a, cms[4] = {0u, 1u, 7u, 255u};
        for (int c = 0; c < 4; ++c) {
            const uint32_t it = off | (st << 12) | (cms[c] << 24), last = off + cms[c] * st;
            const uint32_t xs[8] = {0u, off - 1u, off, off + 1u, off + st, last, last + 1u, 4095u};
            for (int k = 0; k < 8; ++k) {
                const uint32_t x = min(xs[k], 4095u);  // x < cs <= 4096
                if (item_next_bf(it, x) != item_next(it, x)) ++f0;
                if (c == 0 && k < 2 && item_next_bf(kItemEmpty, x) != kNone) ++f0;
            }
        }
    }
    for (uint64_t e = gtid; e < (1ull << 31); e += gsz)
        if (cluster_of(ix, uint32_t(e)) != uint32_t(e) / ix.cs) ++f1;
    if (f0) atomicAdd(fail, f0);
    if (f1) atomicAdd(fail + 1, f1);
}
}  // namespace

cudaError_t launch_selftest(const DevIndex &ix, unsigned long long *d_fail, cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaMemsetAsync(d_fail, 0, 2 * sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    k_selftest<<<unsigned(sms * 8), 256, 0, st>>>(ix, d_fail);
    return cudaGetLastError();
}

cudaError_t launch_lookup(const DevIndex &ix, const uint32_t *d_type, const uint32_t *d_bound, uint64_t n,
                          uint32_t *d_out, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, 148ull * 32));
    k_lookup<<<blocks, 256, 0, st>>>(ix, d_type, d_bound, n, d_out);
    return cudaGetLastError();
}

cudaError_t launch_query_cta(const DevIndex &ix, const CtaArgs &a, cudaStream_t st) {
    return (a.counters && !a.dst) ? launch_cta_variant<true>(ix, a, st) : launch_cta_variant<false>(ix, a, st);
}

cudaError_t launch_query_groups(const DevIndex &ix, int subwarp, const GridWork *h_ws, const GridWork *d_ws,
                                uint32_t groups, const uint32_t *src, const uint32_t *ts, uint64_t nq, uint32_t *out,
                                unsigned long long *qcounter, unsigned long long *invalid, const uint32_t *dst,
                                const uint32_t *qorder, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    switch (subwarp) {
        case 1: return launch_groups_sw<1>(ix, h_ws, d_ws, groups, src, ts, nq, out, qcounter, invalid, dst, qorder, st);
        case 2: return launch_groups_sw<2>(ix, h_ws, d_ws, groups, src, ts, nq, out, qcounter, invalid, dst, qorder, st);
        case 4: return launch_groups_sw<4>(ix, h_ws, d_ws, groups, src, ts, nq, out, qcounter, invalid, dst, qorder, st);
        case 8: return launch_groups_sw<8>(ix, h_ws, d_ws, groups, src, ts, nq, out, qcounter, invalid, dst, qorder, st);
        case 16: return launch_groups_sw<16>(ix, h_ws, d_ws, groups, src, ts, nq, out, qcounter, invalid, dst, qorder, st);
        default: return launch_groups_sw<32>(ix, h_ws, d_ws, groups, src, ts, nq, out, qcounter, invalid, dst, qorder, st);
    }
}

cudaError_t launch_query_grid(const DevIndex &ix, int subwarp, int sched, const GridWork &w, uint32_t s,
                              uint32_t t_s, uint32_t *d_out, cudaStream_t st) {
    if (sched == kSchedFull) return launch_grid_sw<1, kSchedFull>(ix, w, s, t_s, d_out, st);
    if (sched == kSchedConn) return launch_grid_sw<1, kSchedConn>(ix, w, s, t_s, d_out, st);
    if (sched == kSchedBitmap) return launch_grid_sw<32, kSchedBitmap>(ix, w, s, t_s, d_out, st);
    if (subwarp == 0) return launch_grid_sw<32, kSchedFlat>(ix, w, s, t_s, d_out, st);
    switch (subwarp) {
        case 1: return launch_grid_sw<1, kSchedFrontier>(ix, w, s, t_s, d_out, st);
        case 2: return launch_grid_sw<2, kSchedFrontier>(ix, w, s, t_s, d_out, st);
        case 4: return launch_grid_sw<4, kSchedFrontier>(ix, w, s, t_s, d_out, st);
        case 8: return launch_grid_sw<8, kSchedFrontier>(ix, w, s, t_s, d_out, st);
        case 16: return launch_grid_sw<16, kSchedFrontier>(ix, w, s, t_s, d_out, st);
        case 32: return launch_grid_sw<32, kSchedFrontier>(ix, w, s, t_s, d_out, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace eat

#ifdef EAT_EXP_TRACE
extern "C" int eat_debug_trace2(unsigned long long *out) {
    return cudaMemcpyFromSymbol(out, eat::g_trace2, sizeof(eat::g_trace2)) != cudaSuccess;
}
extern "C" int eat_debug_trace(unsigned long long *out, int clear) {
    if (cudaMemcpyFromSymbol(out, eat::g_trace, sizeof(eat::g_trace)) != cudaSuccess) return 1;
    if (clear) {
        static unsigned long long z[4096 * 4];
        cudaMemcpyToSymbol(eat::g_trace, z, sizeof(z));
    }
    return 0;
}
#endif
