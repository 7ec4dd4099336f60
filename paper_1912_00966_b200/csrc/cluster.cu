// cluster.cu -- EAT_KERNEL_CLUSTER: one query per thread-block cluster, e[]
// distributed over the cluster's shared memory (DSMEM).
//
// A cluster of CS CTAs (1024 threads, one CTA per SM, CS a power of two up to
// 16) solves one query at a time with the batched CTA kernel's schedule
// (kernels.cu k_query_cta: select by time window, warp-flattened (vertex,
// type) pairs, chaotic relaxation), but e[] and the two
// frontier bitmaps are spread over the CTAs' shared memory:
//   bitmap word w (vertices 32w .. 32w+31) lives in CTA  w mod CS,  local
//   word w / CS; its 32 arrival times in the same CTA.
// Interleaving by words keeps a spatially compact frontier (locality
// renumbering) spread over every CTA.  Per sweep:
//   1. select: each CTA scans its own words (local shared memory) and lists
//      the selected vertices (sources it owns);
//   2. cluster barrier (every CTA's select is done before anyone marks);
//   3. pairs: a CTA relaxes the out-types of its listed sources; e[v] is read
//      and lowered through DSMEM (ld / atom.min on the owner's shared memory,
//      215 cycles cross-CTA on Blackwell vs ~600 for an L2 hit) and v is
//      marked in the owner's bitmap (atom.or);
//   4. each CTA pushes its window-base and "more" partials into every CTA's
//      control words; cluster barrier; all CTAs read the same values.
// Two cluster barriers (~0.2 us each) per sweep instead of two grid barriers
// (1.3 us each) of the grid kernels: a single query on a mid-size graph (city,
// metro) runs on CS SMs with a much shorter per-sweep critical path.  Batches
// run one query per cluster, clusters taking queries from a counter.
// Relaxation, lookup and fixpoint are the paper's (Alg. 3/6, PAPER.md:175-306,
// atomicMin PAPER.md:403-409); only the schedule and the placement of e[]
// differ.
#include <algorithm>

#include "device_common.cuh"
#include "kernels.cuh"

namespace eat {
namespace {

using namespace dev;

constexpr int kClThreads = 1024;
constexpr uint32_t kClWarps = kClThreads / 32;
constexpr uint32_t kClListCap = 2048;

#ifndef EAT_CL_BAR1
#define EAT_CL_BAR1 0  // 1: a cluster barrier between select and pairs (-x %: cluster_trace.py)
#endif

#ifdef EAT_CL_TRACE
__device__ unsigned long long g_cltrace[1024 * 6];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

// cluster-wide barrier: all threads of all CTAs; release/acquire at cluster
// scope orders every shared (local and DSMEM) access before it
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// address of the same shared-memory location in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t cl_map(uint32_t sa, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sa), "r"(rank));
    return r;
}

__device__ __forceinline__ uint32_t cl_ld(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ void cl_st(uint32_t a, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t cl_min(uint32_t a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.min.u32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v));
    return old;
}

__device__ __forceinline__ void cl_or(uint32_t a, uint32_t v) {
    asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}

__device__ __forceinline__ uint32_t cl_or_old(uint32_t a, uint32_t v) {
    uint32_t old;
    asm volatile("atom.shared::cluster.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(a), "r"(v) : "memory");
    return old;
}

__device__ __forceinline__ void cl_redmin(uint32_t a, uint32_t v) {
    asm volatile("red.shared::cluster.min.u32 [%0], %1;" ::"r"(a), "r"(v));
}

// 32-byte cluster record r, as volatile loads (issued where written, not
// sunk into the branch that consumes them)
__device__ __forceinline__ void ldg_crec(const DevIndex &ix, uint32_t r, uint4 &r0, uint4 &r1) {
    const uint4 *p = ix.crec + 2 * uint64_t(r);
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r0.x), "=r"(r0.y), "=r"(r0.z), "=r"(r0.w) : "l"(p));
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r1.x), "=r"(r1.y), "=r"(r1.z), "=r"(r1.w)
                 : "l"(p + 1));
}

__device__ __forceinline__ uint32_t lds_volatile(const uint32_t *p) { return *reinterpret_cast<const volatile uint32_t *>(p); }

// STAGE: what of the index the CTAs keep in shared memory for their own
// sources (a CTA relaxes only the out-types of the vertices it owns):
//   0 nothing (type_ptr, headers, cluster bases from L2);
//   1 the type range (start, count) of every owned vertex;
//   2 + the 16-byte type headers and cluster bases of the owned vertices'
//     types (the paper's per-type cluster directory staged on chip,
//     PAPER.md:382-390): a relaxation then needs one global access, the
//     hour-cluster record.
// Staged once per launch (every query of the launch reuses it).
// ASYNC: no per-sweep cluster barrier at all.  Every CTA loops on its own
// (take all its marked vertices -> relax them); per CTA, S counts marks and
// R finished vertices (local shared memory): a marking warp adds its tries
// to S (and waits for the add) BEFORE setting the bits, subtracts the tries
// that lowered nothing and the marks that hit an already-set bit after, and
// R grows by the vertices a CTA took once their relaxations (and the marks
// they made) are done; an idle CTA 0 sums every R, then every S (DSMEM):
// equal sums mean nothing was marked or in processing in between (the grid
// kernel's two-wave detector, gasync.cu) -- and a fixpoint is stable.
// (Until round 2 session 3 one pending counter in CTA 0, +tries / -F: every
// marking warp's add would wait on that one contended word.)  Window: all
// active vertices.
template <int STAGE, bool ASYNC>
__global__ void __launch_bounds__(kClThreads, 1)
    k_query_cluster(DevIndex ix, const uint32_t *__restrict__ src, const uint32_t *__restrict__ tsv, uint64_t nq,
                    uint32_t *__restrict__ out, uint32_t *sweeps_out, unsigned long long *qcounter,
                    unsigned long long *invalid, uint32_t tl_cap, uint32_t s1, uint32_t ts1) {
    extern __shared__ uint4 sm4[];
    const uint32_t n = ix.n;
    uint32_t ncta;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
    const uint32_t rank = cl_rank();
    const uint32_t lg = 31u - __clz(ncta);          // CS = 2^lg
    const uint32_t W = (n + 31u) / 32u;              // bitmap words of the whole graph
    const uint32_t Wl = (W + ncta - 1u) >> lg;       // words per CTA
    // layout: hdr_s[tl_cap] | e_loc[32 Wl] | rng[32 Wl] | bmD[Wl] | bmN[Wl] | cb_s[tl_cap]
    uint4 *hdr_s = sm4;                                                   // STAGE 2
    uint32_t *e_loc = reinterpret_cast<uint32_t *>(sm4 + (STAGE == 2 ? tl_cap : 0u));  // arrivals of the owned words
    uint2 *rng = reinterpret_cast<uint2 *>(e_loc + Wl * 32u);             // STAGE >= 1
    uint32_t *bmD = reinterpret_cast<uint32_t *>(rng + (STAGE >= 1 ? Wl * 32u : 0u));  // deferred
    uint32_t *bmN = bmD + Wl;                                             // new: lowered since their last selection
    uint32_t *cb_s = bmN + Wl;                                            // STAGE 2
    uint32_t *a_list = cb_s + (STAGE == 2 ? tl_cap : 0u);                 // ASYNC: [32 Wl] every owned vertex
    __shared__ uint32_t s_list[kClListCap];
    __shared__ uint32_t s_cnt[2], s_more[2];         // per sweep parity: listed / more-work flag (cluster-wide)
    __shared__ uint32_t s_tmin[3];                   // window base, rotating (cluster-wide after the push)
    __shared__ uint32_t s_pmin[2], s_pmore[2];       // this CTA's partials of the sweep (parity)
    __shared__ uint32_t s_q[2];                      // query index (lo, hi) pushed by rank 0
    __shared__ uint32_t s_S, s_R;                    // ASYNC: marks this CTA counted / vertices it finished
    __shared__ uint32_t s_done;                      // ASYNC (CTA 0's copy is the one used): fixpoint detected
    __shared__ uint32_t s_idle;                      // ASYNC: CTA 0 raised s_done
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    const uint32_t window = ix.window;
    const uint32_t e_sa = uint32_t(__cvta_generic_to_shared(e_loc));
    const uint32_t bmN_sa = uint32_t(__cvta_generic_to_shared(bmN));
    const uint32_t more_sa = uint32_t(__cvta_generic_to_shared(s_more));
    const uint32_t tmin_sa = uint32_t(__cvta_generic_to_shared(s_tmin));
    const uint32_t q_sa = uint32_t(__cvta_generic_to_shared(s_q));
    const uint32_t S_sa = uint32_t(__cvta_generic_to_shared(&s_S)), R_sa = uint32_t(__cvta_generic_to_shared(&s_R));
    const uint32_t done0 = cl_map(uint32_t(__cvta_generic_to_shared(&s_done)), 0u);
    // DSMEM address of vertex v's arrival / bitmap word in its owner CTA
    auto e_addr = [&](uint32_t v) {
        const uint32_t w = v >> 5;
        return cl_map(e_sa + 4u * (((w >> lg) << 5) | (v & 31u)), w & (ncta - 1u));
    };
    auto bm_addr = [&](uint32_t v) {
        const uint32_t w = v >> 5;
        return cl_map(bmN_sa + 4u * (w >> lg), w & (ncta - 1u));
    };

    if (STAGE >= 1) {
        // global type range of owned word lw (vertices 32w .. 32w+31)
        auto wrange = [&](uint32_t lw, uint32_t &g0, uint32_t &g1) {
            const uint32_t w = (lw << lg) | rank;
            g0 = __ldg(ix.type_ptr + min(32u * w, n));
            g1 = __ldg(ix.type_ptr + min(32u * w + 32u, n));
        };
        if (STAGE == 2 && wid == 0) {  // local start of each owned word's types (bmD as scratch)
            const uint32_t per = (Wl + 31u) / 32u, lo = min(Wl, lane * per), hi = min(Wl, lo + per);
            uint32_t sum = 0, g0, g1;
            for (uint32_t lw = lo; lw < hi; ++lw) {
                wrange(lw, g0, g1);
                sum += g1 - g0;
            }
            uint32_t incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= uint32_t(o)) incl += y;
            }
            uint32_t run = incl - sum;
            for (uint32_t lw = lo; lw < hi; ++lw) {
                wrange(lw, g0, g1);
                bmD[lw] = run;
                run += g1 - g0;
            }
        }
        __syncthreads();
        for (uint32_t li = tid; li < Wl * 32u; li += kClThreads) {
            const uint32_t lw = li >> 5, v = (((lw << lg) | rank) << 5) | (li & 31u);
            uint2 r = make_uint2(0u, 0u);
            if (v < n) {
                const uint32_t a = __ldg(ix.type_ptr + v);
                r = make_uint2(a, __ldg(ix.type_ptr + v + 1) - a);
                if (STAGE == 2) r.x = bmD[lw] + (a - __ldg(ix.type_ptr + 32u * ((lw << lg) | rank)));
            }
            rng[li] = r;
        }
        if (STAGE == 2) {
            for (uint32_t lw = wid; lw < Wl; lw += kClWarps) {  // a warp per owned word
                uint32_t g0, g1;
                wrange(lw, g0, g1);
                const uint32_t l0 = bmD[lw];
                for (uint32_t t = g0 + lane; t < g1; t += 32u) {
                    hdr_s[l0 + t - g0] = __ldg(ix.type_hdr + t);
                    cb_s[l0 + t - g0] = __ldg(ix.type_cb + t);
                }
            }
        }
        __syncthreads();
    }

    // rank 0 takes the cluster's first query and pushes it to every CTA
    auto fetch_query = [&]() {
        if (rank == 0 && tid == 0) {
            const unsigned long long qi = atomicAdd(qcounter, 1ull);
            const unsigned long long q = qi >= nq ? ~0ull : qi;
            for (uint32_t r = 0; r < ncta; ++r) {
                cl_st(cl_map(q_sa, r), uint32_t(q));
                cl_st(cl_map(q_sa + 4u, r), uint32_t(q >> 32));
            }
        }
    };
    cl_sync();  // every CTA of the cluster has started (DSMEM may be touched only after this)
    fetch_query();
    cl_sync();
    for (;;) {
        const unsigned long long q = (unsigned long long)s_q[0] | ((unsigned long long)s_q[1] << 32);
        if (q == ~0ull) break;
        const uint32_t s = src ? src[q] : s1, ts = src ? tsv[q] : ts1;  // single query: parameters
        uint32_t *orow = out + q * uint64_t(n);
        if (s >= n || ts >= kInf) {
            for (uint32_t i = rank * kClThreads + tid; i < n; i += ncta * kClThreads) orow[i] = kInf;
            if (rank == 0 && tid == 0) {
                atomicAdd(invalid, 1ull);
                if (sweeps_out) sweeps_out[q] = 0;
            }
            cl_sync();  // everyone has read s_q before it is overwritten
            fetch_query();
            cl_sync();
            continue;
        }
        // Initialize (Algorithm 2): every CTA its own words
        for (uint32_t i = tid; i < Wl * 32u; i += kClThreads) e_loc[i] = kInf;
        for (uint32_t i = tid; i < Wl; i += kClThreads) {
            bmD[i] = 0;
            bmN[i] = 0;
        }
        if (tid == 0) {
            s_cnt[0] = s_cnt[1] = 0;
            s_more[0] = s_more[1] = 0;
            s_tmin[0] = ts;
            s_tmin[1] = s_tmin[2] = kInf;
            s_pmin[0] = s_pmin[1] = kInf;
            s_pmore[0] = s_pmore[1] = 0;
            s_S = rank == 0 ? 1u : 0u;  // ASYNC: the source's mark (counted in CTA 0)
            s_R = 0;
            s_done = 0;
        }
        __syncthreads();
        if (tid == 0) {
            const uint32_t si = __ldg(ix.perm + s);  // caller id -> internal id
            const uint32_t w = si >> 5;
            if ((w & (ncta - 1u)) == rank) {
                e_loc[((w >> lg) << 5) | (si & 31u)] = ts;
                bmN[w >> lg] = 1u << (si & 31u);
            }
        }
        cl_sync();
        uint32_t sweeps = 0;
        uint32_t t_cur = 0, t_nxt = 1, t_old = 2;
        if (ASYNC) {
            for (;;) {
                const uint32_t p = sweeps & 1u;
#ifdef EAT_CL_TRACE
                const unsigned long long tr0 = gtimer();
#endif
                // ---- take every marked vertex this CTA owns
                for (uint32_t lw = tid; lw < Wl; lw += kClThreads) {
                    if (!lds_volatile(bmN + lw)) continue;
                    uint32_t word = atomicExch(bmN + lw, 0u);
                    const uint32_t k = __popc(word);
                    if (!k) continue;
                    const uint32_t pos = atomicAdd(&s_cnt[p], k);  // the list holds every owned vertex
                    const uint32_t vbase = ((lw << lg) | rank) << 5;
                    for (uint32_t i = 0; i < k; ++i) {
                        const uint32_t b = __ffs(word) - 1u;
                        word &= word - 1u;
                        a_list[pos + i] = vbase + b;
                    }
                }
                __syncthreads();
                const uint32_t F = s_cnt[p];
                if (tid == 0) s_cnt[p ^ 1u] = 0;
#ifdef EAT_CL_TRACE
                if (tid == 0 && rank == 0 && sweeps < 1024) {
                    g_cltrace[sweeps * 6 + 0] = tr0;
                    g_cltrace[sweeps * 6 + 1] = gtimer();
                    g_cltrace[sweeps * 6 + 5] = F;
                }
#endif
                ++sweeps;
                if (F == 0) {  // idle: is any vertex pending anywhere?
                    if (rank == 0 && wid == 0) {
                        // every CTA's R, then (the addresses depend on the sum: issued
                        // after it returned) every CTA's S; equal -> fixpoint
                        const uint32_t ra = __reduce_add_sync(0xFFFFFFFFu, lane < ncta ? cl_ld(cl_map(R_sa, lane)) : 0u);
                        const uint32_t sb = __reduce_add_sync(
                            0xFFFFFFFFu, lane < ncta ? cl_ld(cl_map(S_sa + (ra & ix.zero), lane)) : 0u);
                        if (lane == 0 && ra == sb) s_done = 1u;
                        __syncwarp();
                    }
                    if (tid == 0) {
                        s_idle = cl_ld(done0) != 0u;
                        if (!s_idle) __nanosleep(64);
                    }
                    __syncthreads();
                    if (s_idle) break;
                    if (sweeps > (1u << 22)) break;  // watchdog (never reached by a correct run)
                    continue;
                }
                const uint32_t g = min(32u, max(1u, (F + kClWarps - 1u) / kClWarps));
        for (uint32_t k0 = 0; k0 < F; k0 += kClWarps * g) {  // strided: warp w takes k0 + w + i * warps (city / country single query -2 %, profiles/r02_ab_cta_strided.jsonl)
                    const uint32_t j = k0 + wid + lane * kClWarps;
                    uint32_t x = 0, p0 = 0, nt = 0;
                    if (lane < g && j < F) {
                        x = a_list[j];
                        if (STAGE >= 1) {
                            const uint2 r = rng[((((x >> 5) >> lg) << 5) | (x & 31u))];
                            p0 = r.x;
                            nt = r.y;
                        } else {
                            p0 = __ldg(ix.type_ptr + x);
                            nt = __ldg(ix.type_ptr + x + 1) - p0;
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
                        uint32_t ea = 0, cand = kNone, tv = 0;  // a try: lower e[tv] (at ea) to cand
                        if (qp < tot) {
                            const uint32_t t = o_p0 + (qp - (o_incl - o_nt));
                            const uint32_t eu = lds_volatile(e_loc + ((((u >> 5) >> lg) << 5) | (u & 31u)));
                            uint32_t cb;
                            TypeRec tr;
                            if (STAGE == 2) {
                                cb = cb_s[t];
                                const uint4 h = hdr_s[t];
                                tr = TypeRec{h.x, h.y, h.z, h.w};
                            } else {
                                cb = __ldg(ix.type_cb + t);
                                tr = load_type(ix, t);
                                tr.last |= cb & ix.zero;
                            }
                            if (eu <= tr.last) {
                                // the hour-cluster record (one global access) is requested
                                // before the DSMEM read of e[v]: the two latencies overlap
                                uint4 r0 = make_uint4(0u, 0u, 0u, 0u), r1 = r0;
                                const uint32_t kc = cluster_of(ix, eu);
                                if (eu > tr.first) ldg_crec(ix, cb + kc, r0, r1);
                                ea = e_addr(tr.v);
                                const uint32_t av = cl_ld(ea);
                                if (max(eu, tr.first) + tr.lam < av) {
                                    const uint32_t tc = eu <= tr.first ? tr.first : cluster_scan<true>(ix, r0, r1, kc, eu);
                                    if (tc + tr.lam < av) {
                                        cand = tc + tr.lam;
                                        tv = tr.v;
                                    }
                                }
                            }
                        }
                        // (relaxing the lowered vertices at once -- continuation, as in
                        // gasync.cu -- is 11 % slower here: r02_ab_cluster_continuation.jsonl)
                        // Lower and mark.  Every lane that tries is counted in CTA 0's
                        // pending counter by a returning add issued with the atomicMins
                        // (one round trip for both) and waited for -- the bit address
                        // depends on its value -- before any bit is set: a mark is
                        // counted before its owner can see (and un-count) it.  Tries
                        // that lowered nothing and marks that hit a set bit are
                        // subtracted after (the counter only over-counts).  (Per-CTA
                        // counters read by a two-wave detector in CTA 0 instead: same
                        // speed, profiles/r02_ab_cluster_termination.jsonl)
                        const uint32_t tm = __ballot_sync(0xFFFFFFFFu, cand != kNone);
                        if (tm) {
                            const uint32_t ld = __ffs(tm) - 1u;
                            uint32_t o = 0;
                            if (lane == ld) o = atomicAdd(&s_S, uint32_t(__popc(tm)));  // local, returning
                            const bool low = cand != kNone && cand < cl_min(ea, cand);
                            o = __shfl_sync(0xFFFFFFFFu, o, ld);
                            const uint32_t wm = __ballot_sync(0xFFFFFFFFu, low);
                            uint32_t dup = 0;
                            if (low) dup = cl_or_old(bm_addr(tv) + (o & ix.zero), 1u << (tv & 31u)) & (1u << (tv & 31u));
                            const uint32_t dm = __ballot_sync(0xFFFFFFFFu, dup != 0u);
                            const uint32_t extra = uint32_t(__popc(tm)) - uint32_t(__popc(wm)) + uint32_t(__popc(dm));
                            if (extra && lane == ld) atomicSub(&s_S, extra);
                        }
                    }
                }
                __syncthreads();  // every relaxation (and mark count) of the F taken vertices is done
                if (tid == 0) atomicAdd(&s_R, F);
#ifdef EAT_CL_TRACE
                if (tid == 0 && rank == 0 && sweeps - 1 < 1024) g_cltrace[(sweeps - 1) * 6 + 3] = gtimer();
#endif
            }
        }
        for (; !ASYNC;) {
#ifdef EAT_CL_TRACE
            if (tid == 0 && rank == 0 && sweeps < 1024) g_cltrace[sweeps * 6 + 0] = gtimer();
#endif
            const uint32_t p = sweeps & 1u;
            uint32_t thr = kInf;
            if (window < kInf) {
                const uint32_t base = s_tmin[t_cur];
                thr = base + min(window, kInf - base);  // saturating
            }
            // ---- 1. select + compact over the owned words
            uint32_t dmin = kInf, ndef = 0;
            for (uint32_t lw = tid; lw < Wl; lw += kClThreads) {
#if EAT_CL_BAR1
                uint32_t word = bmD[lw] | bmN[lw];
                if (!word) continue;
                bmN[lw] = 0;
#else
                // other CTAs may be marking this word right now (no cluster
                // barrier before the select): read-and-clear atomically, a
                // mark that lands later is taken in the next sweep
                const uint32_t nw = lds_volatile(bmN + lw);
                uint32_t word = bmD[lw] | (nw ? atomicExch(bmN + lw, 0u) : 0u);
                if (!word) continue;
#endif
                uint32_t sel = word;
                if (thr < kInf) {
                    sel = 0;
                    uint32_t rest = word;
                    while (rest) {
                        const uint32_t b = __ffs(rest) - 1u;
                        rest &= rest - 1u;
                        const uint32_t a = lds_volatile(e_loc + lw * 32u + b);
                        if (a <= thr) sel |= 1u << b;
                        else dmin = min(dmin, a);
                    }
                }
                const uint32_t vbase = ((lw << lg) | rank) << 5;  // global vertex id of bit 0
                uint32_t taken = 0;
                const uint32_t k = __popc(sel);
                if (k) {
                    const uint32_t pos = atomicAdd(&s_cnt[p], k);
                    const uint32_t put = pos < kClListCap ? min(k, kClListCap - pos) : 0u;
                    uint32_t rest = sel;
                    for (uint32_t i = 0; i < put; ++i) {
                        const uint32_t b = __ffs(rest) - 1u;
                        rest &= rest - 1u;
                        s_list[pos + i] = vbase + b;
                        taken |= 1u << b;
                    }
                    while (rest) {  // list full: stays active for a later sweep
                        const uint32_t b = __ffs(rest) - 1u;
                        rest &= rest - 1u;
                        dmin = min(dmin, lds_volatile(e_loc + lw * 32u + b));
                    }
                }
                bmD[lw] = word & ~taken;
                ndef |= word & ~taken;
            }
            dmin = __reduce_min_sync(0xFFFFFFFFu, dmin);
            if (lane == 0 && dmin < kInf) atomicMin(&s_pmin[p], dmin);
            if (ndef) s_pmore[p] = 1u;
#ifdef EAT_CL_TRACE
            if (tid == 0 && rank == 0 && sweeps < 1024) g_cltrace[sweeps * 6 + 1] = gtimer();
#endif
#if EAT_CL_BAR1
            cl_sync();  // selects done everywhere (bmN cleared) before anyone marks
#else
            __syncthreads();  // this CTA's list is complete
#endif
#ifdef EAT_CL_TRACE
            if (tid == 0 && rank == 0 && sweeps < 1024) g_cltrace[sweeps * 6 + 2] = gtimer();
#endif
            if (tid == 0) {  // slots of the next sweep: everyone is past their last read
                s_cnt[p ^ 1u] = 0;
                s_more[p ^ 1u] = 0;
                s_tmin[t_old] = kInf;
                s_pmin[p ^ 1u] = kInf;
                s_pmore[p ^ 1u] = 0;
            }
            const uint32_t F = min(s_cnt[p], kClListCap);
            // ---- 2. warp-flattened (vertex, type) pairs (as k_query_cta)
            const uint32_t g = min(32u, max(1u, (F + kClWarps - 1u) / kClWarps));
            uint32_t imin = kInf;
        for (uint32_t k0 = 0; k0 < F; k0 += kClWarps * g) {  // strided: warp w takes k0 + w + i * warps
                const uint32_t j = k0 + wid + lane * kClWarps;
                uint32_t x = 0, p0 = 0, nt = 0;
                if (lane < g && j < F) {
                    x = s_list[j];
                    if (STAGE >= 1) {
                        const uint2 r = rng[((((x >> 5) >> lg) << 5) | (x & 31u))];
                        p0 = r.x;
                        nt = r.y;
                    } else {
                        p0 = __ldg(ix.type_ptr + x);
                        nt = __ldg(ix.type_ptr + x + 1) - p0;
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
                    // u is owned by this CTA: local read
                    const uint32_t eu = lds_volatile(e_loc + ((((u >> 5) >> lg) << 5) | (u & 31u)));
                    uint32_t cb;
                    TypeRec tr;
                    if (STAGE == 2) {  // t is a local type index
                        cb = cb_s[t];
                        const uint4 h = hdr_s[t];
                        tr = TypeRec{h.x, h.y, h.z, h.w};
                    } else {
                        cb = __ldg(ix.type_cb + t);
                        tr = load_type(ix, t);
                        tr.last |= cb & ix.zero;  // pins cb's load beside the header's
                    }
                    if (eu > tr.last) continue;
                    const uint32_t ea = e_addr(tr.v);
                    const uint32_t av = cl_ld(ea);
                    if (max(eu, tr.first) + tr.lam >= av) continue;
                    const uint32_t tc = eu <= tr.first ? tr.first : cluster_lookup(ix, cb, eu);
                    const uint32_t cand = tc + tr.lam;
                    if (cand < av) {
                        const uint32_t old = cl_min(ea, cand);
                        if (cand < old) {
                            cl_or(bm_addr(tr.v), 1u << (tr.v & 31u));
                            imin = min(imin, cand);
                        }
                    }
                }
            }
            imin = __reduce_min_sync(0xFFFFFFFFu, imin);
            if (lane == 0 && imin < kInf) {
                atomicMin(&s_pmin[p], imin);
                s_pmore[p] = 1u;
            }
            __syncthreads();
#ifdef EAT_CL_TRACE
            if (tid == 0 && rank == 0 && sweeps < 1024) g_cltrace[sweeps * 6 + 3] = gtimer();
#endif
            // ---- 3. push this CTA's partials into every CTA's control words
            if (tid < ncta) {
                const uint32_t pm = s_pmin[p];
                if (pm < kInf) cl_redmin(cl_map(tmin_sa + 4u * t_nxt, tid), pm);
                if (s_pmore[p]) cl_st(cl_map(more_sa + 4u * p, tid), 1u);
            }
            cl_sync();
#ifdef EAT_CL_TRACE
            if (tid == 0 && rank == 0 && sweeps < 1024) g_cltrace[sweeps * 6 + 4] = gtimer();
#endif
            ++sweeps;
            {
                const uint32_t tmp = t_cur;
                t_cur = t_nxt;
                t_nxt = t_old;
                t_old = tmp;
            }
            if (s_more[p] == 0u) break;  // nothing deferred, nothing lowered anywhere: fixpoint
        }
        // Output in caller ids: CTA `rank` writes a strided share of the row,
        // reading the arrivals through DSMEM
        if ((n & 3u) == 0u && (reinterpret_cast<uintptr_t>(orow) & 15u) == 0u) {
            const uint4 *pv = reinterpret_cast<const uint4 *>(ix.perm);
            uint4 *ov = reinterpret_cast<uint4 *>(orow);
            for (uint32_t i = rank * kClThreads + tid; i < n / 4u; i += ncta * kClThreads) {
                const uint4 pi = __ldg(pv + i);
                ov[i] = make_uint4(cl_ld(e_addr(pi.x)), cl_ld(e_addr(pi.y)), cl_ld(e_addr(pi.z)), cl_ld(e_addr(pi.w)));
            }
        } else {
            for (uint32_t i = rank * kClThreads + tid; i < n; i += ncta * kClThreads)
                orow[i] = cl_ld(e_addr(__ldg(ix.perm + i)));
        }
        if (rank == 0 && tid == 0 && sweeps_out) sweeps_out[q] = sweeps;
        cl_sync();  // every CTA is done reading e[] / s_q of this query
        fetch_query();
        cl_sync();
    }
}

}  // namespace

static size_t cluster_smem_bytes(uint32_t n, int cs, int stage, uint32_t tl_cap, bool async) {
    const size_t W = (n + 31u) / 32u;
    const size_t Wl = (W + size_t(cs) - 1u) / size_t(cs);
    size_t b = Wl * 32u * 4u + 2u * Wl * 4u;
    if (stage >= 1) b += Wl * 32u * 8u;
    if (stage == 2) b += size_t(tl_cap) * 20u;
    if (async) b += Wl * 32u * 4u;
    return b;
}

template <int STAGE, bool ASYNC>
static int cluster_max_active_t(uint32_t n, int cs, uint32_t tl_cap) {
    auto kern = k_query_cluster<STAGE, ASYNC>;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return 0;
    const size_t smem = cluster_smem_bytes(n, cs, STAGE, tl_cap, ASYNC);
    if (smem + fa.sharedSizeBytes > size_t(optin)) return 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess) return 0;
    if (cs > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return 0;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(cs);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(unsigned(cs));
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return nc;
}

int cluster_max_active(uint32_t n, int cs, int stage, uint32_t tl_cap, bool async) {
    if (cs < 1 || cs > 16 || (cs & (cs - 1))) return 0;
    switch (stage * 2 + int(async)) {
        case 5: return cluster_max_active_t<2, true>(n, cs, tl_cap);
        case 4: return cluster_max_active_t<2, false>(n, cs, tl_cap);
        case 3: return cluster_max_active_t<1, true>(n, cs, tl_cap);
        case 2: return cluster_max_active_t<1, false>(n, cs, tl_cap);
        case 1: return cluster_max_active_t<0, true>(n, cs, tl_cap);
        default: return cluster_max_active_t<0, false>(n, cs, tl_cap);
    }
}

template <int STAGE, bool ASYNC>
static cudaError_t launch_cluster_t(const DevIndex &ix, const ClusterArgs &a, unsigned nc, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(a.cs);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(unsigned(a.cs) * nc);
    cfg.blockDim = dim3(kClThreads);
    cfg.dynamicSmemBytes = cluster_smem_bytes(ix.n, a.cs, STAGE, a.tl_cap, ASYNC);
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_query_cluster<STAGE, ASYNC>, ix, a.src, a.ts, a.nq, a.out, a.sweeps, a.qcounter,
                              a.invalid, a.tl_cap, a.s1, a.ts1);
}

cudaError_t launch_query_cluster(const DevIndex &ix, const ClusterArgs &a, cudaStream_t st) {
    const int nc_max = cluster_max_active(ix.n, a.cs, a.stage, a.tl_cap, a.async);
    if (nc_max < 1) return cudaErrorInvalidConfiguration;
    const uint64_t want = a.max_clusters ? std::min<uint64_t>(a.max_clusters, a.nq) : a.nq;
    const unsigned nc = unsigned(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(nc_max), want)));
    cudaError_t e = cudaMemsetAsync(a.qcounter, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return e;
    switch (a.stage * 2 + int(a.async)) {
        case 5: return launch_cluster_t<2, true>(ix, a, nc, st);
        case 4: return launch_cluster_t<2, false>(ix, a, nc, st);
        case 3: return launch_cluster_t<1, true>(ix, a, nc, st);
        case 2: return launch_cluster_t<1, false>(ix, a, nc, st);
        case 1: return launch_cluster_t<0, true>(ix, a, nc, st);
        default: return launch_cluster_t<0, false>(ix, a, nc, st);
    }
}

#ifdef EAT_CL_TRACE
// debug build only: copy the per-sweep timeline of the last cluster query
extern "C" int eat_debug_cluster_trace(unsigned long long *dst, int n) {
    return int(cudaMemcpyFromSymbol(dst, g_cltrace, sizeof(unsigned long long) * size_t(std::min(n, 1024 * 6))));
}
#endif
}  // namespace eat
