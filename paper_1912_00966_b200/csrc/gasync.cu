// gasync.cu -- EAT_KERNEL_GRID_ASYNC: one query on the whole GPU without any
// barrier between relaxations.
//
// The asynchronous schedule of the cluster kernel (cluster.cu ASYNC) over
// global memory, so that graphs whose e[] does not fit a cluster (country)
// and the whole GPU's SMs can use it: a persistent cooperative grid of
// 1024-thread CTAs, one per SM.  e[] and the "marked" bitmap live in global
// memory; bitmap word w (vertices 32w .. 32w+31) is owned by CTA w mod G.
// Every CTA loops on its own:
//   take every marked vertex it owns (atomicExch on its bitmap words, so a
//   mark may land at any time) -> relax their connection types (Alg. 3,
//   PAPER.md:175-190; Cluster-AP lookup, Alg. 6 + PAPER.md:300-306;
//   atomicMin on e[v]) -> mark every v it lowered;
// all active vertices are taken (the paper's topology-driven schedule, any
// order reaches the same fixpoint).
// Termination (no barrier to count "nothing changed" at): per CTA, S counts
// the marks it set (a warp adds every lane that tries to lower an e[v] with
// a returning atomic issued beside the atomicMins and waited for BEFORE the
// bits are set -- the bit address depends on its value; the tries that
// lowered nothing and the marks that hit an already-set bit are subtracted
// after) and R the vertices whose relaxations it finished.  When CTA 0 is idle it sums every R, then
// every S; both are monotone in the true counts and a mark is counted in S
// before its bit is visible, so sum(R) read first == sum(S) read second means
// nothing was marked or in processing at any instant between the two reads
// -- and a fixpoint is stable: it raises the done flag every idle CTA polls.
// Grid barriers only around a query (initialization, output).
#include <algorithm>

#include "device_common.cuh"
#include "kernels.cuh"

namespace eat {
namespace {

using namespace dev;

// Counters of CTA c at cnt[c * kGaCntCta ...]: S of warp k at + 8 k (one
// 32-byte sector each: a warp's returning S add meets no other warp's), R at
// + kGaRWord.  Per-warp S: the add a marking warp waits for is uncontended
// (one counter per CTA: single queries 7-8 % slower, r02_ab_spec_count.jsonl).
constexpr uint32_t kGaRWord = 32u * 8u;
constexpr uint32_t kGaCntCta = kGaRWord + 8u;
static_assert(kGaCntCta <= kGaCntWordsPerCta, "counter block");

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) { return __ldcv(p); }  // fetched again (L2)

// 32-byte cluster record r as volatile loads (issued where written)
__device__ __forceinline__ void ldg_crec_ga(const DevIndex &ix, uint32_t r, uint4 &r0, uint4 &r1) {
    const uint4 *p = ix.crec + 2 * uint64_t(r);
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(r0.x), "=r"(r0.y), "=r"(r0.z), "=r"(r0.w) : "l"(p));
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r1.x), "=r"(r1.y), "=r"(r1.z), "=r"(r1.w)
                 : "l"(p + 1));
}

#ifndef EAT_GA_CONT
#define EAT_GA_CONT 1  // continuation: a warp relaxes the vertices it just lowered (one level): metro -5 %, country -2 %, r02_ab_gasync_cont.jsonl
#endif

constexpr int kGaThreads = 1024;  // one CTA per SM (512 x 2 ... 256 x 8 within +-3 %: r02_gasync_shape.jsonl)
constexpr uint32_t kGaWarps = kGaThreads / 32;

// (A warp-asynchronous variant -- each warp polls and relaxes its own words,
// no CTA barrier at all -- is 1.7-2.8x slower: 4,736 polling warps and one
// warp per word of work, r02_ab_gasync_warp.jsonl.  Also staging the owned
// types' headers in shared memory when they fit
// (metro), or counting marks against credits pre-added to S instead of one
// returning atomic per marking warp, measured no faster / 8 % slower:
// r02_gasync_stage.jsonl, r02_ab_gasync_credits.jsonl.)
__global__ void __launch_bounds__(kGaThreads, 1)
    k_query_gasync(DevIndex ix, GAsyncWork w, uint32_t s, uint32_t ts, uint32_t *__restrict__ out) {
    extern __shared__ uint4 sm4[];
    const uint32_t n = ix.n, G = gridDim.x, c = blockIdx.x;
    const uint32_t W = (n + 31u) / 32u;
    const uint32_t Wl = (W + G - 1u) / G;                      // words owned by this CTA (some may be >= W)
    uint2 *rng = reinterpret_cast<uint2 *>(sm4);               // [32 Wl] type range of every owned vertex
    uint32_t *list = reinterpret_cast<uint32_t *>(rng + Wl * 32u);  // [32 Wl] taken vertices
    __shared__ uint32_t s_cnt[2];
    __shared__ uint32_t s_done;
    __shared__ uint32_t s_red[2];  // CTA 0's detector: sum of R, sum of S
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    const uint64_t gtid = uint64_t(c) * kGaThreads + tid, gsz = uint64_t(G) * kGaThreads;
    uint32_t *bar = w.ctl + kBarWord;  // monotonic grid-barrier counter (zeroed per launch)
    uint32_t bar_epoch = 0;
    uint32_t *myS = w.cnt + c * kGaCntCta + wid * 8u, *myR = w.cnt + c * kGaCntCta + kGaRWord;

    // ---- stage the owned vertices' index; initialize (Alg. 2)
    for (uint32_t li = tid; li < Wl * 32u; li += kGaThreads) {
        const uint32_t gw = (li >> 5) * G + c, v = gw * 32u + (li & 31u);
        uint2 r = make_uint2(0u, 0u);
        if (v < n) {
            const uint32_t a = __ldg(ix.type_ptr + v);
            r = make_uint2(a, __ldg(ix.type_ptr + v + 1) - a);
        }
        rng[li] = r;
    }
    for (uint64_t i = gtid; i < n; i += gsz) w.arr[i] = kInf;
    for (uint64_t i = gtid; i < W; i += gsz) w.bm[i] = 0;
    if (lane == 0) myS[0] = 0;
    if (tid == 0) {
        myR[0] = 0;
        s_cnt[0] = s_cnt[1] = 0;
        s_done = 0;
    }
    if (gtid == 0) w.ctl[0] = 0;  // done flag
    grid_sync(bar, bar_epoch, G);
    if (gtid == 0) {
        const uint32_t si = __ldg(ix.perm + s);
        w.arr[si] = ts;
        w.bm[si >> 5] = 1u << (si & 31u);
        atomicAdd(w.cnt + ((si >> 5) % G) * kGaCntCta, 1u);  // the source's mark, counted by its owner (warp 0's S)
    }
    grid_sync(bar, bar_epoch, G);

    // candidate arrival at v = tr.v through type t of a source with arrival
    // eu (Alg. 3 up to the atomicMin); kNone if it cannot lower e[v]
    auto prep = [&](uint32_t eu, uint32_t t, uint32_t &v) -> uint32_t {
        const uint32_t cb = __ldg(ix.type_cb + t);
        TypeRec tr = load_type(ix, t);
        tr.last |= cb & ix.zero;
        v = tr.v;
        if (eu > tr.last) return kNone;
        uint4 r0 = make_uint4(0u, 0u, 0u, 0u), r1 = r0;
        const uint32_t kc = cluster_of(ix, eu);
        if (eu > tr.first) ldg_crec_ga(ix, cb + kc, r0, r1);  // overlaps the e[v] read
        const uint32_t av = __ldcg(w.arr + tr.v);
        if (max(eu, tr.first) + tr.lam >= av) return kNone;
        const uint32_t tc = eu <= tr.first ? tr.first : cluster_scan<true>(ix, r0, r1, kc, eu);
        const uint32_t cand = tc + tr.lam;
        return cand < av ? cand : kNone;
    };
    // relax type t of a source with arrival eu; returns the target it lowered
    auto relax = [&](uint32_t eu, uint32_t t) -> uint32_t {
        uint32_t v;
        const uint32_t cand = prep(eu, t, v);
        return (cand != kNone && cand < atomicMin(w.arr + v, cand)) ? v : kNone;
    };
    // set bit v of the marked bitmap; 1 if it was already set.  `o` is the
    // value a returning S add gave this warp: the address depends on it, so
    // the bit is set only after that add is performed (counted before seen)
    auto set_mark = [&](uint32_t v, uint32_t o) -> uint32_t {
        const uint32_t bit = 1u << (v & 31u);
        return (atomicOr(w.bm + (v >> 5) + (o & ix.zero), bit) & bit) != 0u;
    };
    // mark the lanes' lowered vertices (wm: ballot of mv != kNone; warp-uniform)
    auto mark = [&](uint32_t mv, uint32_t wm) {
        if (!wm) return;
        const uint32_t ld = __ffs(wm) - 1u;
        uint32_t o = 0;
        if (lane == ld) o = atomicAdd(myS, uint32_t(__popc(wm)));  // counted in S first
        o = __shfl_sync(0xFFFFFFFFu, o, ld);
        const uint32_t dm = __ballot_sync(0xFFFFFFFFu, mv != kNone && set_mark(mv, o));
        if (dm && lane == ld) atomicSub(myS, uint32_t(__popc(dm)));
    };
    // lower e[v] to cand (lanes with cand != kNone) and mark the v lowered:
    // the S add is issued with the atomicMins, speculatively for every lane
    // that tries (one round trip for both), and waited for before any bit is
    // set; tries that did not lower e[v] and marks that hit a set bit are
    // subtracted afterwards (S only ever over-counts: termination is delayed,
    // never early)
    auto lower_mark = [&](uint32_t v, uint32_t cand) {
        const uint32_t tm = __ballot_sync(0xFFFFFFFFu, cand != kNone);
        if (!tm) return;
        const uint32_t ld = __ffs(tm) - 1u;
        uint32_t o = 0;
        if (lane == ld) o = atomicAdd(myS, uint32_t(__popc(tm)));
        const bool low = cand != kNone && cand < atomicMin(w.arr + v, cand);
        o = __shfl_sync(0xFFFFFFFFu, o, ld);
        const uint32_t wm = __ballot_sync(0xFFFFFFFFu, low);
        const uint32_t dm = __ballot_sync(0xFFFFFFFFu, low && set_mark(v, o));
        const uint32_t extra = uint32_t(__popc(tm)) - uint32_t(__popc(wm)) + uint32_t(__popc(dm));
        if (extra && lane == ld) atomicSub(myS, extra);
    };

    uint32_t iters = 0;
    for (;;) {
        const uint32_t p = iters & 1u;
        ++iters;
        // ---- take every marked vertex this CTA owns
        for (uint32_t lw = tid; lw < Wl; lw += kGaThreads) {
            const uint32_t gw = lw * G + c;
            if (gw >= W || !ld_volatile(w.bm + gw)) continue;
            uint32_t word = atomicExch(w.bm + gw, 0u);
            const uint32_t k = __popc(word);
            if (!k) continue;
            const uint32_t pos = atomicAdd(&s_cnt[p], k);  // the list holds every owned vertex
            for (uint32_t i = 0; i < k; ++i) {
                const uint32_t b = __ffs(word) - 1u;
                word &= word - 1u;
                list[pos + i] = (lw << 5) | b;  // local index
            }
        }
        __syncthreads();
        const uint32_t F = s_cnt[p];
        if (tid == 0) s_cnt[p ^ 1u] = 0;
        if (F == 0) {  // idle: termination detection (CTA 0) / poll
            if (c == 0) {  // every R, then every S (all of CTA 0's threads read)
                if (tid == 0) s_red[0] = s_red[1] = 0u;
                __syncthreads();
                uint32_t ra = 0;
                for (uint32_t x = tid; x < G; x += kGaThreads) ra += ld_volatile(w.cnt + x * kGaCntCta + kGaRWord);
                ra = __reduce_add_sync(0xFFFFFFFFu, ra);
                if (lane == 0 && ra) atomicAdd(&s_red[0], ra);
                __syncthreads();  // every R read returned before any S read is issued
                uint32_t sb = 0;
                for (uint32_t x = tid; x < 32u * G; x += kGaThreads)
                    sb += ld_volatile(w.cnt + (x >> 5) * kGaCntCta + (x & 31u) * 8u);
                sb = __reduce_add_sync(0xFFFFFFFFu, sb);
                if (lane == 0 && sb) atomicAdd(&s_red[1], sb);
                __syncthreads();
                if (tid == 0 && s_red[0] == s_red[1]) __stcg(w.ctl, 1u);
            }
            if (tid == 0) {
                s_done = ld_volatile(w.ctl);
                if (!s_done) __nanosleep(100);
            }
            __syncthreads();
            if (s_done || iters > (1u << 22)) break;  // (watchdog: never reached by a correct run)
            continue;
        }
        const uint32_t g = min(32u, max(1u, (F + kGaWarps - 1u) / kGaWarps));
        for (uint32_t k0 = 0; k0 < F; k0 += kGaWarps * g) {  // strided: warp w takes k0 + w + i * warps (city / country single query -2 %, profiles/r02_ab_cta_strided.jsonl)
            const uint32_t j = k0 + wid + lane * kGaWarps;
            uint32_t x = 0, p0 = 0, nt = 0;  // x: global vertex id
            if (lane < g && j < F) {
                const uint32_t li = list[j];
                x = ((li >> 5) * G + c) * 32u + (li & 31u);
                const uint2 r = rng[li];
                p0 = r.x;
                nt = r.y;
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
                uint32_t mv = kNone;  // vertex this lane lowered (to be marked)
                if (qp < tot) mv = relax(__ldcg(w.arr + u), o_p0 + (qp - (o_incl - o_nt)));
                uint32_t wm = __ballot_sync(0xFFFFFFFFu, mv != kNone);
#if EAT_GA_CONT
                if (wm) {
                    // continuation: the vertices this warp just lowered are relaxed by
                    // the warp at once (one level), instead of marked for their owners
                    uint32_t cp0 = 0, cnt = 0;
                    if (mv != kNone) {
                        cp0 = __ldg(ix.type_ptr + mv);
                        cnt = __ldg(ix.type_ptr + mv + 1) - cp0;
                    }
                    uint32_t cin = cnt;
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, cin, o);
                        if (lane >= uint32_t(o)) cin += y;
                    }
                    const uint32_t ctot = __shfl_sync(0xFFFFFFFFu, cin, 31);
                    const uint32_t cx = mv;
                    for (uint32_t cbase = 0; cbase < ctot; cbase += 32u) {
                        const uint32_t cq = cbase + lane;
                        uint32_t L2 = 0;
#pragma unroll
                        for (uint32_t step = 16; step > 0; step >>= 1) {
                            const uint32_t v = __shfl_sync(0xFFFFFFFFu, cin, L2 + step - 1u);
                            if (v <= cq) L2 += step;
                        }
                        const uint32_t c_incl = __shfl_sync(0xFFFFFFFFu, cin, L2);
                        const uint32_t c_nt = __shfl_sync(0xFFFFFFFFu, cnt, L2);
                        const uint32_t c_p0 = __shfl_sync(0xFFFFFFFFu, cp0, L2);
                        const uint32_t cu = __shfl_sync(0xFFFFFFFFu, cx, L2);
                        uint32_t v2 = 0, cand2 = kNone;
                        if (cq < ctot) cand2 = prep(__ldcg(w.arr + cu), c_p0 + (cq - (c_incl - c_nt)), v2);
                        lower_mark(v2, cand2);
                    }
                    wm = 0;
                }
#endif
                mark(mv, wm);
            }
        }
        __syncthreads();  // every relaxation (and its mark count) of the F taken vertices is done
        if (tid == 0) atomicAdd(myR, F);
    }
    if (gtid == 0) w.ctl[8] = iters;  // rank 0's iterations (eat_stats.last_sweeps)
    grid_sync(bar, bar_epoch, G);
    // ---- output in caller ids (16-byte stores when aligned)
    if ((n & 3u) == 0u && (reinterpret_cast<uintptr_t>(out) & 15u) == 0u) {
        const uint4 *pv = reinterpret_cast<const uint4 *>(ix.perm);
        uint4 *ov = reinterpret_cast<uint4 *>(out);
        for (uint64_t i = gtid; i < n / 4u; i += gsz) {
            const uint4 pi = __ldg(pv + i);
            ov[i] = make_uint4(__ldcg(w.arr + pi.x), __ldcg(w.arr + pi.y), __ldcg(w.arr + pi.z), __ldcg(w.arr + pi.w));
        }
    } else {
        for (uint64_t i = gtid; i < n; i += gsz) out[i] = __ldcg(w.arr + __ldg(ix.perm + i));
    }
}

size_t gasync_smem(uint32_t n, int G) {
    const size_t W = (n + 31u) / 32u, Wl = (W + size_t(G) - 1u) / size_t(G);
    return Wl * 32u * (8u + 4u);
}

}  // namespace

int gasync_grid(uint32_t n) {
    int dev = 0, sms = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k_query_gasync) != cudaSuccess) return 0;
    const size_t smem = gasync_smem(n, sms);
    if (smem + fa.sharedSizeBytes > size_t(optin)) return 0;
    if (cudaFuncSetAttribute(k_query_gasync, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)) != cudaSuccess)
        return 0;
    int per_sm = 0;  // every CTA must be resident (they wait on each other): one per SM
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_gasync, kGaThreads, smem) != cudaSuccess ||
        per_sm < 1)
        return 0;
    return sms;
}

cudaError_t launch_query_gasync(const DevIndex &ix, const GAsyncWork &w, uint32_t s, uint32_t t_s, uint32_t *d_out,
                                cudaStream_t st) {
    const int G = gasync_grid(ix.n);
    if (G < 1) return cudaErrorInvalidConfiguration;
    cudaError_t e = cudaMemsetAsync(w.ctl + kBarWord, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    DevIndex ixc = ix;
    GAsyncWork wc = w;
    void *args[] = {&ixc, &wc, &s, &t_s, &d_out};
    return cudaLaunchCooperativeKernel((const void *)k_query_gasync, dim3(unsigned(G)), dim3(kGaThreads), args,
                                       gasync_smem(ix.n, G), st);
}

}  // namespace eat
