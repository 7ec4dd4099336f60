// async.cu -- CTA-partitioned asynchronous single-query kernel (EAT_KERNEL_ASYNC).
//
// One query on the whole GPU without a grid barrier per sweep (SURVEY 8(a)
// a9/a10, §7 step 7).  CTA c owns the internal vertex range [c*span,
// (c+1)*span) (contiguous after locality renumbering) with its e[] slice in
// shared memory, and the out-types of those vertices.  A query runs in rounds:
//   1. drain: messages from other CTAs (vertices of this range whose e[]
//      another CTA lowered in the previous round) are folded into the
//      shared slice and activated;
//   2. local phase: relaxation sweeps of the owned active vertices, separated
//      by CTA barriers, until the range is locally quiescent.  A target owned
//      by this CTA is lowered with a shared-memory atomicMin; any other
//      target with a global atomicMin on the e[] mirror plus, if it improved,
//      a message into the owner's inbox (deduplicated by a per-vertex flag);
//   3. one grid barrier; stop when no message was sent in the round.
// Every improvement is also applied to the global mirror, which holds the
// result.  The relaxation, lookup and fixpoint are the paper's (Alg. 3/6,
// PAPER.md:175-306, atomicMin PAPER.md:403-409); only the schedule differs
// (sweeps are local; exchange rounds replace global sweeps).
#include <algorithm>

#include "async.cuh"
#include "device_common.cuh"

namespace eat {
namespace {

using namespace dev;

constexpr int kAsyncThreads = 1024;
constexpr uint32_t kAsyncListCap = 2048;

__global__ void __launch_bounds__(kAsyncThreads, 1) k_query_async(DevIndex ix, AsyncWork w, uint32_t span, uint32_t s,
                                                                  uint32_t ts, uint32_t *out) {
    constexpr uint32_t kWarps = kAsyncThreads / 32;
    extern __shared__ uint32_t sm[];
    const uint32_t n = ix.n;
    const uint32_t P = gridDim.x, c = blockIdx.x;
    const uint32_t lo = min(n, c * span), hi = min(n, lo + span), own = hi - lo;
    const uint32_t Wl = (span + 31u) / 32u;
    const uint32_t spad = (span + 3u) & ~3u;
    uint32_t *sarr = sm;
    volatile uint32_t *vsarr = sm;
    uint32_t *bmD = sm + spad;
    uint32_t *bmN = bmD + Wl;
    __shared__ uint32_t s_list[kAsyncListCap];
    __shared__ uint32_t s_cnt[2], s_more[2];
    const uint32_t tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    const uint64_t gtid = uint64_t(c) * kAsyncThreads + tid, gsz = uint64_t(P) * kAsyncThreads;
    uint32_t *bar = w.ctl + kBarWord;  // monotonic barrier counter (zeroed per launch)
    uint32_t bar_epoch = 0;

    // ---- init (Algorithm 2)
    for (uint64_t i = gtid; i < n; i += gsz) {
        w.garr[i] = kInf;
        w.inflag[i] = 0;
    }
    for (uint64_t i = gtid; i < 2ull * P; i += gsz) w.inbox_cnt[i] = 0;
    if (gtid == 0) {
        w.ctl[0] = w.ctl[1] = w.ctl[2] = 0;
        w.ctl[8] = 0;
        w.ctl[9] = 0;
    }
    for (uint32_t i = tid; i < span; i += kAsyncThreads) sarr[i] = kInf;
    for (uint32_t i = tid; i < Wl; i += kAsyncThreads) bmD[i] = bmN[i] = 0;
    if (tid == 0) s_cnt[0] = s_cnt[1] = s_more[0] = s_more[1] = 0;
    grid_sync(bar, bar_epoch);
    const uint32_t si = __ldg(ix.perm + s);
    if (tid == 0 && si >= lo && si < hi) {
        sarr[si - lo] = ts;
        bmN[(si - lo) >> 5] |= 1u << ((si - lo) & 31u);
        w.garr[si] = ts;
    }
    __syncthreads();

    uint32_t total_sweeps = 0;
    for (uint32_t r = 0;; ++r) {
        const uint32_t pin = r & 1u;  // inbox parity written in this round
        // ---- 1. drain the previous round's messages
        if (r > 0) {
            const uint32_t pprev = pin ^ 1u;
            const uint32_t k = ld_cg(w.inbox_cnt + pprev * P + c);
            for (uint32_t i = tid; i < k; i += kAsyncThreads) {
                const uint32_t v = ld_cg(w.inbox + uint64_t(pprev) * n + lo + i);
                atomicExch(w.inflag + v, 0u);
                __threadfence();
                const uint32_t g = ld_cg(w.garr + v);
                const uint32_t vl = v - lo;
                if (g < sarr[vl]) {
                    sarr[vl] = g;  // each v appears once per inbox
                    atomicOr(bmN + (vl >> 5), 1u << (vl & 31u));
                }
            }
            __syncthreads();
            if (tid == 0) {
                w.inbox_cnt[pprev * P + c] = 0;
                if (c == 0) w.ctl[(r + 1u) % 3u] = 0;  // message counter of the next round
            }
        }
        // ---- 2. local phase to quiescence
        uint32_t nmsg = 0;
        for (uint32_t sw = 0;; ++sw) {
            const uint32_t p = sw & 1u;
            uint32_t ndef = 0;
            for (uint32_t wd = tid; wd < Wl; wd += kAsyncThreads) {
                const uint32_t word = bmD[wd] | bmN[wd];
                if (!word) continue;
                bmN[wd] = 0;
                const uint32_t k = __popc(word);
                const uint32_t pos = atomicAdd(&s_cnt[p], k);
                const uint32_t put = pos < kAsyncListCap ? min(k, kAsyncListCap - pos) : 0u;
                uint32_t rest = word, taken = 0;
                for (uint32_t i = 0; i < put; ++i) {
                    const uint32_t b = __ffs(rest) - 1u;
                    rest &= rest - 1u;
                    s_list[pos + i] = wd * 32u + b;
                    taken |= 1u << b;
                }
                bmD[wd] = word & ~taken;
                ndef += __popc(word & ~taken);
            }
            ndef = __reduce_add_sync(0xFFFFFFFFu, ndef);
            if (lane == 0 && ndef) atomicAdd(&s_more[p], ndef);
            __syncthreads();
            if (tid == 0) {
                s_cnt[p ^ 1u] = 0;
                s_more[p ^ 1u] = 0;
            }
            const uint32_t F = min(s_cnt[p], kAsyncListCap);
            const uint32_t g = min(32u, max(1u, (F + kWarps - 1u) / kWarps));
            uint32_t nimpr = 0;
            for (uint32_t k0 = wid * g; k0 < F; k0 += kWarps * g) {
                const uint32_t j = k0 + lane;
                uint32_t xl = 0, p0 = 0, nt = 0;
                if (lane < g && j < F) {
                    xl = s_list[j];
                    p0 = __ldg(ix.type_ptr + lo + xl);
                    nt = __ldg(ix.type_ptr + lo + xl + 1) - p0;
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
                    const uint32_t ul = __shfl_sync(0xFFFFFFFFu, xl, L);
                    if (qp >= tot) continue;
                    const uint32_t t = o_p0 + (qp - (o_incl - o_nt));
                    const uint32_t eu = vsarr[ul];
                    const TypeRec tr = load_type(ix, t);
                    if (eu > tr.last) continue;
                    const bool local = tr.v >= lo && tr.v < hi;
                    const uint32_t av = local ? vsarr[tr.v - lo] : ld_cg(w.garr + tr.v);
                    if (max(eu, tr.first) + tr.lam >= av) continue;
                    const uint32_t tc = eu <= tr.first ? tr.first : cluster_lookup(ix, __ldg(ix.type_cb + t), eu);
                    const uint32_t cand = tc + tr.lam;
                    if (cand >= av) continue;
                    if (local) {
                        const uint32_t vl = tr.v - lo;
                        const uint32_t old = atomicMin(sarr + vl, cand);
                        if (cand < old) {
                            atomicOr(bmN + (vl >> 5), 1u << (vl & 31u));
                            atomicMin(w.garr + tr.v, cand);  // mirror (RED: no return used)
                            ++nimpr;
                        }
                    } else {
                        const uint32_t old = atomicMin(w.garr + tr.v, cand);
                        if (cand < old) {
                            __threadfence();
                            if (atomicExch(w.inflag + tr.v, 1u) == 0u) {
                                const uint32_t owner = tr.v / span;
                                const uint32_t pos = atomicAdd(w.inbox_cnt + pin * P + owner, 1u);
                                w.inbox[uint64_t(pin) * n + uint64_t(owner) * span + pos] = tr.v;
                                ++nmsg;
                            }
                        }
                    }
                }
            }
            nimpr = __reduce_add_sync(0xFFFFFFFFu, nimpr);
            if (lane == 0 && nimpr) atomicAdd(&s_more[p], nimpr);
            __syncthreads();
            ++total_sweeps;
            if (s_more[p] == 0u) {
                // leave the parity slots clean for the next round's sweep 0
                __syncthreads();
                if (tid == 0) s_cnt[0] = s_cnt[1] = s_more[0] = s_more[1] = 0;
                __syncthreads();
                break;
            }
        }
        (void)own;
        nmsg = __reduce_add_sync(0xFFFFFFFFu, nmsg);
        if (lane == 0 && nmsg) atomicAdd(w.ctl + r % 3u, nmsg);
        // ---- 3. exchange barrier
        grid_sync(bar, bar_epoch);
        if (ld_cg(w.ctl + r % 3u) == 0u) {
            if (tid == 0) {
                atomicMax(w.ctl + 9, total_sweeps);
                if (c == 0) w.ctl[8] = r + 1u;
            }
            break;
        }
    }
    grid_sync(bar, bar_epoch);
    for (uint64_t i = gtid; i < n; i += gsz) out[i] = ld_cg(w.garr + __ldg(ix.perm + i));
}

}  // namespace

size_t async_smem_bytes(uint32_t span) {
    const size_t spad = (span + 3u) & ~3u, Wl = (span + 31u) / 32u;
    return (spad + 2 * Wl) * sizeof(uint32_t);
}

cudaError_t async_alloc(AsyncWork &w, uint32_t n, uint32_t max_parts) {
    cudaError_t e;
    if ((e = cudaMalloc(&w.garr, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.inflag, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.inbox, 2ull * n * 4 + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.inbox_cnt, 2ull * max_parts * 4 + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.ctl, kCtlWords * 4)) != cudaSuccess) return e;
    return cudaMemset(w.ctl, 0, kCtlWords * 4);
}

void async_free(AsyncWork &w) {
    void *ptrs[] = {w.garr, w.inflag, w.inbox, w.inbox_cnt, w.ctl};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    w = AsyncWork{};
}

int async_parts(uint32_t n) {
    int dev = 0, sms = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, k_query_async) != cudaSuccess) return 0;
    const uint32_t P = uint32_t(sms);
    const uint32_t span = (n + P - 1) / P;
    if (async_smem_bytes(span) + fa.sharedSizeBytes > size_t(optin)) return 0;
    return int(P);
}

cudaError_t launch_query_async(const DevIndex &ix, const AsyncWork &w, uint32_t s, uint32_t t_s, uint32_t *d_out,
                               cudaStream_t st) {
    const int P = async_parts(ix.n);
    if (P <= 0) return cudaErrorInvalidConfiguration;
    const uint32_t span = (ix.n + uint32_t(P) - 1) / uint32_t(P);
    const size_t smem = async_smem_bytes(span);
    cudaError_t e = cudaFuncSetAttribute(k_query_async, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_query_async, kAsyncThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    e = cudaMemsetAsync(w.ctl + kBarWord, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    DevIndex ixc = ix;
    AsyncWork wc = w;
    uint32_t spanv = span;
    void *args[] = {&ixc, &wc, &spanv, &s, &t_s, &d_out};
    return cudaLaunchCooperativeKernel((const void *)k_query_async, dim3(unsigned(P)), dim3(kAsyncThreads), args, smem,
                                       st);
}

}  // namespace eat
