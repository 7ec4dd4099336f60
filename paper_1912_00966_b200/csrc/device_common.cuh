// device_common.cuh -- device helpers shared by kernels.cu and partition.cu:
// the Cluster-AP lookup (Algorithm 6),
// the type-record load, a grid-wide barrier and warp-aggregated worklist push.
#pragma once
#include <cuda/atomic>
#include <cuda_runtime.h>

#include "eat_internal.h"
#include "kernels.cuh"

namespace eat {
namespace dev {

constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t ld_cg(const uint32_t *p) { return __ldcg(p); }

// ceil(a / s) for 1 <= a, s < 2^12 (Algorithm 6's ceil-div):
// floor((a + s - 0.5) / s) in fp32 with the approximate reciprocal (MUFU.RCP,
// relative error < 2^-21).  The exact quotient (a + s - 0.5)/s lies at least
// 0.5/s from every integer while the rounding error is below 8191 * 2^-21 / s,
// so the floor is exact -- no integer fix-up (checked exhaustively on the
// device by eat_selftest).
__device__ __forceinline__ uint32_t ceil_div12(uint32_t a, uint32_t s) {
    float r;  // approximate reciprocal (MUFU.RCP), no range fix-up: s is a small integer
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__uint2float_rn(s)));
    return __float2uint_rd((__uint2float_rn(a + s) - 0.5f) * r);
}


// First term >= x of one packed AP item, as an offset inside the cluster;
// kNone if the item is empty or all its terms are < x.  Algorithm 6 lines 3-8
// (PAPER.md:288-294): x <= start -> start; start < x <= end ->
// start + ceil((x - start) / difference) * difference.
__device__ __forceinline__ uint32_t item_next(uint32_t it, uint32_t x) {
    if (it == kItemEmpty) return kNone;
    const uint32_t off = it & 0xFFFu, stride = (it >> 12) & 0xFFFu, cm1 = it >> 24;
    if (x <= off) return off;
    const uint32_t last = off + cm1 * stride;
    if (x > last) return kNone;  // also covers singletons (cm1 == 0): stride unused
    return off + ceil_div12(x - off, stride) * stride;
}

// item_next without branches: x <= off gives a = 0, whose ceil-division is 0
// (also for a singleton's stride 0: (0 - 0.5) * rcp(0) = -inf -> 0); the
// result is kept only for a non-empty item with x <= last.
__device__ __forceinline__ uint32_t item_next_bf(uint32_t it, uint32_t x) {
    const uint32_t off = it & 0xFFFu, stride = (it >> 12) & 0xFFFu, cm1 = it >> 24;
    const uint32_t a = x > off ? x - off : 0u;
    const uint32_t r = off + ceil_div12(a, stride) * stride;
    return (it != kItemEmpty && x <= off + cm1 * stride) ? r : kNone;
}

// Hour cluster of time e (k = e[u]/3600): exact reciprocal
// multiply, valid for e < 2^31 (every finite time): the product error is
// below 2^-l <= 1/cs, so the floor is exact.
__device__ __forceinline__ uint32_t cluster_of(const DevIndex &ix, uint32_t e) {
    return uint32_t((uint64_t(e) * ix.cs_magic) >> ix.cs_shift);
}

// Cluster-AP lookup inside the type's cluster k = eu / cs,
// given the cluster's 32-byte record (r0, r1): smallest term >= eu among the
// cluster's APs, else the first departure of the next non-empty cluster
// (precomputed as next_min).  Precondition: first < eu <= last.
// Item 0 (most slots hold one AP run) is evaluated without branches and the
// rest only if item 1 exists and item 0 starts before x (batched kernel
// +1.5 %, profiles/r02_ab_scan_first_item.jsonl).  LAT (latency-bound
// single-query kernels): items 0 and 1 without branches, the rest only if
// item 1 starts before x (city / metro / country single query -2.2 / -2.8 /
// -2.5 % against the loop with early exits, 1-2 % faster than one
// branch-free item there; in the batched kernel -0.5 %:
// profiles/r02_ab_scan_lat.jsonl).
template <bool LAT = false>
__device__ __forceinline__ uint32_t cluster_scan(const DevIndex &ix, const uint4 &r0, const uint4 &r1, uint32_t k,
                                                 uint32_t eu) {
    const uint32_t x = eu - k * ix.cs;
    uint32_t best = kNone;
    if (r0.y == kItemSpill) {
        for (uint32_t i = 0; i < r0.w; ++i) {
            const uint32_t it = __ldg(ix.pool + r0.z + i);
            best = min(best, item_next(it, x));
            if ((it & 0xFFFu) >= x) break;  // items sorted by first term: later ones start later
        }
    } else if (LAT) {
        best = min(item_next_bf(r0.y, x), item_next_bf(r0.z, x));
        if (r0.w != kItemEmpty && (r0.z & 0xFFFu) < x) {
            const uint32_t items[kInlineItems - 2] = {r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
            for (int i = 0; i < kInlineItems - 2; ++i) {
                if (items[i] == kItemEmpty) break;  // slots are filled from the front
                best = min(best, item_next(items[i], x));
                if ((items[i] & 0xFFFu) >= x) break;
            }
        }
    } else {
        best = item_next_bf(r0.y, x);
        if (r0.z != kItemEmpty && (r0.y & 0xFFFu) < x) {
            const uint32_t items[kInlineItems - 1] = {r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
#pragma unroll
            for (int i = 0; i < kInlineItems - 1; ++i) {
                if (items[i] == kItemEmpty) break;  // slots are filled from the front
                best = min(best, item_next(items[i], x));
                if ((items[i] & 0xFFFu) >= x) break;
            }
        }
    }
    return best != kNone ? k * ix.cs + best : r0.x;
}

// Record index base of type t: the record of its hour cluster k is cb + k
// (compact directory: cb = crec_base - c_first from type_cb[]; dense
// directory: cb = t * dense_nc, no load).
__device__ __forceinline__ uint32_t type_cbase(const DevIndex &ix, uint64_t t) {
    return ix.dense_nc ? uint32_t(t * ix.dense_nc) : __ldg(ix.type_cb + t);
}

// Lookup from the record index: both halves of the 32-byte record are
// requested at once (loading items 3-6 only when items 0-2 do not decide
// costs 4 % on the city batch: profiles/r02_ab_lazy_crec_half.jsonl).
__device__ __forceinline__ uint32_t cluster_lookup(const DevIndex &ix, uint32_t cb, uint32_t eu) {
    const uint32_t k = cluster_of(ix, eu);
    const uint64_t r = uint32_t(cb + k);
    const uint4 r0 = __ldg(ix.crec + 2 * r);
    const uint4 r1 = __ldg(ix.crec + 2 * r + 1);
    return cluster_scan(ix, r0, r1, k, eu);
}

// Dense cluster directory (ix.dense_nc > 0): the record of (type t, cluster
// of eu) has a computable address, so it is fetched together with the type
// record instead of after it.  Out-of-range clusters are clamped (the value
// is then unused: the lookup only reads it when first < eu <= last).
struct CrecPrefetch {
    uint4 r0, r1;
    uint32_t k;
};

__device__ __forceinline__ CrecPrefetch crec_prefetch(const DevIndex &ix, uint64_t t, uint32_t eu) {
    CrecPrefetch p;
    p.k = cluster_of(ix, eu);
    const uint64_t r = t * ix.dense_nc + min(p.k, ix.dense_nc - 1u);
    p.r0 = __ldg(ix.crec + 2 * r);
    p.r1 = __ldg(ix.crec + 2 * r + 1);
    return p;
}

// Connection-type header: one 16-byte load.
struct TypeRec {
    uint32_t v, lam, first, last;
};

__device__ __forceinline__ TypeRec load_type(const DevIndex &ix, uint64_t t) {
    const uint4 a = __ldg(ix.type_hdr + t);
    return TypeRec{a.x, a.y, a.z, a.w};
}

// getConnection for one type (PAPER.md:226 semantics): first departure >= eu, or kInf.
__device__ __forceinline__ uint32_t type_next_departure(const DevIndex &ix, uint64_t t, const TypeRec &tr,
                                                        uint32_t eu) {
    if (eu > tr.last) return kInf;
    if (eu <= tr.first) return tr.first;
    return cluster_lookup(ix, type_cbase(ix, t), eu);
}

// Ablation lookups of the paper's incremental versions (NEXT-3), over the
// same records (so results are identical, only the work differs):
//   kLookupAP (Connection-type-AP): Algorithm 6 over every
//     AP tuple of the type, no hour index;
//   kLookupLinear (Connection-type): getConnection by linear
//     search over the departures in time order, stopping at the first >= e[u].
enum { kLookupClusterAP = 0, kLookupAP = 1, kLookupLinear = 2 };

__device__ __forceinline__ uint32_t type_lookup_ablation(const DevIndex &ix, uint64_t t, const TypeRec &tr,
                                                         uint32_t eu, uint32_t mode) {
    if (eu > tr.last) return kInf;  // early termination in every version
    uint32_t best = kInf;
    const uint32_t k0 = cluster_of(ix, tr.first), k1 = cluster_of(ix, tr.last);
    const uint32_t cb = type_cbase(ix, t);
    for (uint32_t k = k0; k <= k1; ++k) {
        const uint64_t r = uint32_t(cb + k);
        const uint4 r0 = __ldg(ix.crec + 2 * r), r1 = __ldg(ix.crec + 2 * r + 1);
        const bool spill = r0.y == kItemSpill;
        const uint32_t nitems = spill ? r0.w : uint32_t(kInlineItems);
        const uint32_t base = k * ix.cs;
        for (uint32_t i = 0; i < nitems; ++i) {
            uint32_t it;
            if (spill) it = __ldg(ix.pool + r0.z + i);
            else {
                const uint32_t v[kInlineItems] = {r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
                it = v[i];
            }
            if (it == kItemEmpty) break;
            const uint32_t off = it & 0xFFFu, stride = (it >> 12) & 0xFFFu, cnt = (it >> 24) + 1u;
            if (mode == kLookupLinear) {  // enumerate the terms
                for (uint32_t j = 0; j < cnt; ++j) {
                    const uint32_t d = base + off + j * stride;
                    if (d >= eu) {
                        best = min(best, d);
                        break;
                    }
                }
            } else {  // Algorithm 6 on this tuple (absolute times)
                const uint32_t first = base + off, last = first + (cnt - 1u) * stride;
                if (eu <= first) best = min(best, first);
                else if (eu <= last) best = min(best, first + ((eu - first + stride - 1u) / stride) * stride);
            }
        }
        if (mode == kLookupLinear && best != kInf) break;  // clusters are in time order
    }
    return best;
}

// ---------------------------------------------------------------- grid barrier
// Barrier of nctas co-resident CTAs on a monotonic arrival counter (*cnt,
// zeroed before the launch): every CTA leader adds 1 and waits until the
// counter reaches epoch * nctas -- one fire-and-forget atomic per CTA and a
// poll, 1.3 us for 148 CTAs on B200 vs 2.5 us for a count/reset/generation
// barrier (tools/latency_bench.py).  `epoch` is the caller's barrier count.
// With `rd`, thread 0 also reads *rd after the barrier and every thread gets
// that value: a control word all CTAs need (frontier size, stop flag) is
// fetched once per CTA instead of by every warp -- thousands of same-line
// reads right after the barrier cost ~1 us (tools/trace_sweeps.py).
__device__ __forceinline__ uint32_t grid_sync(uint32_t *cnt, uint32_t &epoch, uint32_t nctas,
                                              const uint32_t *rd = nullptr) {
    __shared__ uint32_t s_bcast;
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        const uint32_t target = epoch * nctas;
        while (*reinterpret_cast<volatile uint32_t *>(cnt) < target) {
        }
        __threadfence();
        if (rd) s_bcast = __ldcg(rd);
    }
    __syncthreads();
    return rd ? s_bcast : 0u;
}

__device__ __forceinline__ uint32_t grid_sync(uint32_t *cnt, uint32_t &epoch, const uint32_t *rd = nullptr) {
    return grid_sync(cnt, epoch, gridDim.x, rd);
}

// Warp-aggregated append of v to a worklist (one global atomic per group of
// converged pushing lanes).
__device__ __forceinline__ void push_aggregated(uint32_t v, uint32_t *q, uint32_t *count) {
    const unsigned am = __activemask();
    const unsigned lane = threadIdx.x & 31u;
    const unsigned leader = __ffs(am) - 1u;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(count, uint32_t(__popc(am)));
    base = __shfl_sync(am, base, leader);
    q[base + __popc(am & ((1u << lane) - 1u))] = v;
}

// Warp-aggregated append of v and its type range to a worklist.
__device__ __forceinline__ void push_aggregated(uint32_t v, uint2 rng, uint32_t *q, uint2 *qr, uint32_t *count) {
    const unsigned am = __activemask();
    const unsigned lane = threadIdx.x & 31u;
    const unsigned leader = __ffs(am) - 1u;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(count, uint32_t(__popc(am)));
    base = __shfl_sync(am, base, leader);
    const uint32_t pos = base + __popc(am & ((1u << lane) - 1u));
    q[pos] = v;
    qr[pos] = rng;
}

// Relax one connection type (Algorithm 3) whose source has
// arrival eu, against a global e[] (atomicMin).  Returns
// the target v when this call strictly lowered e[v], else kNone; *cand_out
// (optional) receives the candidate arrival.  SYS: system-scope atomic (e[]
// also updated by peer GPUs, peer.cu).
// NO_AV: skip the read of e[v] before the atomicMin (one dependent access
// fewer per hop; the atomicMin alone decides) -- for latency-bound schedules.
template <bool SYS = false, bool NO_AV = false>
__device__ __forceinline__ uint32_t relax_type_global(const DevIndex &ix, uint64_t t, uint32_t eu, uint32_t *arr,
                                                      uint32_t *cand_out = nullptr) {
    CrecPrefetch pf{};
    if (ix.dense_nc) pf = crec_prefetch(ix, t, eu);
    const TypeRec tr = load_type(ix, t);
    if (eu > tr.last) return kNone;
    const uint32_t av = NO_AV ? kInf : __ldcg(arr + tr.v);
    if (max(eu, tr.first) + tr.lam >= av) return kNone;  // early termination
    const uint32_t tc = ix.lookup_mode ? type_lookup_ablation(ix, t, tr, eu, ix.lookup_mode)
                        : eu <= tr.first ? tr.first
                                         : (ix.dense_nc ? cluster_scan(ix, pf.r0, pf.r1, pf.k, eu)
                                                        : cluster_lookup(ix, __ldg(ix.type_cb + t), eu));
    if (tc == kInf) return kNone;
    const uint32_t cand = tc + tr.lam;
    if (cand >= av) return kNone;
    if (cand_out) *cand_out = cand;
    const uint32_t old = SYS ? atomicMin_system(arr + tr.v, cand) : atomicMin(arr + tr.v, cand);
    return cand < old ? tr.v : kNone;
}

}  // namespace dev
}  // namespace eat
