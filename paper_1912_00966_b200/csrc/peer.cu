// peer.cu -- edge-partitioned single query with an in-kernel exchange over
// peer memory (NEXT-2).  See peer.cuh for the layout and deployments.
//
// One query = rounds.  In round r every partition p:
//   1. drains the inbox of round r-1 (owned vertices another partition
//      lowered) into its local frontier;
//   2. runs frontier sweeps over its owned sources to local quiescence (the
//      Cluster-AP relaxation of kernels.cu, with continuation), separated by
//      barriers of its own CTA group.  An owned target is lowered in the
//      local replica; any other target is lowered in the local replica and,
//      if that improved it, in the owner's e[] with a system-scope atomicMin
//      through the peer pointer -- and if the owner's value improved, the
//      vertex is appended (once per round, flag) to the owner's inbox;
//   3. meets every partition at a cross-partition barrier; the query ends
//      after the first round in which no partition sent a message.
// Correctness: every lowering of e[v] by a non-owner either is followed by a
// message (so the owner relaxes v again with the lowered value) or happens
// while v is already queued for the next round; local phases reach
// quiescence; so "no message in a round" means no vertex has pending work,
// i.e. the fixpoint -- which is unique, so results
// are bit-identical to every other kernel's.
#include <algorithm>
#include <cuda/atomic>

#include "device_common.cuh"
#include "peer.cuh"

namespace eat {
namespace {

using namespace dev;

constexpr int kPeerThreads = 1024;  // one CTA per SM per group, as the grid kernels

__device__ __forceinline__ uint32_t ld_sys(uint32_t *p) {
    return cuda::atomic_ref<uint32_t, cuda::thread_scope_system>(*p).load(cuda::memory_order_relaxed);
}

// Barrier of all partitions (every group of every launch, possibly on other
// GPUs): the group meets, then its leader meets the other leaders on the
// system-scope counter pair in partition 0's block, then the group meets again.
__device__ __forceinline__ void peer_sync(uint32_t *lbar, uint32_t &lep, uint32_t nctas, uint32_t *gctl, uint32_t P,
                                          bool leader) {
    __threadfence_system();  // this thread's peer writes before anyone leaves the barrier
    grid_sync(lbar, lep, nctas);
    if (leader && threadIdx.x == 0) {
        cuda::atomic_ref<uint32_t, cuda::thread_scope_system> cnt(gctl[0]);
        cuda::atomic_ref<uint32_t, cuda::thread_scope_system> gen(gctl[1]);
        const uint32_t g = gen.load(cuda::memory_order_relaxed);
        __threadfence_system();
        if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == P - 1u) {
            cnt.store(0u, cuda::memory_order_relaxed);
            gen.fetch_add(1u, cuda::memory_order_release);
        } else {
            while (gen.load(cuda::memory_order_acquire) == g) {
            }
        }
        __threadfence_system();
    }
    grid_sync(lbar, lep, nctas);
}

__device__ __forceinline__ uint32_t owner_of(const PeerCtx &ctx, uint32_t v) {
    uint32_t o = 0;
    while (o + 1u < ctx.P && v >= ctx.part[o].hi) ++o;
    return o;
}

template <int SW>
__global__ void __launch_bounds__(kPeerThreads) k_peer_query(const DevIndex *__restrict__ ixs,
                                                             const PeerCtx *__restrict__ ctxp, PeerLocal *locs,
                                                             uint32_t s, uint32_t ts) {
    const PeerCtx &ctx = *ctxp;
    const uint32_t cpg = ctx.ctas_per_group;
    const uint32_t g = blockIdx.x / cpg, crank = blockIdx.x % cpg;
    const uint32_t p = ctx.part0 + g;
    const DevIndex &ix = ixs[g];
    const PeerLocal loc = locs[g];
    const PeerPart me = ctx.part[p];
    const uint32_t n = ix.n, lo = me.lo, hi = me.hi, own = hi - lo;
    const uint64_t gtid = uint64_t(crank) * kPeerThreads + threadIdx.x, gsz = uint64_t(cpg) * kPeerThreads;
    uint32_t *lbar = loc.ctl + kBarWord;  // the group's monotonic barrier counter (zeroed per launch)
    uint32_t lep = 0;
    const bool leader = crank == 0;
    const uint32_t rbase = ld_cg(loc.ctl + 10);  // absolute round of this query's round 0 (slots, parity)

    // The previous query's k_peer_gather on another rank may still read this
    // block's e[] through its IPC mapping: no partition re-initializes before
    // every partition has entered this query (its gather is stream-ordered
    // before this launch).
    peer_sync(lbar, lep, cpg, ctx.gctl, ctx.P, leader);
    // ---- Initialize (Algorithm 2): every replica, flags, frontier
    for (uint64_t i = gtid; i < n; i += gsz) {
        me.arr[i] = kInf;
        loc.stamp[i] = 0;
    }
    for (uint64_t i = gtid; i < 2ull * own; i += gsz) me.inflag[i] = 0;
    if (gtid == 0) {
        loc.ctl[0] = loc.ctl[1] = loc.ctl[2] = 0;
        me.inbox_cnt[0] = me.inbox_cnt[1] = 0;
    }
    peer_sync(lbar, lep, cpg, ctx.gctl, ctx.P, leader);  // nobody relaxes into a replica before it is initialized
    if (gtid == 0) {
        const uint32_t si = __ldg(ix.perm + s);  // caller id -> internal id
        if (si >= lo && si < hi) {
            me.arr[si] = ts;
            loc.q0[0] = si;
            loc.ctl[0] = 1;
        }
    }
    grid_sync(lbar, lep, cpg);

    const uint32_t wl = threadIdx.x & 31u;
    uint32_t sweep = 0, r = 0;
    for (;; ++r) {
        const uint32_t ra = rbase + r, pin = ra & 1u;
        // ---- 1. drain the previous round's inbox into this sweep's queue
        if (r > 0) {
            const uint32_t pp = pin ^ 1u;
            const uint32_t k = ld_sys(me.inbox_cnt + pp);
            uint32_t *qc = (sweep & 1u) ? loc.q1 : loc.q0;
            for (uint64_t i = gtid; i < k; i += gsz) {
                const uint32_t v = ld_sys(me.inbox + uint64_t(pp) * own + i);
                me.inflag[uint64_t(pp) * own + (v - lo)] = 0u;
                if (atomicExch(loc.stamp + v, sweep) != sweep) push_aggregated(v, qc, loc.ctl + sweep % 3u);
            }
        }
        if (p == 0 && leader && threadIdx.x == 0)  // message slot of the next round (read two barriers ago)
            cuda::atomic_ref<uint32_t, cuda::thread_scope_system>(ctx.gctl[2 + (ra + 1u) % 3u])
                .store(0u, cuda::memory_order_relaxed);
        uint32_t cnt_cur = grid_sync(lbar, lep, cpg, loc.ctl + sweep % 3u);  // this sweep's frontier size
        if (r > 0 && gtid == 0) me.inbox_cnt[pin ^ 1u] = 0;  // refilled only in round r+1

        // ---- 2. local sweeps to quiescence
        uint32_t nmsg = 0;
        for (;;) {
            const uint32_t c_nxt = (sweep + 1u) % 3u, c_old = (sweep + 2u) % 3u;
            if (gtid == 0) loc.ctl[c_old] = 0;
            const uint32_t cnt = cnt_cur;
            // half-warps per vertex when the frontier outnumbers the warps (as kernels.cu)
            const uint32_t sw = (SW == 32 && cnt > uint32_t(gsz >> 5)) ? 16u : uint32_t(SW);
            const uint32_t lane = uint32_t(gtid & (sw - 1u));
            const unsigned smask = sw == 32u ? 0xFFFFFFFFu : (((1u << sw) - 1u) << (wl & ~(sw - 1u)));
            const uint32_t *qc = (sweep & 1u) ? loc.q1 : loc.q0;
            uint32_t *qn = (sweep & 1u) ? loc.q0 : loc.q1;
            for (uint64_t it = gtid / sw; it < cnt; it += gsz / sw) {
                uint32_t x = ld_cg(qc + it);
                uint32_t budget = ix.cont_budget;
                uint32_t eu = ld_cg(me.arr + x);
                uint32_t p0 = __ldg(ix.type_ptr + x), p1 = __ldg(ix.type_ptr + x + 1);
                for (;;) {
                    uint32_t cv = kNone;
                    for (uint32_t t = p0 + lane; t < p1; t += sw) {
                        uint32_t cand;
                        const uint32_t v = relax_type_global<true>(ix, t, eu, me.arr, &cand);
                        if (v == kNone) continue;
                        if (v >= lo && v < hi) {  // owned: continue from it, or queue it
                            if (budget > 0 && cv == kNone) cv = v;
                            else if (atomicExch(loc.stamp + v, sweep + 1u) != sweep + 1u)
                                push_aggregated(v, qn, loc.ctl + c_nxt);
                            continue;
                        }
                        // owned elsewhere: lower the owner's e[v] through the peer pointer
                        const PeerPart &po = ctx.part[owner_of(ctx, v)];
                        if (cand < atomicMin_system(po.arr + v, cand)) {
                            const uint32_t own_o = po.hi - po.lo;
                            if (atomicExch_system(po.inflag + uint64_t(pin) * own_o + (v - po.lo), 1u) == 0u) {
                                const uint32_t pos = atomicAdd_system(po.inbox_cnt + pin, 1u);
                                po.inbox[uint64_t(pin) * own_o + pos] = v;
                                ++nmsg;
                            }
                        }
                    }
                    const unsigned cm = __ballot_sync(smask, cv != kNone) & smask;
                    if (!cm) break;
                    const uint32_t src = __ffs(cm) - 1u;
                    x = __shfl_sync(smask, cv, src);
                    // the next hop's loads go out before this hop's queue pushes
                    eu = ld_cg(me.arr + x);
                    p0 = __ldg(ix.type_ptr + x);
                    p1 = __ldg(ix.type_ptr + x + 1);
                    if (cv != kNone && wl != src && atomicExch(loc.stamp + cv, sweep + 1u) != sweep + 1u)
                        push_aggregated(cv, qn, loc.ctl + c_nxt);
                    --budget;
                }
            }
            cnt_cur = grid_sync(lbar, lep, cpg, loc.ctl + c_nxt);
            ++sweep;
            if (cnt_cur == 0u) break;
        }

        // ---- 3. exchange barrier; stop after a round without messages
        nmsg = __reduce_add_sync(0xFFFFFFFFu, nmsg);
        if (wl == 0 && nmsg) atomicAdd_system(ctx.gctl + 2 + ra % 3u, nmsg);
        peer_sync(lbar, lep, cpg, ctx.gctl, ctx.P, leader);
        if (ld_sys(ctx.gctl + 2 + ra % 3u) == 0u) break;
    }
    if (gtid == 0) {
        loc.ctl[8] = sweep;
        loc.ctl[9] = r + 1u;
        loc.ctl[10] = rbase + r + 1u;
    }
}

// out[i] = e[perm[i]] read from its owner's block (peer loads).
__global__ void k_peer_gather(const PeerCtx *__restrict__ ctxp, const uint32_t *__restrict__ perm, uint32_t n,
                              uint32_t *__restrict__ out) {
    const PeerCtx &ctx = *ctxp;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t v = __ldg(perm + i);
        out[i] = __ldcv(ctx.part[owner_of(ctx, v)].arr + v);
    }
}

template <int SW>
cudaError_t launch_peer_sw(const DevIndex *d_ix, const PeerCtx &ctx, const PeerCtx *d_ctx, PeerLocal *d_loc,
                           uint32_t s, uint32_t t_s, cudaStream_t st) {
    DevIndex *ixp = const_cast<DevIndex *>(d_ix);
    PeerCtx *cp = const_cast<PeerCtx *>(d_ctx);
    void *args[] = {&ixp, &cp, &d_loc, &s, &t_s};
    return cudaLaunchCooperativeKernel((const void *)k_peer_query<SW>, dim3(ctx.groups * ctx.ctas_per_group),
                                       dim3(kPeerThreads), args, 0, st);
}

}  // namespace

size_t peer_block_bytes(uint32_t n, uint32_t own) {
    return (size_t(n) + 4ull * own + 2 + 16) * sizeof(uint32_t);
}

PeerPart peer_part_view(void *base, uint32_t n, uint32_t lo, uint32_t hi) {
    uint32_t *b = static_cast<uint32_t *>(base);
    const uint64_t own = hi - lo;
    PeerPart pp{};
    pp.arr = b;
    pp.inflag = b + n;
    pp.inbox = b + n + 2 * own;
    pp.inbox_cnt = b + n + 4 * own;
    pp.lo = lo;
    pp.hi = hi;
    return pp;
}

uint32_t *peer_gctl(void *base0, uint32_t n, uint32_t own0) {
    return static_cast<uint32_t *>(base0) + n + 4ull * own0 + 2;
}

cudaError_t peer_local_alloc(PeerLocal &l, uint32_t n) {
    cudaError_t e;
    if ((e = cudaMalloc(&l.q0, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&l.q1, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&l.stamp, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&l.ctl, kCtlWords * 4)) != cudaSuccess) return e;
    return cudaMemset(l.ctl, 0, kCtlWords * 4);
}

void peer_local_free(PeerLocal &l) {
    void *ptrs[] = {l.q0, l.q1, l.stamp, l.ctl};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    l = PeerLocal{};
}

cudaError_t peer_query(const DevIndex *d_ix, const PeerCtx &ctx, const PeerCtx *d_ctx, const PeerLocal *h_loc,
                       PeerLocal *d_loc, const uint32_t *d_perm, uint32_t n, int subwarp, uint32_t s, uint32_t t_s,
                       uint32_t *d_out, cudaStream_t st) {
    cudaError_t e;
    for (uint32_t g = 0; g < ctx.groups; ++g)  // group barrier counters restart at 0
        if ((e = cudaMemsetAsync(h_loc[g].ctl + kBarWord, 0, sizeof(uint32_t), st)) != cudaSuccess) return e;
    switch (subwarp) {
        case 1: e = launch_peer_sw<1>(d_ix, ctx, d_ctx, d_loc, s, t_s, st); break;
        case 2: e = launch_peer_sw<2>(d_ix, ctx, d_ctx, d_loc, s, t_s, st); break;
        case 4: e = launch_peer_sw<4>(d_ix, ctx, d_ctx, d_loc, s, t_s, st); break;
        case 8: e = launch_peer_sw<8>(d_ix, ctx, d_ctx, d_loc, s, t_s, st); break;
        case 16: e = launch_peer_sw<16>(d_ix, ctx, d_ctx, d_loc, s, t_s, st); break;
        default: e = launch_peer_sw<32>(d_ix, ctx, d_ctx, d_loc, s, t_s, st); break;
    }
    if (e != cudaSuccess) return e;
    k_peer_gather<<<unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 8)), 256, 0, st>>>(d_ctx, d_perm, n, d_out);
    return cudaGetLastError();
}

// Resident CTAs per SM of the peer kernel (the cooperative launch needs them all resident).
int peer_ctas_per_sm() {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_peer_query<32>, kPeerThreads, 0);
    int v = per_sm;
    for (int sw : {1, 2, 4, 8, 16}) {
        int x = 0;
        switch (sw) {
            case 1: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, k_peer_query<1>, kPeerThreads, 0); break;
            case 2: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, k_peer_query<2>, kPeerThreads, 0); break;
            case 4: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, k_peer_query<4>, kPeerThreads, 0); break;
            case 8: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, k_peer_query<8>, kPeerThreads, 0); break;
            default: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&x, k_peer_query<16>, kPeerThreads, 0); break;
        }
        v = std::min(v, x);
    }
    return std::min(v, grid_ctas_per_sm());
}

}  // namespace eat
