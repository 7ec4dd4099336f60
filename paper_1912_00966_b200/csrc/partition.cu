// partition.cu -- edge-partitioned single query.
//
// Rank g owns the out-types of internal vertices [lo, hi) (contiguous after
// locality renumbering, balanced by type count) and a full e[] replica.  A
// query runs in exchange rounds:
//   1. local phase (k_part_round): the frontier is every owned v whose e[v]
//      dropped since the last exchange (e[v] < prev[v]); sweeps of the
//      Cluster-AP relaxation (same lookup as kernels.cu) run until the local
//      frontier is empty (or for a fixed number of sweeps); lowering a vertex
//      another rank owns sets the "remote" flag;
//   2. exchange: ncclAllReduce(min) over e[] ++ flag word (n+1 uint32) --
//      EAT_INF = 0x7FFFFFFF orders identically as uint32 and int32;
//   3. stop when no rank lowered a non-owned vertex (flag word stays 1).
// The fixpoint is the same as the single-GPU sweep's (relaxations commute
// under min), so results are bit-identical.
#include <algorithm>
#include <thread>

#include "device_common.cuh"
#include "partition.cuh"

namespace eat {
namespace {

using namespace dev;

constexpr int kPartThreads = 1024;  // one CTA per SM, as the grid kernels

template <int SW>
__global__ void __launch_bounds__(kPartThreads) k_part_round(DevIndex ix, PartWork w, uint32_t lo, uint32_t hi,
                                                             int first, uint32_t s, uint32_t ts) {
    const uint32_t n = ix.n;
    const uint64_t gtid = blockIdx.x * uint64_t(kPartThreads) + threadIdx.x;
    const uint64_t gsz = uint64_t(gridDim.x) * kPartThreads;
    uint32_t *bar = w.ctl + kBarWord;  // monotonic barrier counter (zeroed per launch)
    uint32_t bar_epoch = 0;
    if (first) {
        for (uint64_t i = gtid; i < n; i += gsz) {
            w.arr[i] = kInf;
            w.prev[i] = kInf;
            w.stamp[i] = 0;
        }
        if (gtid == 0) w.ctl[8] = 0, w.ctl[10] = 0;
        grid_sync(bar, bar_epoch);
        if (gtid == 0) w.arr[__ldg(ix.perm + s)] = ts;  // caller id -> internal id
    }
    if (gtid == 0) {
        w.arr[n] = 1u;  // exchange flag: 1 = no remote vertex lowered by this rank
        w.ctl[0] = 0;
        w.ctl[1] = 0;
        w.ctl[2] = 0;
    }
    grid_sync(bar, bar_epoch);
    // initial local frontier: owned vertices lowered since the last exchange
    for (uint64_t v = lo + gtid; v < hi; v += gsz)
        if (ld_cg(w.arr + v) < ld_cg(w.prev + v)) push_aggregated(uint32_t(v), w.q0, w.ctl + 0);
    uint32_t cnt_cur = grid_sync(bar, bar_epoch, w.ctl + 0);  // sweep 0's frontier size
    const uint32_t base = ld_cg(w.ctl + 10);
    bool remote = false;
    uint32_t sweep = 0;
    const uint32_t wl = threadIdx.x & 31u;
    for (;;) {
        const uint32_t c_nxt = (sweep + 1u) % 3u, c_old = (sweep + 2u) % 3u;
        if (gtid == 0) w.ctl[c_old] = 0;
        const uint32_t cnt = cnt_cur;
        // half-warps per vertex when the frontier outnumbers the warps (as kernels.cu)
        const uint32_t sw = (SW == 32 && cnt > uint32_t(gsz >> 5)) ? 16u : uint32_t(SW);
        const uint32_t lane = uint32_t(gtid & (sw - 1u));
        const unsigned smask = sw == 32u ? 0xFFFFFFFFu : (((1u << sw) - 1u) << (wl & ~(sw - 1u)));
        const uint32_t *qc = (sweep & 1u) ? w.q1 : w.q0;
        uint32_t *qn = (sweep & 1u) ? w.q0 : w.q1;
        const uint32_t stamp = base + sweep + 1u;
        // continuation as in the grid frontier kernel (kernels.cu): an owned
        // vertex lowered by this sub-warp is relaxed by it in the same sweep
        // (up to ix.cont_budget extra vertices per frontier vertex)
        for (uint64_t it = gtid / sw; it < cnt; it += gsz / sw) {
            uint32_t x = ld_cg(qc + it);
            uint32_t budget = ix.cont_budget;
            uint32_t eu = ld_cg(w.arr + x);
            uint32_t p0 = __ldg(ix.type_ptr + x), p1 = __ldg(ix.type_ptr + x + 1);
            for (;;) {
                uint32_t cv = kNone;
                for (uint32_t t = p0 + lane; t < p1; t += sw) {
                    const uint32_t v = relax_type_global(ix, t, eu, w.arr);
                    if (v == kNone) continue;
                    if (v >= lo && v < hi) {
                        if (budget > 0 && cv == kNone) cv = v;
                        else if (atomicExch(w.stamp + v, stamp) != stamp) push_aggregated(v, qn, w.ctl + c_nxt);
                    } else {
                        remote = true;
                    }
                }
                const unsigned cm = __ballot_sync(smask, cv != kNone) & smask;
                if (!cm) break;
                const uint32_t src = __ffs(cm) - 1u;
                x = __shfl_sync(smask, cv, src);
                // the next hop's loads go out before this hop's queue pushes
                eu = ld_cg(w.arr + x);
                p0 = __ldg(ix.type_ptr + x);
                p1 = __ldg(ix.type_ptr + x + 1);
                if (cv != kNone && wl != src && atomicExch(w.stamp + cv, stamp) != stamp)
                    push_aggregated(cv, qn, w.ctl + c_nxt);
                --budget;
            }
        }
        cnt_cur = grid_sync(bar, bar_epoch, w.ctl + c_nxt);
        ++sweep;
        if (cnt_cur == 0u) break;
        if (w.local_sweeps_per_round && sweep >= w.local_sweeps_per_round) {
            // bounded local phase: leftover frontier vertices stay "lowered since
            // the last exchange" only if prev is not refreshed for them, so
            // force them into the next round by invalidating their prev entry.
            const uint32_t left = ld_cg(w.ctl + c_nxt);
            const uint32_t *ql = (sweep & 1u) ? w.q1 : w.q0;
            for (uint64_t it = gtid; it < left; it += gsz) w.stamp[ld_cg(ql + it)] = 0xFFFFFFFFu;
            break;
        }
    }
    if (__any_sync(0xFFFFFFFFu, remote) && (threadIdx.x & 31u) == 0) atomicExch(w.arr + n, 0u);
    grid_sync(bar, bar_epoch);
    // prev := what this rank contributes to the exchange; vertices left on a
    // bounded local frontier (stamp == ~0) keep prev = INF so they re-enter.
    for (uint64_t i = gtid; i < n; i += gsz) {
        const bool left = w.local_sweeps_per_round && ld_cg(w.stamp + i) == 0xFFFFFFFFu;
        w.prev[i] = left ? kInf : ld_cg(w.arr + i);
        if (left) {
            w.stamp[i] = 0;
            atomicExch(w.arr + n, 0u);
        }
    }
    if (gtid == 0) {
        w.ctl[8] += sweep;
        w.ctl[10] = base + sweep + 1u;
    }
}

__global__ void k_min_merge(uint32_t *dst, const uint32_t *src, uint64_t count) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < count; i += uint64_t(gridDim.x) * blockDim.x)
        dst[i] = min(dst[i], src[i]);
}

__global__ void k_gather(DevIndex ix, const uint32_t *arr, uint32_t *out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < ix.n; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = arr[ix.perm[i]];
}

template <int SW>
cudaError_t launch_round_sw(const DevIndex &ix, const PartWork &w, uint32_t lo, uint32_t hi, bool first, uint32_t s,
                            uint32_t ts, cudaStream_t st) {
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_part_round<SW>, kPartThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    per_sm = std::min(per_sm, grid_ctas_per_sm());
    DevIndex ixc = ix;
    PartWork wc = w;
    int f = first ? 1 : 0;
    void *args[] = {&ixc, &wc, &lo, &hi, &f, &s, &ts};
    return cudaLaunchCooperativeKernel((const void *)k_part_round<SW>, dim3(unsigned(sms * per_sm)),
                                       dim3(kPartThreads), args, 0, st);
}

}  // namespace

cudaError_t part_alloc(PartWork &w, uint32_t n) {
    w.n = n;
    cudaError_t e;
    if ((e = cudaMalloc(&w.arr, (n + 1ull) * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.prev, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.q0, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.q1, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.stamp, n * 4ull + 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.ctl, kCtlWords * 4)) != cudaSuccess) return e;
    if ((e = cudaMemset(w.ctl, 0, kCtlWords * 4)) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&w.h_flag, 64)) != cudaSuccess) return e;
    return cudaSuccess;
}

void part_free(PartWork &w) {
    void *ptrs[] = {w.arr, w.prev, w.q0, w.q1, w.stamp, w.ctl};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    if (w.h_flag) cudaFreeHost(w.h_flag);
    w = PartWork{};
}

cudaError_t launch_part_round(const DevIndex &ix, const PartWork &w, uint32_t lo, uint32_t hi, int subwarp,
                              bool first, uint32_t s, uint32_t t_s, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(w.ctl + kBarWord, 0, sizeof(uint32_t), st);
    if (e != cudaSuccess) return e;
    switch (subwarp) {
        case 0: return launch_round_sw<8>(ix, w, lo, hi, first, s, t_s, st);
        case 1: return launch_round_sw<1>(ix, w, lo, hi, first, s, t_s, st);
        case 2: return launch_round_sw<2>(ix, w, lo, hi, first, s, t_s, st);
        case 4: return launch_round_sw<4>(ix, w, lo, hi, first, s, t_s, st);
        case 8: return launch_round_sw<8>(ix, w, lo, hi, first, s, t_s, st);
        case 16: return launch_round_sw<16>(ix, w, lo, hi, first, s, t_s, st);
        case 32: return launch_round_sw<32>(ix, w, lo, hi, first, s, t_s, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_min_merge(uint32_t *dst, const uint32_t *src, uint64_t count, cudaStream_t st) {
    if (!count) return cudaSuccess;
    k_min_merge<<<unsigned(std::min<uint64_t>((count + 255) / 256, 148 * 16)), 256, 0, st>>>(dst, src, count);
    return cudaGetLastError();
}

cudaError_t launch_gather(const DevIndex &ix, const uint32_t *arr, uint32_t *out, cudaStream_t st) {
    k_gather<<<unsigned(std::min<uint64_t>((ix.n + 255) / 256, 148 * 16)), 256, 0, st>>>(ix, arr, out);
    return cudaGetLastError();
}

// Wait for stream st while polling the communicator for asynchronous
// errors (a failed or aborted peer), so a rank never blocks forever in
// cudaStreamSynchronize behind a collective that cannot complete.
eat_status wait_polling(cudaStream_t st, ncclComm_t comm, std::string &err) {
    for (uint64_t spin = 0;; ++spin) {
        const cudaError_t e = cudaStreamQuery(st);
        if (e == cudaSuccess) return EAT_OK;
        if (e != cudaErrorNotReady) {
            err = std::string("round sync: ") + cudaGetErrorString(e);
            return EAT_ECUDA;
        }
        if (comm && (spin & 63u) == 0) {
            ncclResult_t ae = ncclSuccess;
            const ncclResult_t r = ncclCommGetAsyncError(comm, &ae);
            if (r != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress)) {
                err = std::string("NCCL asynchronous error: ") + ncclGetErrorString(r != ncclSuccess ? r : ae);
                ncclCommAbort(comm);  // unblocks the stream; the communicator is unusable afterwards
                return EAT_ENCCL;
            }
        }
        if (spin > 64) std::this_thread::yield();
    }
}

eat_status part_query(const DevIndex &ix, PartWork &w, ncclComm_t comm, uint32_t lo, uint32_t hi, int subwarp,
                      uint32_t s, uint32_t t_s, uint32_t *d_out, cudaStream_t st, uint32_t *rounds, uint32_t *sweeps,
                      std::string &err) {
    auto cuda_fail = [&](cudaError_t e, const char *what) {
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return EAT_ECUDA;
    };
    cudaError_t e;
    uint32_t r = 0;
    for (;; ++r) {
        if ((e = launch_part_round(ix, w, lo, hi, subwarp, r == 0, s, t_s, st)) != cudaSuccess)
            return cuda_fail(e, "part round");
        if (comm) {
            ncclResult_t nr = ncclAllReduce(w.arr, w.arr, size_t(ix.n) + 1, ncclUint32, ncclMin, comm, st);
            if (nr != ncclSuccess) {
                err = std::string("ncclAllReduce: ") + ncclGetErrorString(nr);
                return EAT_ENCCL;
            }
        }
        if ((e = cudaMemcpyAsync(w.h_flag, w.arr + ix.n, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
            return cuda_fail(e, "flag copy");
        const eat_status ws = wait_polling(st, comm, err);
        if (ws != EAT_OK) {
            if (ws == EAT_ENCCL) w.comm_dead = true;
            return ws;
        }
        if (w.h_flag[0] == 1u) break;
        if (r > 4u * ix.n + 16u) {
            err = "edge-partitioned query did not converge";
            return EAT_ECUDA;
        }
    }
    if ((e = launch_gather(ix, w.arr, d_out, st)) != cudaSuccess) return cuda_fail(e, "gather");
    if ((e = cudaMemcpyAsync(w.h_flag + 1, w.ctl + 8, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        return cuda_fail(e, "sweeps copy");
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "final sync");
    w.h_sweeps = w.h_flag[1];
    if (rounds) *rounds = r + 1;
    if (sweeps) *sweeps = w.h_sweeps;
    return EAT_OK;
}

eat_status part_query_loopback(const std::vector<DevIndex> &ix, std::vector<PartWork *> &w,
                               const std::vector<uint32_t> &lo, const std::vector<uint32_t> &hi, int subwarp,
                               uint32_t s, uint32_t t_s, uint32_t *d_out, cudaStream_t st, uint32_t *rounds,
                               uint32_t *sweeps, std::string &err) {
    auto cuda_fail = [&](cudaError_t e, const char *what) {
        err = std::string(what) + ": " + cudaGetErrorString(e);
        return EAT_ECUDA;
    };
    const size_t P = ix.size();
    const uint64_t words = uint64_t(ix[0].n) + 1;
    cudaError_t e;
    uint32_t r = 0;
    for (;; ++r) {
        for (size_t p = 0; p < P; ++p)
            if ((e = launch_part_round(ix[p], *w[p], lo[p], hi[p], subwarp, r == 0, s, t_s, st)) != cudaSuccess)
                return cuda_fail(e, "part round");
        // exchange: min over partitions of e[] ++ flag, then broadcast
        for (size_t p = 1; p < P; ++p)
            if ((e = launch_min_merge(w[0]->arr, w[p]->arr, words, st)) != cudaSuccess) return cuda_fail(e, "min merge");
        for (size_t p = 1; p < P; ++p)
            if ((e = cudaMemcpyAsync(w[p]->arr, w[0]->arr, words * 4, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
                return cuda_fail(e, "broadcast");
        if ((e = cudaMemcpyAsync(w[0]->h_flag, w[0]->arr + ix[0].n, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
            return cuda_fail(e, "flag copy");
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "round sync");
        if (w[0]->h_flag[0] == 1u) break;
        if (r > 4u * ix[0].n + 16u) {
            err = "edge-partitioned query did not converge";
            return EAT_ECUDA;
        }
    }
    if ((e = launch_gather(ix[0], w[0]->arr, d_out, st)) != cudaSuccess) return cuda_fail(e, "gather");
    uint32_t total = 0;
    for (size_t p = 0; p < P; ++p) {
        if ((e = cudaMemcpyAsync(w[p]->h_flag + 1, w[p]->ctl + 8, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
            return cuda_fail(e, "sweeps copy");
    }
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_fail(e, "final sync");
    for (size_t p = 0; p < P; ++p) total = std::max(total, w[p]->h_flag[1]);
    if (rounds) *rounds = r + 1;
    if (sweeps) *sweeps = total;
    return EAT_OK;
}

}  // namespace eat
