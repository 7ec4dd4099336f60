// api.cu -- the C ABI of libeat.so (include/eat.h): handle lifecycle, device
// upload (north-star subsystem 2: SoA arrays packed for 128-bit loads),
// query drivers for the kernels in kernels.cu, and the edge-partitioned
// multi-GPU driver (NCCL min-allreduce of e[] per exchange round).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "eat.h"
#include "eat_internal.h"
#include "kernels.cuh"
#include "async.cuh"
#include "partition.cuh"
#include "peer.cuh"

namespace {

thread_local std::string g_err;

eat_status fail(eat_status s, const std::string &msg) {
    g_err = msg;
    return s;
}

#define CUDA_TRY(expr)                                                                           \
    do {                                                                                         \
        cudaError_t _e = (expr);                                                                 \
        if (_e != cudaSuccess)                                                                   \
            return fail(EAT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));          \
    } while (0)

#define NCCL_TRY(expr)                                                                           \
    do {                                                                                         \
        ncclResult_t _r = (expr);                                                                \
        if (_r != ncclSuccess) return fail(EAT_ENCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
    } while (0)

template <class T>
cudaError_t dalloc_copy(T **dst, const T *src, size_t count, size_t &bytes) {
    *dst = nullptr;
    size_t b = std::max<size_t>(count, 1) * sizeof(T);
    cudaError_t e = cudaMalloc(dst, b);
    if (e != cudaSuccess) return e;
    bytes += b;
    if (count) e = cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

}  // namespace

// One uploaded slice of the packed index: the out-types of internal
// sources [lo, hi) (everything for a replicated handle).
struct Slice {
    uint32_t lo = 0, hi = 0;
    uint32_t *type_ptr = nullptr, *type_hdr = nullptr, *type_cb = nullptr, *crec = nullptr, *pool = nullptr,
             *type_src = nullptr;
    eat::DevIndex ix{};
    eat::PartWork pw{};
    uint64_t num_crec = 0, num_pool = 0;
};

struct eat_handle {
    std::mutex mu;
    eat::HostIndex hx;
    bool host_only = false;
    int device = 0;
    uint32_t kernel = EAT_KERNEL_AUTO;   // resolved single-query kernel
    uint32_t subwarp = 8;
    uint32_t mode = EAT_MODE_REPLICATED;
    uint32_t window = EAT_INF;           // CTA schedule time window (EAT_INF = all active vertices)
    uint32_t group_window = EAT_INF;     // the same for batches on CTA groups (k_query_groups)
    uint32_t cta_threads = 320;          // CTA-kernel variant (batched queries)
    uint32_t lookup_mode = 0;            // 0 Cluster-AP; NEXT-3 ablations 1 (Connection-type-AP), 2 (linear)
    uint32_t cont_budget = 1;            // grid frontier kernel: continuation hops per frontier vertex
    std::vector<uint4> raw;              // EAT_KERNEL_CONNECTION: raw connections until upload
    uint4 *d_conns = nullptr;
    bool arr16 = true;                   // batched CTA kernel keeps e[] as uint16 offsets (+ uint32 recompute)
    uint32_t *d_ovf[3] = {nullptr, nullptr, nullptr};  // overflow lists: device API, pipeline stages 0/1
    uint64_t ovf_cap[3] = {0, 0, 0};
    cudaStream_t stream = nullptr;
    // device index: slices[0] is this handle's index (whole, or its own edge
    // partition); a loopback edge-partitioned handle holds all P partitions
    std::vector<Slice> slices;
    uint32_t *d_perm = nullptr;
    eat::DevIndex ix{};   // == slices[0].ix
    size_t index_bytes = 0;
    bool loopback = false;
    // single-query scratch
    eat::GridWork gw{};
    uint32_t *d_gacnt = nullptr;         // EAT_KERNEL_GRID_ASYNC: per-CTA counters
    std::vector<eat::GridWork> bgw;   // batched queries without shared-memory e[]: one scratch per CTA group
    eat::GridWork *d_bgw = nullptr;
    eat::AsyncWork aw{};
    uint32_t *d_out1 = nullptr, *h_out1 = nullptr;
    uint32_t *d_q1 = nullptr;  // [2]: s, t_s for the CTA kernel
    uint32_t *d_sweeps1 = nullptr;
    uint32_t *d_rounds1 = nullptr;   // async kernel: exchange rounds of the last query
    unsigned long long *d_counter = nullptr, *d_invalid = nullptr;
    unsigned long long *d_work = nullptr;  // EAT_BUILD_COUNTERS: 6 work counters
    // batched scratch: two pipeline stages (stream, queries, output rows, query counter, host staging)
    cudaStream_t bstream[2] = {nullptr, nullptr};
    uint32_t *d_bsrc[2] = {nullptr, nullptr}, *d_bts[2] = {nullptr, nullptr}, *d_bout[2] = {nullptr, nullptr};
    uint32_t *h_stage[2] = {nullptr, nullptr};
    unsigned long long *d_bcounter = nullptr;  // [2]
    cudaEvent_t bev[4] = {nullptr, nullptr, nullptr, nullptr};  // chunk kernel done [0..1], rows copied [2..3]
    // end of the last device work enqueued on this handle: the next call's
    // stream waits for it (the handle's scratch is shared, and two cooperative
    // grid kernels must never run concurrently)
    cudaEvent_t order_ev = nullptr;
    uint64_t bcap = 0, stage_cap = 0;
    // direct mode (pinned host output, CTA kernel): all queries in one launch,
    // rows stored by the kernel straight into the mapped host buffer
    uint32_t *d_dsrc = nullptr, *d_dts = nullptr;
    uint64_t dcap = 0;
    bool e2e_direct = true;
    // streamed mode (pinned output, batched CTA kernel): rows go to device
    // memory; per-chunk completion flags in mapped host memory let the host
    // copy finished chunks with the copy engine while the kernel still runs
    int e2e_mode = 1;                 // 0 chunk pipeline, 1 direct (kernel stores into mapped host rows), 2 streamed (-1.5 %: profiles/r02_e2e_modes.jsonl)
    uint32_t *d_srows = nullptr;      // [scap][n] device rows
    uint64_t scap = 0;
    unsigned int *h_done = nullptr, *d_done = nullptr;  // mapped per-query finished flags
    uint64_t done_cap = 0;
    int cta_grid = 0;
    uint32_t single_cta_threads = 1024;  // CTA variant of a lone query: 1024 when it fits, else cta_threads
    uint32_t cluster_ctas = 0;           // EAT_KERNEL_CLUSTER: CTAs per cluster (resolved at build)
    int cluster_stage = 0;               // ... index staged in shared memory (cluster.cu STAGE)
    bool cluster_async = true;           // EAT_KERNEL_CLUSTER: asynchronous (EAT_BUILD_CLUSTER_SYNC: sweeps)
    uint32_t cluster_window = EAT_INF;   // ... schedule window (all active vertices unless set: fastest, r02_cluster_*)
    uint32_t cluster_tl = 0;             // ... most types owned by one CTA
    bool batch_groups = false;  // batches on k_query_groups even when e[] fits shared memory (kernel FRONTIER)
    eat::SortScratch qsort[3];  // k_query_groups query order by source locality, per overflow/pipeline slot
    bool sort_batches = true;   // EAT_SORT_BATCHES=0 disables (A/B)
    // edge partition
    uint32_t part_rank = 0, part_count = 1, part_lo = 0, part_hi = 0;
    ncclComm_t comm = nullptr;
    // EAT_EXCHANGE_PEER (peer.cu): this process's exchange blocks (all P in
    // loopback), blocks of other ranks mapped by CUDA IPC, the launch context
    uint32_t exchange = EAT_EXCHANGE_ALLREDUCE;
    std::vector<void *> peer_own;     // blocks allocated here
    std::vector<void *> peer_mapped;  // blocks opened with cudaIpcOpenMemHandle (multi-process)
    std::vector<eat::PeerLocal> peer_loc;
    eat::PeerCtx peer_ctx{};
    eat::PeerCtx *d_peer_ctx = nullptr;
    eat::DevIndex *d_peer_ix = nullptr;
    eat::PeerLocal *d_peer_loc = nullptr;
    bool peer_ready = false;
    // EDGE_PARTITIONED + ALLREDUCE: local sweeps per exchange round (0 = to quiescence)
    uint32_t local_sweeps = 0;
    // REPLICATED on several devices: replicas of this handle on devices[1..]
    // (same index, own scratch); eat_query_many shards across {this} + replicas
    std::vector<eat_handle *> replicas;
    // stats
    eat_stats st{};
};

namespace {

// Scratch of one grid-kernel query (bitmaps only for the bitmap schedules).
cudaError_t gridwork_alloc(eat::GridWork &w, uint64_t n, bool bitmaps) {
    const uint64_t W = (n + 31ull) / 32ull;
    cudaError_t e;
    if ((e = cudaMalloc(&w.arr, n * 4ull)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.q0, n * 4ull)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.q1, n * 4ull)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.r0, n * 8ull)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.r1, n * 8ull)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.stamp, n * 4ull)) != cudaSuccess) return e;
    if (bitmaps && (e = cudaMalloc(&w.bm, 3 * W * 4ull)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&w.ctl, eat::kCtlWords * 4)) != cudaSuccess) return e;
    return cudaMemset(w.ctl, 0, eat::kCtlWords * 4);
}

void gridwork_free(eat::GridWork &w) {
    void *ptrs[] = {w.arr, w.q0, w.q1, w.r0, w.r1, w.stamp, w.bm, w.ctl};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    w = eat::GridWork{};
}

void release_device(eat_handle *h) {
    if (h->host_only) return;
    cudaSetDevice(h->device);
    gridwork_free(h->gw);
    if (h->d_gacnt) cudaFree(h->d_gacnt);
    h->d_gacnt = nullptr;
    for (eat::GridWork &w : h->bgw) gridwork_free(w);
    if (h->d_bgw) cudaFree(h->d_bgw);
    if (h->d_srows) cudaFree(h->d_srows);
    if (h->h_done) cudaFreeHost(h->h_done);
    void *ptrs[] = {h->d_perm,  h->d_out1, h->d_q1,      h->d_sweeps1,  h->d_counter,  h->d_invalid,
                    h->d_bsrc[0], h->d_bts[0], h->d_bout[0], h->d_bsrc[1], h->d_bts[1], h->d_bout[1],
                    h->d_bcounter, h->d_work, h->d_rounds1, h->d_ovf[0], h->d_ovf[1], h->d_ovf[2],
                    h->d_conns, h->d_dsrc, h->d_dts};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    eat::async_free(h->aw);
    for (eat::SortScratch &sc : h->qsort) eat::sort_scratch_free(sc);
    for (Slice &sl : h->slices) {
        void *sp[] = {sl.type_ptr, sl.type_hdr, sl.type_cb, sl.crec, sl.pool, sl.type_src};
        for (void *p : sp)
            if (p) cudaFree(p);
        eat::part_free(sl.pw);
    }
    if (h->h_out1) cudaFreeHost(h->h_out1);
    for (int i = 0; i < 2; ++i) {
        if (h->h_stage[i]) cudaFreeHost(h->h_stage[i]);
        if (h->bstream[i]) cudaStreamDestroy(h->bstream[i]);
    }
    for (cudaEvent_t ev : h->bev)
        if (ev) cudaEventDestroy(ev);
    if (h->order_ev) cudaEventDestroy(h->order_ev);
    if (h->comm) ncclCommDestroy(h->comm);
    for (void *p : h->peer_mapped)
        if (p) cudaIpcCloseMemHandle(p);
    for (void *p : h->peer_own)
        if (p) cudaFree(p);
    for (eat::PeerLocal &l : h->peer_loc) eat::peer_local_free(l);
    void *pp[] = {h->d_peer_ctx, h->d_peer_ix, h->d_peer_loc};
    for (void *p : pp)
        if (p) cudaFree(p);
    if (h->stream) cudaStreamDestroy(h->stream);
}

// Upload the out-types of internal sources [lo, hi) as one slice (offsets
// rebased to the slice).  type_ptr keeps all n+1 entries (empty outside).
eat_status upload_slice(eat_handle *h, uint32_t lo, uint32_t hi, Slice &sl) {
    const eat::HostIndex &x = h->hx;
    const uint32_t n = x.n;
    sl.lo = lo;
    sl.hi = hi;
    const uint32_t t_lo = x.type_ptr[lo], t_hi = x.type_ptr[hi];
    const uint64_t T = t_hi - t_lo;
    uint64_t r_lo = 0, r_hi = 0, p_lo = 0, p_hi = 0;
    if (T) {
        r_lo = x.type_rec[uint64_t(t_lo) * eat::kTypeWords + 4];
        r_hi = (t_hi < x.num_types) ? x.type_rec[uint64_t(t_hi) * eat::kTypeWords + 4] : x.num_crec;
        // pool range: spilled records in [r_lo, r_hi) are contiguous in pool order
        p_lo = x.pool.size();
        p_hi = 0;
        for (uint64_t r = r_lo; r < r_hi; ++r)
            if (x.crec[r * eat::kCrecWords + 1] == eat::kItemSpill) {
                p_lo = std::min<uint64_t>(p_lo, x.crec[r * eat::kCrecWords + 2]);
                p_hi = std::max<uint64_t>(p_hi, uint64_t(x.crec[r * eat::kCrecWords + 2]) + x.crec[r * eat::kCrecWords + 3]);
            }
        if (p_hi < p_lo) p_lo = p_hi = 0;
    }
    std::vector<uint32_t> tptr(uint64_t(n) + 1);
    for (uint64_t i = 0; i <= n; ++i) {
        uint32_t c = std::min(std::max(x.type_ptr[i], t_lo), t_hi);
        tptr[i] = c - t_lo;
    }
    // device type records: 16-byte headers {v, lambda, first, last} (one
    // 128-bit load), the cluster-record base crec_base - c_first in its own
    // array (read only by lookups), the source in type_src (full sweep only);
    // the host record's u and padding words never reach the device
    std::vector<uint32_t> thdr(4 * T), tcb(T), tsrc(T);
    for (uint64_t t = 0; t < T; ++t) {
        const uint32_t *r = x.type_rec.data() + (uint64_t(t_lo) + t) * eat::kTypeWords;
        for (int k = 0; k < 4; ++k) thdr[4 * t + k] = r[k];
        tcb[t] = (r[4] - uint32_t(r_lo)) - r[5];  // mod 2^32: cb + k with k >= c_first stays in range
        tsrc[t] = r[6];
    }
    std::vector<uint32_t> crec(x.crec.begin() + r_lo * eat::kCrecWords, x.crec.begin() + r_hi * eat::kCrecWords);
    for (uint64_t r = 0; r < r_hi - r_lo; ++r)
        if (crec[r * eat::kCrecWords + 1] == eat::kItemSpill) crec[r * eat::kCrecWords + 2] -= uint32_t(p_lo);
    size_t &b = h->index_bytes;
    CUDA_TRY(dalloc_copy(&sl.type_ptr, tptr.data(), tptr.size(), b));
    CUDA_TRY(dalloc_copy(&sl.type_hdr, thdr.data(), thdr.size(), b));
    CUDA_TRY(dalloc_copy(&sl.type_cb, tcb.data(), tcb.size(), b));
    CUDA_TRY(dalloc_copy(&sl.crec, crec.data(), crec.size(), b));
    CUDA_TRY(dalloc_copy(&sl.pool, x.pool.data() + p_lo, p_hi - p_lo, b));
    CUDA_TRY(dalloc_copy(&sl.type_src, tsrc.data(), tsrc.size(), b));
    sl.ix.n = n;
    sl.ix.cs = x.cs;
    sl.ix.dense_nc = x.dense_nc;
    sl.ix.lookup_mode = h->lookup_mode;
    sl.ix.cont_budget = h->cont_budget;
    sl.ix.zero = 0;
    {
        uint32_t l = 0;
        while ((1u << l) < x.cs) ++l;  // ceil(log2 cs)
        sl.ix.cs_shift = 31u + l;
        sl.ix.cs_magic = uint32_t((1ull << (31u + l)) / x.cs + 1ull);
    }
    sl.ix.window = h->window;
    sl.ix.cta_threads = h->cta_threads;
    sl.ix.num_types = T;
    sl.ix.type_ptr = sl.type_ptr;
    sl.ix.type_hdr = reinterpret_cast<const uint4 *>(sl.type_hdr);
    sl.ix.type_cb = sl.type_cb;
    sl.ix.crec = reinterpret_cast<const uint4 *>(sl.crec);
    sl.ix.pool = sl.pool;
    sl.ix.type_src = sl.type_src;
    sl.ix.perm = h->d_perm;
    sl.num_crec = r_hi - r_lo;
    sl.num_pool = p_hi - p_lo;
    return EAT_OK;
}

// Copy the peer launch context (and, once, the slices' indexes and the local
// scratch descriptors) to the device.
eat_status peer_publish(eat_handle *h) {
    const size_t G = h->slices.size();
    if (!h->d_peer_ctx) CUDA_TRY(cudaMalloc(&h->d_peer_ctx, sizeof(eat::PeerCtx)));
    if (!h->d_peer_ix) {
        std::vector<eat::DevIndex> ixs;
        for (const Slice &sl : h->slices) ixs.push_back(sl.ix);
        CUDA_TRY(cudaMalloc(&h->d_peer_ix, G * sizeof(eat::DevIndex)));
        CUDA_TRY(cudaMemcpy(h->d_peer_ix, ixs.data(), G * sizeof(eat::DevIndex), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMalloc(&h->d_peer_loc, G * sizeof(eat::PeerLocal)));
        CUDA_TRY(cudaMemcpy(h->d_peer_loc, h->peer_loc.data(), G * sizeof(eat::PeerLocal), cudaMemcpyHostToDevice));
    }
    CUDA_TRY(cudaMemcpy(h->d_peer_ctx, &h->peer_ctx, sizeof(eat::PeerCtx), cudaMemcpyHostToDevice));
    return EAT_OK;
}

// EAT_EXCHANGE_PEER: one zeroed exchange block per partition held here (all
// P in loopback, else this rank's; the others arrive with eat_peer_connect),
// local frontier scratch, the launch context.
eat_status peer_setup(eat_handle *h) {
    const eat::HostIndex &x = h->hx;
    const uint32_t n = x.n, P = h->part_count;
    if (P > eat::kMaxPeerParts) return fail(EAT_EINVAL, "EAT_EXCHANGE_PEER supports at most 16 partitions");
    eat::PeerCtx &c = h->peer_ctx;
    c = eat::PeerCtx{};
    c.P = P;
    c.groups = uint32_t(h->slices.size());
    c.part0 = h->loopback ? 0u : h->part_rank;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int per_sm = eat::peer_ctas_per_sm();
    if (per_sm < 1 || uint32_t(sms * per_sm) < c.groups) return fail(EAT_EUNSUPPORTED, "peer kernel does not fit the device");
    c.ctas_per_group = uint32_t(sms * per_sm) / c.groups;
    h->peer_loc.resize(c.groups);
    for (uint32_t g = 0; g < c.groups; ++g) {
        const uint32_t p = c.part0 + g;
        uint32_t lo = 0, hi = 0;
        eat::partition_range(x, p, P, lo, hi);
        void *blk = nullptr;
        CUDA_TRY(cudaMalloc(&blk, eat::peer_block_bytes(n, hi - lo)));
        h->peer_own.push_back(blk);
        CUDA_TRY(cudaMemset(blk, 0, eat::peer_block_bytes(n, hi - lo)));
        c.part[p] = eat::peer_part_view(blk, n, lo, hi);
        if (p == 0) c.gctl = eat::peer_gctl(blk, n, hi - lo);
        if (eat::peer_local_alloc(h->peer_loc[g], n) != cudaSuccess) return fail(EAT_ENOMEM, "cannot allocate peer scratch");
    }
    h->peer_ready = h->loopback || P == 1;
    return peer_publish(h);
}

eat_status upload(eat_handle *h) {
    const eat::HostIndex &x = h->hx;
    const uint32_t n = x.n;
    CUDA_TRY(dalloc_copy(&h->d_perm, x.perm.data(), x.perm.size(), h->index_bytes));
    uint32_t nslices = h->loopback ? h->part_count : 1;
    h->slices.resize(nslices);
    for (uint32_t r = 0; r < nslices; ++r) {
        uint32_t lo = 0, hi = n;
        if (h->mode == EAT_MODE_EDGE_PARTITIONED)
            eat::partition_range(x, h->loopback ? r : h->part_rank, h->part_count, lo, hi);
        eat_status e = upload_slice(h, lo, hi, h->slices[r]);
        if (e != EAT_OK) return e;
    }
    const Slice &s0 = h->slices[0];
    h->ix = s0.ix;
    h->part_lo = s0.lo;
    h->part_hi = s0.hi;
    h->st.num_types = s0.ix.num_types;
    h->st.num_cluster_records = s0.num_crec;
    h->st.num_spill_items = s0.num_pool;
    h->st.index_bytes = h->index_bytes;
    // scratch
    CUDA_TRY(gridwork_alloc(h->gw, n, true));
    CUDA_TRY(cudaMalloc(&h->d_out1, n * 4ull));
    CUDA_TRY(cudaMallocHost(&h->h_out1, n * 4ull + 64));
    CUDA_TRY(cudaMalloc(&h->d_q1, 2 * 4));
    CUDA_TRY(cudaMalloc(&h->d_sweeps1, 4));
    CUDA_TRY(cudaMemset(h->d_sweeps1, 0, 4));
    CUDA_TRY(cudaMalloc(&h->d_rounds1, 4));
    CUDA_TRY(cudaMemset(h->d_rounds1, 0, 4));
    CUDA_TRY(cudaMalloc(&h->d_counter, 8));
    CUDA_TRY(cudaMalloc(&h->d_invalid, 8));
    CUDA_TRY(cudaMemset(h->d_invalid, 0, 8));
    if (h->mode == EAT_MODE_EDGE_PARTITIONED && h->exchange == EAT_EXCHANGE_ALLREDUCE)
        for (Slice &sl : h->slices) {
            if (eat::part_alloc(sl.pw, n) != cudaSuccess) return fail(EAT_ENOMEM, "cannot allocate partition scratch");
            sl.pw.local_sweeps_per_round = h->local_sweeps;
        }
    if (h->mode == EAT_MODE_EDGE_PARTITIONED && h->exchange == EAT_EXCHANGE_PEER) return peer_setup(h);
    return EAT_OK;
}

// Edge-partitioned query on this handle: NCCL ranks, or all partitions of a
// loopback handle on one device.
eat_status run_partitioned(eat_handle *h, uint32_t s, uint32_t t_s, uint32_t *d_out, cudaStream_t st) {
    uint32_t rounds = 0, sweeps = 0;
    eat_status e;
    if (h->exchange == EAT_EXCHANGE_PEER) {
        if (!h->peer_ready) return fail(EAT_ESTATE, "EAT_EXCHANGE_PEER: call eat_peer_connect on every rank first");
        CUDA_TRY(eat::peer_query(h->d_peer_ix, h->peer_ctx, h->d_peer_ctx, h->peer_loc.data(), h->d_peer_loc, h->d_perm,
                                 h->hx.n, int(h->subwarp), s, t_s, d_out, st));
        uint32_t w[2] = {0, 0};
        CUDA_TRY(cudaMemcpyAsync(w, h->peer_loc[0].ctl + 8, 8, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        for (size_t g = 1; g < h->peer_loc.size(); ++g) {
            uint32_t sg = 0;
            CUDA_TRY(cudaMemcpy(&sg, h->peer_loc[g].ctl + 8, 4, cudaMemcpyDeviceToHost));
            w[0] = std::max(w[0], sg);
        }
        h->st.last_rounds = w[1];
        h->h_out1[h->hx.n] = w[0];
        CUDA_TRY(cudaMemcpyAsync(h->d_sweeps1, h->h_out1 + h->hx.n, 4, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        return EAT_OK;
    }
    if (h->loopback) {
        std::vector<eat::DevIndex> ixs;
        std::vector<eat::PartWork *> ws;
        std::vector<uint32_t> lo, hi;
        for (Slice &sl : h->slices) {
            ixs.push_back(sl.ix);
            ws.push_back(&sl.pw);
            lo.push_back(sl.lo);
            hi.push_back(sl.hi);
        }
        e = eat::part_query_loopback(ixs, ws, lo, hi, int(h->subwarp), s, t_s, d_out, st, &rounds, &sweeps, g_err);
    } else {
        Slice &sl = h->slices[0];
        if (h->part_count > 1 && !h->comm)
            return fail(EAT_ESTATE, "the NCCL communicator was aborted after an asynchronous error; rebuild the handle");
        e = eat::part_query(sl.ix, sl.pw, h->comm, sl.lo, sl.hi, int(h->subwarp), s, t_s, d_out, st, &rounds,
                            &sweeps, g_err);
        if (sl.pw.comm_dead) h->comm = nullptr;  // ncclCommAbort freed it
    }
    if (e != EAT_OK) return e;
    h->st.last_rounds = rounds;
    h->h_out1[h->hx.n] = sweeps;  // staged for d_sweeps1
    CUDA_TRY(cudaMemcpyAsync(h->d_sweeps1, h->h_out1 + h->hx.n, 4, cudaMemcpyHostToDevice, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    return EAT_OK;
}

// CTA groups (queries in flight) of the batched kernel when e[] does not fit
// shared memory: nq / 8, at most 296 (two 512-thread CTAs per group); metro
// 2,048 queries 19.8k q/s at 148-592 groups, country 512 queries best at 64
// (tools/sweep_groups.py, profiles/r01_sweep_group_shape.jsonl).
// EAT_BATCH_GROUPS overrides.
constexpr uint32_t kBatchGroupsMax = 296;

// Default time window of batches on CTA groups (e[] in global memory): metro
// 1,024 queries 46.4k q/s at 2400 s vs 43.6k at 1200 s and 38.5k at 600 or
// 7200 s (profiles/r02_ab_groups_flat_schedule.jsonl).  An explicit
// eat_build_opts.window_seconds applies to both batch kernels.
constexpr uint32_t kDefaultGroupWindow = 2400;

// Largest graph whose single queries AUTO runs on the one-CTA kernel.
constexpr uint32_t kAutoCtaMaxVertices = 2048;

// Most connection types owned by one CTA of a cs-CTA cluster (bitmap word w
// of 32 vertices belongs to CTA w mod cs; cluster.cu).
uint32_t cluster_tl_cap(const eat::HostIndex &hx, uint32_t cs) {
    const uint32_t n = hx.n, W = (n + 31u) / 32u;
    std::vector<uint64_t> cnt(cs, 0);
    for (uint32_t w = 0; w < W; ++w)
        cnt[w % cs] += hx.type_ptr[std::min(32u * w + 32u, n)] - hx.type_ptr[std::min(32u * w, n)];
    return uint32_t(std::min<uint64_t>(*std::max_element(cnt.begin(), cnt.end()), 0xFFFFFFFFu));
}

// EAT_KERNEL_CLUSTER configuration: the largest cluster (or `want` CTAs)
// the device schedules for this graph, at the deepest index staging that fits
// beside e[] and at least `min_stage`.  Sets cluster_ctas/stage/tl.
bool pick_cluster(eat_handle *h, uint32_t want, int min_stage) {
    const char *env = getenv("EAT_CLUSTER_STAGE");  // A/B knob: highest staging level tried
    const int max_stage = env ? std::max(0, std::min(2, atoi(env))) : 2;
    for (uint32_t c = 16; c >= 2; c >>= 1) {
        if (want && c != want) continue;
        const uint32_t tl = cluster_tl_cap(h->hx, c);
        for (int stg = max_stage; stg >= min_stage; --stg)
            if (eat::cluster_max_active(h->hx.n, int(c), stg, tl, h->cluster_async) > 0) {
                h->cluster_ctas = c;
                h->cluster_stage = stg;
                h->cluster_tl = tl;
                return true;
            }
    }
    h->cluster_ctas = 0;
    return false;
}

// EAT_KERNEL_GRID_ASYNC: fits (per-CTA slices in shared memory) + per-CTA counters.
bool pick_gasync(eat_handle *h) {
    const int G = eat::gasync_grid(h->hx.n);
    if (G < 1) return false;
    if (!h->d_gacnt && cudaMalloc(&h->d_gacnt, size_t(G) * eat::kGaCntWordsPerCta * sizeof(uint32_t)) != cudaSuccess) return false;
    return true;
}

eat_status resolve_kernel(eat_handle *h, uint32_t requested) {
    h->cta_grid = eat::cta_grid_size(h->hx.n, int(h->cta_threads), h->arr16);
    // a lone query takes the widest CTA (1024 threads, uint32 e[]) when its
    // larger static shared memory still fits beside e[]; else the batch variant
    h->single_cta_threads = eat::cta_grid_size(h->hx.n, 1024, false) > 0 ? 1024u : h->cta_threads;
    h->st.smem_vertices_max = 0;
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const size_t avail = size_t(optin) - eat::cta_static_smem() - 64;
    h->st.smem_vertices_max = uint32_t(avail * 32 / (4 * 32 + 2 * 4));
    uint32_t k = requested;
    const bool async_ok = eat::async_parts(h->hx.n) > 0;
    // AUTO for single queries: the one-CTA kernel for small graphs (tiny:
    // 0.08 vs 0.10 ms), else the grid frontier kernel (city 0.45 vs 0.64 ms,
    // and the only choice once e[] exceeds shared memory; faster than ASYNC
    // on metro/country).  Batches always use the CTA kernel
    // when e[] fits (throughput).
    if (k == EAT_KERNEL_AUTO) {
        if (h->cta_grid > 0 && h->hx.n <= kAutoCtaMaxVertices) k = EAT_KERNEL_CTA;
        // graphs whose whole index (e[], type ranges, headers, cluster bases)
        // fits the shared memory of a 16-CTA cluster: the asynchronous cluster
        // kernel -- city p50 0.50 -> 0.24 ms over 100 seeded queries
        // (profiles/r02_latency_kernels.jsonl)
        else if (h->mode == EAT_MODE_REPLICATED && pick_cluster(h, 16, 2)) k = EAT_KERNEL_CLUSTER;
        // else the barrier-free grid kernel (metro p50 1.04 -> ~0.7 ms, country
        // s0 2.09 -> ~1.1 ms vs FRONTIER; r02_gasync_*.jsonl)
        else if (h->mode == EAT_MODE_REPLICATED && pick_gasync(h)) k = EAT_KERNEL_GRID_ASYNC;
        else k = EAT_KERNEL_FRONTIER;
    }
    else if (k == EAT_KERNEL_FRONTIER)
        h->batch_groups = true;  // explicit FRONTIER: batches use its schedule too (grouped grid kernel)
    if (k == EAT_KERNEL_CTA && (h->cta_grid == 0 || eat::cta_grid_size(h->hx.n, int(h->single_cta_threads), false) == 0))
        return fail(EAT_EUNSUPPORTED, "EAT_KERNEL_CTA: arrival array does not fit shared memory");
    if (k == EAT_KERNEL_ASYNC && !async_ok)
        return fail(EAT_EUNSUPPORTED, "EAT_KERNEL_ASYNC: a 1/SM-count slice of the arrival array does not fit shared memory");
    if (k > EAT_KERNEL_GRID_ASYNC) return fail(EAT_EINVAL, "unknown kernel");
    if (k == EAT_KERNEL_GRID_ASYNC && !pick_gasync(h))
        return fail(EAT_EUNSUPPORTED, "EAT_KERNEL_GRID_ASYNC: the per-CTA vertex slices do not fit shared memory");
    if (k == EAT_KERNEL_CLUSTER && !pick_cluster(h, h->cluster_ctas, 0))
        return fail(EAT_EUNSUPPORTED, "EAT_KERNEL_CLUSTER: e[] does not fit the shared memory of a schedulable cluster");
    if (k == EAT_KERNEL_CONNECTION) {  // raw connections on the device (ablation schedule)
        CUDA_TRY(cudaMalloc(&h->d_conns, std::max<size_t>(h->raw.size(), 1) * sizeof(uint4)));
        CUDA_TRY(cudaMemcpy(h->d_conns, h->raw.data(), h->raw.size() * sizeof(uint4), cudaMemcpyHostToDevice));
        h->ix.conns = h->d_conns;
        h->ix.num_conns = h->raw.size();
        h->slices[0].ix.conns = h->d_conns;
        h->slices[0].ix.num_conns = h->raw.size();
        std::vector<uint4>().swap(h->raw);
    }
    if (k == EAT_KERNEL_ASYNC) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (eat::async_alloc(h->aw, h->hx.n, uint32_t(sms)) != cudaSuccess)
            return fail(EAT_ENOMEM, "cannot allocate async-kernel scratch");
    }
    h->kernel = k;
    h->st.kernel = k;
    return EAT_OK;
}

eat_status check_query(const eat_handle *h, uint32_t s, uint32_t t_s) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    if (h->host_only) return fail(EAT_ESTATE, "handle was built with EAT_BUILD_HOST_ONLY");
    if (s >= h->hx.n) return fail(EAT_EINVAL, "invalid source vertex id");
    if (t_s >= EAT_INF) return fail(EAT_ERANGE, "t_s >= EAT_INF");
    return EAT_OK;
}

// Enqueue one single query on stream st writing caller-ordered e[] to d_out.
eat_status enqueue_single(eat_handle *h, uint32_t s, uint32_t t_s, uint32_t *d_out, cudaStream_t st) {
    if (h->mode == EAT_MODE_EDGE_PARTITIONED)
        return fail(EAT_ESTATE, "edge-partitioned handles run through eat_query / eat_query_device (internal)");
    if (h->kernel == EAT_KERNEL_CTA) {
        uint32_t q[2] = {s, t_s};
        CUDA_TRY(cudaMemcpyAsync(h->d_q1, q, sizeof(q), cudaMemcpyHostToDevice, st));
        // a lone query gets the widest CTA (1024 threads, uint32 e[]): it has the SM to itself
        eat::CtaArgs a;
        a.src = h->d_q1;
        a.ts = h->d_q1 + 1;
        a.nq = 1;
        a.out = d_out;
        a.sweeps = h->d_sweeps1;
        a.qcounter = h->d_counter;
        a.invalid = h->d_invalid;
        a.threads = int(h->single_cta_threads);
        a.arr16 = false;
        a.grid_cap = 1;
        CUDA_TRY(eat::launch_query_cta(h->ix, a, st));
    } else if (h->kernel == EAT_KERNEL_CLUSTER) {
        eat::ClusterArgs a;  // (s, t_s) by value: no copy ahead of the launch
        a.s1 = s;
        a.ts1 = t_s;
        a.nq = 1;
        a.out = d_out;
        a.sweeps = h->d_sweeps1;
        a.qcounter = h->d_counter;
        a.invalid = h->d_invalid;
        a.cs = int(h->cluster_ctas);
        a.stage = h->cluster_stage;
        a.tl_cap = h->cluster_tl;
        a.async = h->cluster_async;
        a.max_clusters = 1;
        eat::DevIndex cix = h->ix;
        cix.window = h->cluster_window;
        CUDA_TRY(eat::launch_query_cluster(cix, a, st));
    } else if (h->kernel == EAT_KERNEL_GRID_ASYNC) {
        eat::GAsyncWork w{h->gw.arr, h->gw.bm, h->d_gacnt, h->gw.ctl};
        CUDA_TRY(eat::launch_query_gasync(h->ix, w, s, t_s, d_out, st));
        CUDA_TRY(cudaMemcpyAsync(h->d_sweeps1, h->gw.ctl + 8, 4, cudaMemcpyDeviceToDevice, st));
    } else if (h->kernel == EAT_KERNEL_ASYNC) {
        CUDA_TRY(eat::launch_query_async(h->ix, h->aw, s, t_s, d_out, st));
        CUDA_TRY(cudaMemcpyAsync(h->d_sweeps1, h->aw.ctl + 9, 4, cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(h->d_rounds1, h->aw.ctl + 8, 4, cudaMemcpyDeviceToDevice, st));
    } else {
        int sched = h->kernel == EAT_KERNEL_FULL_SWEEP ? eat::kSchedFull
                    : h->kernel == EAT_KERNEL_CONNECTION ? eat::kSchedConn
                    : h->kernel == EAT_KERNEL_BITMAP     ? eat::kSchedBitmap
                                                         : eat::kSchedFrontier;
        CUDA_TRY(eat::launch_query_grid(h->ix, int(h->subwarp), sched, h->gw, s, t_s, d_out, st));
        CUDA_TRY(cudaMemcpyAsync(h->d_sweeps1, h->gw.ctl + 8, 4, cudaMemcpyDeviceToDevice, st));
    }
    return EAT_OK;
}

// Orders device work of successive calls on one handle across streams:
// the call's stream waits for the previous call's work, then records its own.
struct HandleOrder {
    eat_handle *h;
    cudaStream_t st;
    HandleOrder(eat_handle *h_, cudaStream_t st_) : h(h_), st(st_) {
        if (!h->order_ev) cudaEventCreateWithFlags(&h->order_ev, cudaEventDisableTiming);
        cudaStreamWaitEvent(st, h->order_ev, 0);
    }
    ~HandleOrder() { cudaEventRecord(h->order_ev, st); }
};


// Option fields of a handle (validated); shared by the primary handle and
// its replicas on other devices.
eat_status apply_opts(eat_handle *h, const eat_build_opts &o) {
    const uint32_t sw = o.subwarp == 0 ? 32u : (o.subwarp == 64 ? 0u : o.subwarp);  // 0 internally = flattened
    if (sw != 0 && sw != 1 && sw != 2 && sw != 4 && sw != 8 && sw != 16 && sw != 32)
        return fail(EAT_EINVAL, "subwarp must be 0 (default 32), 1, 2, 4, 8, 16, 32 or 64 (flattened pairs)");
    if (o.mode > EAT_MODE_EDGE_PARTITIONED) return fail(EAT_EINVAL, "unknown mode");
    if (o.kernel > EAT_KERNEL_GRID_ASYNC) return fail(EAT_EINVAL, "unknown kernel");
    if (o.lookup > 2) return fail(EAT_EINVAL, "lookup must be 0 (Cluster-AP), 1 (Connection-type-AP) or 2 (linear)");
    const uint32_t pc = o.part_count ? o.part_count : 1;
    if (o.mode == EAT_MODE_EDGE_PARTITIONED && o.part_rank >= pc)
        return fail(EAT_EINVAL, "edge partition needs part_rank < part_count");
    h->subwarp = sw;
    h->mode = o.mode;
    h->window = o.window_seconds == 0 ? EAT_DEFAULT_WINDOW : o.window_seconds;
    h->group_window = o.window_seconds == 0 ? kDefaultGroupWindow : o.window_seconds;
    h->cluster_window = o.window_seconds == 0 ? EAT_INF : o.window_seconds;
    h->cta_threads = o.cta_threads == 0 ? 320u : o.cta_threads;
    if (h->cta_threads != 512 && h->cta_threads != 384 && h->cta_threads != 320 && h->cta_threads != 256 &&
        h->cta_threads != 192 && h->cta_threads != 128)
        return fail(EAT_EINVAL, "cta_threads must be 128, 192, 256, 320, 384 or 512");
    if (o.arr_bits != 0 && o.arr_bits != 16 && o.arr_bits != 32) return fail(EAT_EINVAL, "arr_bits must be 0, 16 or 32");
    h->arr16 = o.arr_bits == 16;
    if (o.continuation != EAT_CONT_NONE && o.continuation > 64)
        return fail(EAT_EINVAL, "continuation must be 0 (default 1), 1..64 or EAT_CONT_NONE");
    h->cont_budget = o.continuation == 0 ? 1u : (o.continuation == EAT_CONT_NONE ? 0u : o.continuation);
    if (const char *dv = getenv("EAT_E2E_DIRECT")) h->e2e_direct = atoi(dv) != 0;  // A/B
    if (const char *mv = getenv("EAT_E2E_MODE")) h->e2e_mode = atoi(mv);            // A/B: 0 pipeline, 1 direct, 2 streamed
    if (const char *sv = getenv("EAT_SORT_BATCHES")) h->sort_batches = atoi(sv) != 0;  // A/B
    h->part_rank = o.part_rank;
    h->part_count = pc;
    if (o.exchange > EAT_EXCHANGE_PEER) return fail(EAT_EINVAL, "exchange must be EAT_EXCHANGE_ALLREDUCE or EAT_EXCHANGE_PEER");
    h->exchange = o.exchange;
    if (o.local_sweeps && (o.mode != EAT_MODE_EDGE_PARTITIONED || o.exchange != EAT_EXCHANGE_ALLREDUCE))
        return fail(EAT_EINVAL, "local_sweeps applies to EDGE_PARTITIONED handles with EAT_EXCHANGE_ALLREDUCE");
    h->local_sweeps = o.local_sweeps;
    if (o.cluster_ctas && (o.cluster_ctas < 2 || o.cluster_ctas > 16 || (o.cluster_ctas & (o.cluster_ctas - 1))))
        return fail(EAT_EINVAL, "cluster_ctas must be 2, 4, 8 or 16");
    h->cluster_ctas = o.cluster_ctas;
    // all partitions in this process (one device) unless this is one rank of
    // several processes (NCCL id given, or EAT_BUILD_MULTIPROCESS for PEER)
    h->loopback = o.mode == EAT_MODE_EDGE_PARTITIONED && pc > 1 &&
                  (o.exchange == EAT_EXCHANGE_PEER ? !(o.flags & EAT_BUILD_MULTIPROCESS) : !o.nccl_unique_id);
    h->host_only = (o.flags & EAT_BUILD_HOST_ONLY) != 0;
    h->cluster_async = !(o.flags & EAT_BUILD_CLUSTER_SYNC) && !(getenv("EAT_CLUSTER_ASYNC") && atoi(getenv("EAT_CLUSTER_ASYNC")) == 0);
    h->lookup_mode = o.lookup;
    return EAT_OK;
}

// Device part of eat_build on `device` (-1: current): stream, upload,
// kernel choice, counters, NCCL communicator.  On error the caller releases.
eat_status device_setup(eat_handle *h, const eat_build_opts &o, int device) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(EAT_ECUDA, "no CUDA device available (libeat has no CPU fallback)");
    if (device >= 0) {
        if (device >= ndev) return fail(EAT_EINVAL, "device ordinal out of range");
        h->device = device;
    } else {
        cudaGetDevice(&h->device);
    }
    if (cudaSetDevice(h->device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess)
        return fail(EAT_ECUDA, "cannot initialise CUDA device");
    eat_status est = upload(h);
    if (est != EAT_OK) return est;
    if ((est = resolve_kernel(h, o.kernel)) != EAT_OK) return est;
    if (o.flags & EAT_BUILD_COUNTERS) {
        if (cudaMalloc(&h->d_work, eat::kWorkCounters * sizeof(unsigned long long)) != cudaSuccess ||
            cudaMemset(h->d_work, 0, eat::kWorkCounters * sizeof(unsigned long long)) != cudaSuccess)
            return fail(EAT_ENOMEM, "cannot allocate work counters");
    }
    if (h->mode == EAT_MODE_EDGE_PARTITIONED && !h->loopback && h->exchange == EAT_EXCHANGE_ALLREDUCE &&
        h->part_count > 1) {
        ncclUniqueId id;
        std::memcpy(&id, o.nccl_unique_id, sizeof(id));
        ncclResult_t r = ncclCommInitRank(&h->comm, int(h->part_count), id, int(o.part_rank));
        if (r != ncclSuccess) return fail(EAT_ENCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    return EAT_OK;
}

}  // namespace

extern "C" {

uint32_t eat_abi_version(void) { return EAT_ABI_VERSION; }

const char *eat_last_error(void) { return g_err.c_str(); }

eat_status eat_build(const eat_timetable *tt, const eat_build_opts *opts, eat_handle **out) {
    if (!tt || !out) return fail(EAT_EINVAL, "NULL timetable or output handle pointer");
    eat_build_opts o{};
    if (opts) o = *opts;
    eat::BuildParams p;
    p.cs = o.cluster_seconds ? o.cluster_seconds : 3600;
    p.renumber = o.renumber;
    if (o.cluster_dir > 2) return fail(EAT_EINVAL, "cluster_dir must be 0 (auto), 1 (dense) or 2 (compact)");
    p.dense = o.cluster_dir;
    std::vector<int> devs;
    if (o.num_devices > 1) {
        if (!o.devices) return fail(EAT_EINVAL, "num_devices > 1 needs a devices array");
        if (o.mode != EAT_MODE_REPLICATED)
            return fail(EAT_EUNSUPPORTED, "several devices per handle: REPLICATED mode only (edge partitions are one rank per device)");
        if (o.kernel == EAT_KERNEL_CONNECTION) return fail(EAT_EUNSUPPORTED, "EAT_KERNEL_CONNECTION is single-device");
        for (uint32_t i = 0; i < o.num_devices; ++i) {
            if (o.devices[i] < 0) return fail(EAT_EINVAL, "negative device ordinal");
            for (int d : devs)
                if (d == o.devices[i]) return fail(EAT_EINVAL, "device listed twice");
            devs.push_back(o.devices[i]);
        }
        o.device = devs[0];
    }
    eat_handle *h = new (std::nothrow) eat_handle();
    if (!h) return fail(EAT_ENOMEM, "out of host memory");
    eat_status est = apply_opts(h, o);
    if (est != EAT_OK) {
        delete h;
        return est;
    }
    std::string msg;
    int rc = EAT_OK;
    eat::SubtripStats sts;
    try {
        if (o.subtrips) {
            // NEXT-1 data enhancement: index the timetable
            // plus sub-trip shortcuts; arrival times are unchanged
            std::vector<uint32_t> U, V, D, L;
            rc = eat::make_subtrips(tt->num_connections, tt->u, tt->v, tt->dep, tt->dur, tt->trip, o.subtrips, U, V,
                                    D, L, sts, msg);
            if (rc == EAT_OK)
                rc = eat::build_host_index(tt->num_vertices, U.size(), U.data(), V.data(), D.data(), L.data(), tt->xy,
                                           p, h->hx, msg);
        } else {
            rc = eat::build_host_index(tt->num_vertices, tt->num_connections, tt->u, tt->v, tt->dep, tt->dur, tt->xy,
                                       p, h->hx, msg);
        }
    } catch (const std::bad_alloc &) {
        rc = EAT_ENOMEM;
        msg = "out of host memory during build";
    }
    if (rc != EAT_OK) {
        delete h;
        return fail(eat_status(rc), msg);
    }
    eat_stats &s = h->st;
    s.num_vertices = h->hx.n;
    s.num_clusters = h->hx.num_clusters;
    s.num_connections = tt->num_connections;
    s.num_shortcuts = sts.shortcuts;
    s.num_devices = devs.empty() ? 1u : uint32_t(devs.size());
    if (o.kernel == EAT_KERNEL_CONNECTION && !h->host_only) {
        // Connection-version ablation (Alg. 4): keep the raw connections (internal ids)
        const uint64_t m = tt->num_connections;
        h->raw.resize(m);
        for (uint64_t i = 0; i < m; ++i)
            h->raw[i] = make_uint4(h->hx.perm[tt->u[i]], h->hx.perm[tt->v[i]], tt->dep[i], tt->dep[i] + tt->dur[i]);
    }
    s.num_types = h->hx.num_types;
    s.num_edges = h->hx.num_edges;
    s.num_cluster_records = h->hx.num_crec;
    s.num_items = h->hx.num_items;
    s.num_spill_items = h->hx.pool.size();
    s.build_ms = h->hx.build_ms;
    if (h->host_only) {
        *out = h;
        return EAT_OK;
    }
    est = device_setup(h, o, o.device);
    // replicas on devices[1..] (REPLICATED, query sharding in eat_query_many):
    // same options, a copy of the host index, their own device scratch
    for (size_t i = 1; est == EAT_OK && i < devs.size(); ++i) {
        eat_handle *r = new (std::nothrow) eat_handle();
        if (!r) {
            est = fail(EAT_ENOMEM, "out of host memory");
            break;
        }
        h->replicas.push_back(r);
        if ((est = apply_opts(r, o)) != EAT_OK) break;
        try {
            r->hx = h->hx;
        } catch (const std::bad_alloc &) {
            est = fail(EAT_ENOMEM, "out of host memory (replica index copy)");
            break;
        }
        r->st = h->st;
        est = device_setup(r, o, devs[i]);
        // the replica serves device queries only: drop its host copy of the index
        std::vector<uint32_t>().swap(r->hx.type_rec);
        std::vector<uint32_t>().swap(r->hx.crec);
        std::vector<uint32_t>().swap(r->hx.pool);
    }
    if (est != EAT_OK) {
        std::string keep = g_err;
        for (eat_handle *r : h->replicas) {
            release_device(r);
            delete r;
        }
        release_device(h);
        delete h;
        g_err = keep;
        return est;
    }
    *out = h;
    return EAT_OK;
}

void eat_free(eat_handle *h) {
    if (!h) return;
    for (eat_handle *r : h->replicas) {
        release_device(r);
        delete r;
    }
    release_device(h);
    delete h;
}

eat_status eat_get_stats(const eat_handle *hc, eat_stats *out) {
    if (!hc || !out) return fail(EAT_EINVAL, "NULL argument");
    eat_handle *h = const_cast<eat_handle *>(hc);
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->host_only) {
        cudaSetDevice(h->device);
        uint32_t sw = 0;
        unsigned long long inv = 0;
        CUDA_TRY(cudaMemcpy(&sw, h->d_sweeps1, 4, cudaMemcpyDeviceToHost));
        CUDA_TRY(cudaMemcpy(&inv, h->d_invalid, 8, cudaMemcpyDeviceToHost));
        h->st.last_sweeps = sw;
        h->st.invalid_queries = inv;
        h->st.cta_grid = uint32_t(h->cta_grid);
        h->st.cta_threads = h->cta_threads;
        h->st.cluster_ctas = h->kernel == EAT_KERNEL_CLUSTER ? h->cluster_ctas : 0u;
        if (h->kernel == EAT_KERNEL_ASYNC && h->mode != EAT_MODE_EDGE_PARTITIONED) {
            uint32_t rr = 0;
            CUDA_TRY(cudaMemcpy(&rr, h->d_rounds1, 4, cudaMemcpyDeviceToHost));
            h->st.last_rounds = rr;
        }
        if (h->d_work) {
            unsigned long long w[eat::kWorkCounters];
            CUDA_TRY(cudaMemcpy(w, h->d_work, sizeof(w), cudaMemcpyDeviceToHost));
            h->st.select_cycles = w[6];
            h->st.pair_cycles = w[7];
            h->st.select_loop_cycles = w[8];
            h->st.pair_loop_cycles = w[9];
            h->st.vertex_visits = w[0];
            h->st.type_evals = w[1];
            h->st.cluster_reads = w[2];
            h->st.spill_items_read = w[3];
            h->st.improvements = w[4];
            h->st.sweeps_total = w[5];
            h->st.edge_evals = w[10];
            h->st.cluster_runs = w[11];
            h->st.cluster_singles = w[12];
            h->st.fallbacks = w[13];
            h->st.select_bits = w[14];
        }
    }
    *out = h->st;
    return EAT_OK;
}

eat_status eat_query_device(eat_handle *h, uint32_t s, uint32_t t_s, uint32_t *d_out, void *cuda_stream) {
    eat_status e = check_query(h, s, t_s);
    if (e != EAT_OK) return e;
    if (!d_out) return fail(EAT_EINVAL, "NULL output");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    HandleOrder order(h, st);
    if (h->mode == EAT_MODE_EDGE_PARTITIONED) return run_partitioned(h, s, t_s, d_out, st);
    return enqueue_single(h, s, t_s, d_out, st);
}

eat_status eat_query(eat_handle *h, uint32_t s, uint32_t t_s, uint32_t *out_arr) {
    eat_status e = check_query(h, s, t_s);
    if (e != EAT_OK) return e;
    if (!out_arr) return fail(EAT_EINVAL, "NULL output");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    if (h->order_ev) CUDA_TRY(cudaEventSynchronize(h->order_ev));  // device calls still in flight
    if (h->mode == EAT_MODE_EDGE_PARTITIONED) {
        e = run_partitioned(h, s, t_s, h->d_out1, h->stream);
        if (e != EAT_OK) return e;
    } else {
        e = enqueue_single(h, s, t_s, h->d_out1, h->stream);
        if (e != EAT_OK) return e;
    }
    // page-locked output: one D2H straight into it; else through the pinned stage
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, out_arr) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    CUDA_TRY(cudaMemcpyAsync(pinned ? out_arr : h->h_out1, h->d_out1, h->hx.n * 4ull, cudaMemcpyDeviceToHost,
                             h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (!pinned) std::memcpy(out_arr, h->h_out1, h->hx.n * 4ull);
    return EAT_OK;
}

}  // extern "C"

namespace {

eat_status query_targets_impl(eat_handle *h, const uint32_t *sources, const uint32_t *times, const uint32_t *dsts,
                              uint64_t nq, uint32_t *out);

// Run fn(handle, q0, count) for the query shards of a (possibly multi-device)
// handle: contiguous chunks proportional to nothing but the device count
// (replicas are identical), one host thread per device.  First error wins.
template <class F>
eat_status shard_queries(eat_handle *h, uint64_t nq, F fn) {
    if (h->replicas.empty()) return fn(h, 0, nq);
    std::vector<eat_handle *> hs{h};
    hs.insert(hs.end(), h->replicas.begin(), h->replicas.end());
    const uint64_t D = hs.size();
    std::vector<eat_status> rc(D, EAT_OK);
    std::vector<std::string> err(D);
    std::vector<std::thread> th;
    for (uint64_t d = 0; d < D; ++d) {
        const uint64_t q0 = nq * d / D, q1 = nq * (d + 1) / D;
        th.emplace_back([&, d, q0, q1] {
            if (q1 > q0) rc[d] = fn(hs[d], q0, q1 - q0);
            if (rc[d] != EAT_OK) err[d] = g_err;  // g_err is thread-local
        });
    }
    for (auto &t : th) t.join();
    for (uint64_t d = 0; d < D; ++d)
        if (rc[d] != EAT_OK) return fail(rc[d], "device " + std::to_string(hs[d]->device) + ": " + err[d]);
    return EAT_OK;
}

// Enqueue a batch of device-resident queries on st (CTA kernel), or, when e[]
// does not fit shared memory, one single-query launch after another.
// Launch the batched CTA kernel (uint16 pass + uint32 recompute of overflows);
// `slot` selects the overflow list (0: device API, 1/2: pipeline stages).
eat_status launch_batch_cta(eat_handle *h, const uint32_t *d_sources, const uint32_t *d_times, uint64_t nq,
                            uint32_t *d_out, cudaStream_t st, unsigned long long *d_qcounter, int slot,
                            const uint32_t *d_dst) {
    if (h->arr16 && h->ovf_cap[slot] < nq + 1) {
        if (h->d_ovf[slot]) {
            CUDA_TRY(cudaStreamSynchronize(st));
            cudaFree(h->d_ovf[slot]);
        }
        h->d_ovf[slot] = nullptr;
        h->ovf_cap[slot] = 0;
        CUDA_TRY(cudaMalloc(&h->d_ovf[slot], (nq + 1) * 4));
        h->ovf_cap[slot] = nq + 1;
    }
    eat::CtaArgs a;
    a.src = d_sources;
    a.ts = d_times;
    a.nq = nq;
    a.out = d_out;
    a.qcounter = d_qcounter;
    a.invalid = h->d_invalid;
    a.counters = h->d_work;
    a.dst = d_dst;
    a.threads = int(h->cta_threads);
    a.arr16 = h->arr16;
    if (h->arr16) {
        a.ovf_list = h->d_ovf[slot] + 1;
        a.ovf_cnt = h->d_ovf[slot];
    }
    // more queries than resident CTAs: hand them out by departure time (the
    // expensive ones first, a short last wave; N = 8 share of the city batch
    // 1.49 -> 1.35 ms, profiles/r02_order_by_time.jsonl)
    // Not for the direct e2e launch (slot 1), whose rows cross PCIe as the
    // queries finish: cheap queries last would finish in a burst at the end and
    // their rows would queue on the link (e2e 1.106M -> 0.99M q/s, also with
    // coarse time buckets: profiles/r02_order_by_time_e2e.jsonl); in caller
    // order the row traffic is spread over the whole launch.
    if (h->sort_batches && nq > uint64_t(h->cta_grid) && slot != 1) {
        CUDA_TRY(eat::sort_queries_by_time(d_times, nq, 0, h->qsort[slot], st));
        a.qorder = h->qsort[slot].v1;
    }
    CUDA_TRY(eat::launch_query_cta(h->ix, a, st));
    return EAT_OK;
}

// Batched queries whose e[] does not fit shared memory: CTA groups of one
// cooperative launch take queries in turn (k_query_groups); dst != NULL:
// goal-directed, out[q] = e[dst[q]].
eat_status launch_batch_groups(eat_handle *h, const uint32_t *d_sources, const uint32_t *d_times, uint64_t nq,
                               uint32_t *d_out, cudaStream_t st, unsigned long long *d_qcounter, const uint32_t *d_dst,
                               int slot) {
    uint32_t groups = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(kBatchGroupsMax, nq / 8)));
    // scratch is ~32 B per vertex per group: keep it under 4 GB
    groups = uint32_t(std::min<uint64_t>(groups, std::max<uint64_t>(1, (4ull << 30) / (32ull * h->hx.n + 1))));
    if (const char *gv = getenv("EAT_BATCH_GROUPS")) groups = uint32_t(std::max(1, std::min(592, atoi(gv))));
    groups = uint32_t(std::min<uint64_t>(groups, nq));
    if (h->bgw.size() < groups) {
        CUDA_TRY(cudaStreamSynchronize(st));
        while (h->bgw.size() < groups) {
            h->bgw.emplace_back();
            CUDA_TRY(gridwork_alloc(h->bgw.back(), h->hx.n, false));
        }
        if (h->d_bgw) cudaFree(h->d_bgw);
        h->d_bgw = nullptr;
        CUDA_TRY(cudaMalloc(&h->d_bgw, h->bgw.size() * sizeof(eat::GridWork)));
        CUDA_TRY(cudaMemcpy(h->d_bgw, h->bgw.data(), h->bgw.size() * sizeof(eat::GridWork), cudaMemcpyHostToDevice));
    }
    // more queries than groups: hand them out in source-locality order
    const uint32_t *qorder = nullptr;
    if (h->sort_batches && nq > groups) {
        eat::SortScratch &sc = h->qsort[slot];
        if (sc.cap < nq) CUDA_TRY(cudaStreamSynchronize(st));
        CUDA_TRY(eat::sort_queries_by_source(h->ix, d_sources, nq, sc, st));
        qorder = sc.v1;
    }
    eat::DevIndex gix = h->ix;
    gix.window = h->group_window;
    CUDA_TRY(eat::launch_query_groups(gix, h->subwarp == 0 ? 32 : int(h->subwarp), h->bgw.data(), h->d_bgw, groups,
                                      d_sources, d_times, nq, d_out, d_qcounter, h->d_invalid, d_dst, qorder, st));
    return EAT_OK;
}

eat_status enqueue_batch(eat_handle *h, const uint32_t *d_sources, const uint32_t *d_times, uint64_t nq,
                         uint32_t *d_out, cudaStream_t st, unsigned long long *d_qcounter, int slot = 0) {
    // (batches on the cluster kernel, one query per 2/4/8-CTA cluster: metro
    // 1,024 queries 38.7k / 23.8k / 12.8k q/s vs 46.1k on k_query_groups --
    // profiles/r02_ab_metro_batch_cluster.jsonl; not used)
    if (h->cta_grid > 0 && !h->batch_groups) return launch_batch_cta(h, d_sources, d_times, nq, d_out, st, d_qcounter, slot, nullptr);
    return launch_batch_groups(h, d_sources, d_times, nq, d_out, st, d_qcounter, nullptr, slot);
}

// Parallel host copy (staging -> caller memory).
void host_copy(void *dst, const void *src, size_t bytes) {
    const size_t nt = std::min<size_t>(8, std::max<size_t>(1, bytes >> 22));
    if (nt <= 1) {
        std::memcpy(dst, src, bytes);
        return;
    }
    std::vector<std::thread> th;
    for (size_t t = 0; t < nt; ++t) {
        const size_t a = bytes * t / nt, b = bytes * (t + 1) / nt;
        th.emplace_back([=] { std::memcpy(static_cast<char *>(dst) + a, static_cast<const char *>(src) + a, b - a); });
    }
    for (auto &x : th) x.join();
}

}  // namespace

extern "C" {

eat_status eat_query_many_device(eat_handle *h, const uint32_t *d_sources, const uint32_t *d_times, uint64_t nq,
                                 uint32_t *d_out, void *cuda_stream) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    if (h->host_only) return fail(EAT_ESTATE, "handle was built with EAT_BUILD_HOST_ONLY");
    if (nq == 0) return EAT_OK;
    if (!d_sources || !d_times || !d_out) return fail(EAT_EINVAL, "NULL argument");
    if (h->mode == EAT_MODE_EDGE_PARTITIONED)
        return fail(EAT_ESTATE, "batched queries need a replicated handle (query-parallel sharding)");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    HandleOrder order(h, st);
    return enqueue_batch(h, d_sources, d_times, nq, d_out, st, h->d_counter);
}

eat_status eat_query_many_target_device(eat_handle *h, const uint32_t *d_sources, const uint32_t *d_times,
                                        const uint32_t *d_dsts, uint64_t nq, uint32_t *d_out, void *cuda_stream) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    if (h->host_only) return fail(EAT_ESTATE, "handle was built with EAT_BUILD_HOST_ONLY");
    if (nq == 0) return EAT_OK;
    if (!d_sources || !d_times || !d_dsts || !d_out) return fail(EAT_EINVAL, "NULL argument");
    if (h->mode == EAT_MODE_EDGE_PARTITIONED)
        return fail(EAT_ESTATE, "batched queries need a replicated handle (query-parallel sharding)");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    HandleOrder order(h, st);
    if (h->cta_grid > 0 && !h->batch_groups) return launch_batch_cta(h, d_sources, d_times, nq, d_out, st, h->d_counter, 0, d_dsts);
    // e[] too large for shared memory: CTA groups, e[dst] of each query
    return launch_batch_groups(h, d_sources, d_times, nq, d_out, st, h->d_counter, d_dsts, 0);
}

eat_status eat_query_many_target(eat_handle *h, const uint32_t *sources, const uint32_t *times, const uint32_t *dsts,
                                 uint64_t nq, uint32_t *out) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    if (h->host_only) return fail(EAT_ESTATE, "handle was built with EAT_BUILD_HOST_ONLY");
    if (nq == 0) return EAT_OK;
    if (!sources || !times || !dsts || !out) return fail(EAT_EINVAL, "NULL argument");
    for (uint64_t q = 0; q < nq; ++q) {
        if (sources[q] >= h->hx.n || dsts[q] >= h->hx.n)
            return fail(EAT_EINVAL, "invalid source or destination vertex id at index " + std::to_string(q));
        if (times[q] >= EAT_INF) return fail(EAT_ERANGE, "t_s >= EAT_INF at index " + std::to_string(q));
    }
    return shard_queries(h, nq, [&](eat_handle *hh, uint64_t q0, uint64_t c) {
        return query_targets_impl(hh, sources + q0, times + q0, dsts + q0, c, out + q0);
    });
}

}  // extern "C"

namespace {

eat_status query_targets_impl(eat_handle *h, const uint32_t *sources, const uint32_t *times, const uint32_t *dsts,
                              uint64_t nq, uint32_t *out) {
    uint32_t *d = nullptr;
    {
        std::lock_guard<std::mutex> lk(h->mu);
        CUDA_TRY(cudaSetDevice(h->device));
    if (h->order_ev) CUDA_TRY(cudaEventSynchronize(h->order_ev));  // device calls still in flight
        CUDA_TRY(cudaMallocAsync(&d, nq * 16, h->stream));
        CUDA_TRY(cudaMemcpyAsync(d, sources, nq * 4, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(cudaMemcpyAsync(d + nq, times, nq * 4, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(cudaMemcpyAsync(d + 2 * nq, dsts, nq * 4, cudaMemcpyHostToDevice, h->stream));
    }
    eat_status e = eat_query_many_target_device(h, d, d + nq, d + 2 * nq, nq, d + 3 * nq, h->stream);
    std::lock_guard<std::mutex> lk(h->mu);
    if (e == EAT_OK) {
        CUDA_TRY(cudaMemcpyAsync(out, d + 3 * nq, nq * 4, cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(cudaStreamSynchronize(h->stream));
    }
    cudaFreeAsync(d, h->stream);
    return e;
}

// Streamed batch into page-locked host rows (caller holds h->mu): one
// persistent CTA-kernel launch writes rows to device memory and counts each
// finished row in its chunk's flag (mapped host memory); this thread copies
// every completed chunk with the copy engine (cudaMemcpyAsync on a second
// stream) while the kernel keeps relaxing later queries.  Queries are taken
// in order, so chunks complete roughly in order; the tail is one chunk.
eat_status query_many_streamed(eat_handle *h, const uint32_t *sources, const uint32_t *times, uint64_t nq,
                               uint32_t *out) {
    const uint64_t n = h->hx.n;
    constexpr uint32_t kShift = 8;  // 256 queries (10 MB of city rows) per chunk
    const uint64_t nch = (nq + (1u << kShift) - 1) >> kShift;
    if (!h->bstream[0])
        for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamCreateWithFlags(&h->bstream[i], cudaStreamNonBlocking));
    if (!h->d_bcounter) CUDA_TRY(cudaMalloc(&h->d_bcounter, 2 * sizeof(unsigned long long)));
    if (h->dcap < nq) {
        if (h->d_dsrc) cudaFree(h->d_dsrc);
        if (h->d_dts) cudaFree(h->d_dts);
        h->d_dsrc = h->d_dts = nullptr;
        h->dcap = 0;
        CUDA_TRY(cudaMalloc(&h->d_dsrc, nq * 4));
        CUDA_TRY(cudaMalloc(&h->d_dts, nq * 4));
        h->dcap = nq;
    }
    if (h->scap < nq) {
        if (h->d_srows) cudaFree(h->d_srows);
        h->d_srows = nullptr;
        h->scap = 0;
        CUDA_TRY(cudaMalloc(&h->d_srows, nq * n * 4));
        h->scap = nq;
    }
    if (h->done_cap < nq) {
        if (h->h_done) cudaFreeHost(h->h_done);
        h->h_done = nullptr;
        h->done_cap = 0;
        CUDA_TRY(cudaHostAlloc(&h->h_done, nq * sizeof(unsigned int), cudaHostAllocMapped));
        CUDA_TRY(cudaHostGetDevicePointer(&h->d_done, h->h_done, 0));
        h->done_cap = nq;
    }
    std::memset(h->h_done, 0, nq * sizeof(unsigned int));
    cudaStream_t ks = h->bstream[0], cs = h->bstream[1];
    CUDA_TRY(cudaMemcpyAsync(h->d_dsrc, sources, nq * 4, cudaMemcpyHostToDevice, ks));
    CUDA_TRY(cudaMemcpyAsync(h->d_dts, times, nq * 4, cudaMemcpyHostToDevice, ks));
    eat::CtaArgs a;
    a.src = h->d_dsrc;
    a.ts = h->d_dts;
    a.nq = nq;
    a.out = h->d_srows;
    a.qcounter = h->d_bcounter;
    a.invalid = h->d_invalid;
    a.threads = int(h->cta_threads);
    a.done = h->d_done;
    CUDA_TRY(eat::launch_query_cta(h->ix, a, ks));
    const volatile unsigned int *flags = h->h_done;
    uint64_t seen = 0;  // rows [0, seen) are known finished
    for (uint64_t c = 0; c < nch; ++c) {
        const uint64_t q0 = c << kShift, q1 = std::min<uint64_t>(q0 + (uint64_t(1) << kShift), nq);
        for (uint64_t spin = 0; seen < q1; ++spin) {
            if (flags[seen]) {
                ++seen;
                continue;
            }
            if ((spin & 1023u) == 1023u) {  // a failed kernel never finishes the chunk
                const cudaError_t ke = cudaStreamQuery(ks);
                if (ke != cudaSuccess && ke != cudaErrorNotReady) return fail(EAT_ECUDA, cudaGetErrorString(ke));
                if (ke == cudaSuccess && !flags[seen]) return fail(EAT_ECUDA, "streamed batch: row not flagged");
                std::this_thread::yield();
            }
        }
        CUDA_TRY(cudaMemcpyAsync(out + q0 * n, h->d_srows + q0 * n, (q1 - q0) * n * 4, cudaMemcpyDeviceToHost, cs));
    }
    CUDA_TRY(cudaStreamSynchronize(ks));
    CUDA_TRY(cudaStreamSynchronize(cs));
    return EAT_OK;
}

eat_status query_many_impl(eat_handle *h, const uint32_t *sources, const uint32_t *times, uint64_t nq,
                           uint32_t *out) {
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    if (h->order_ev) CUDA_TRY(cudaEventSynchronize(h->order_ev));  // device calls still in flight
    const uint64_t n = h->hx.n;
    // Two-stage pipeline over chunks of queries (stream i&1): H2D queries ->
    // batched kernel -> D2H rows, so chunk i+1 computes while chunk i copies.
    // Output rows go straight to `out` when it is pinned (page-locked) host
    // memory, else through pinned staging buffers and a parallel host copy.
    cudaPointerAttributes pa{};
    const bool pinned = cudaPointerGetAttributes(&pa, out) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (pinned && h->e2e_mode == 2 && h->cta_grid > 0 && !h->batch_groups && !h->arr16 && !h->d_work)
        return query_many_streamed(h, sources, times, nq, out);
    if (pinned && pa.devicePointer && h->e2e_direct && h->e2e_mode != 0) {
        // Direct: one persistent launch over all queries; each CTA (or CTA
        // group) stores its finished rows into the page-locked host buffer
        // over PCIe (mapped pointer), so the D2H traffic overlaps the
        // relaxation of the other queries with no chunk head/tail.
        if (!h->bstream[0])
            for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamCreateWithFlags(&h->bstream[i], cudaStreamNonBlocking));
        if (!h->d_bcounter) CUDA_TRY(cudaMalloc(&h->d_bcounter, 2 * sizeof(unsigned long long)));
        if (h->dcap < nq) {
            if (h->d_dsrc) cudaFree(h->d_dsrc);
            if (h->d_dts) cudaFree(h->d_dts);
            h->d_dsrc = h->d_dts = nullptr;
            h->dcap = 0;
            CUDA_TRY(cudaMalloc(&h->d_dsrc, nq * 4));
            CUDA_TRY(cudaMalloc(&h->d_dts, nq * 4));
            h->dcap = nq;
        }
        cudaStream_t st = h->bstream[0];
        CUDA_TRY(cudaMemcpyAsync(h->d_dsrc, sources, nq * 4, cudaMemcpyHostToDevice, st));
        CUDA_TRY(cudaMemcpyAsync(h->d_dts, times, nq * 4, cudaMemcpyHostToDevice, st));
        eat_status e = enqueue_batch(h, h->d_dsrc, h->d_dts, nq, static_cast<uint32_t *>(pa.devicePointer), st,
                                     h->d_bcounter, 1);
        if (e != EAT_OK) return e;
        CUDA_TRY(cudaStreamSynchronize(st));
        return EAT_OK;
    }
    const uint64_t chunk =
        std::max<uint64_t>(1, std::min<uint64_t>(nq, std::min<uint64_t>(1024, (256ull << 20) / (4 * n))));
    if (!h->bstream[0])
        for (int i = 0; i < 2; ++i) CUDA_TRY(cudaStreamCreateWithFlags(&h->bstream[i], cudaStreamNonBlocking));
    if (!h->d_bcounter) CUDA_TRY(cudaMalloc(&h->d_bcounter, 2 * sizeof(unsigned long long)));
    if (h->bcap < chunk) {
        for (int i = 0; i < 2; ++i) {
            void *ptrs[] = {h->d_bsrc[i], h->d_bts[i], h->d_bout[i]};
            for (void *p : ptrs)
                if (p) cudaFree(p);
            h->d_bsrc[i] = h->d_bts[i] = h->d_bout[i] = nullptr;
        }
        h->bcap = 0;
        for (int i = 0; i < 2; ++i) {
            CUDA_TRY(cudaMalloc(&h->d_bsrc[i], chunk * 4));
            CUDA_TRY(cudaMalloc(&h->d_bts[i], chunk * 4));
            CUDA_TRY(cudaMalloc(&h->d_bout[i], chunk * n * 4));
        }
        h->bcap = chunk;
    }
    if (!pinned && h->stage_cap < chunk) {
        for (int i = 0; i < 2; ++i) {
            if (h->h_stage[i]) cudaFreeHost(h->h_stage[i]);
            h->h_stage[i] = nullptr;
        }
        h->stage_cap = 0;
        for (int i = 0; i < 2; ++i) CUDA_TRY(cudaMallocHost(&h->h_stage[i], chunk * n * 4));
        h->stage_cap = chunk;
    }
    // Kernels (and their inputs) in order on stream 0, row copies on stream 1:
    // chunk i's copy overlaps chunk i+1's kernel; chunk i+2 reuses the buffers
    // after chunk i's copy.  One compute stream keeps cooperative grid-group
    // launches (graphs without shared-memory e[]) from running concurrently.
    if (!h->bev[0])
        for (int i = 0; i < 4; ++i) CUDA_TRY(cudaEventCreateWithFlags(&h->bev[i], cudaEventDisableTiming));
    cudaStream_t cs = h->bstream[0], ks = h->bstream[1];
    const uint64_t nchunks = (nq + chunk - 1) / chunk;
    for (uint64_t i = 0; i <= nchunks; ++i) {
        if (i < nchunks) {
            const int b = int(i & 1);
            const uint64_t q0 = i * chunk, c = std::min(chunk, nq - q0);
            if (i >= 2) CUDA_TRY(cudaStreamWaitEvent(cs, h->bev[2 + b], 0));  // chunk i-2's rows copied out
            CUDA_TRY(cudaMemcpyAsync(h->d_bsrc[b], sources + q0, c * 4, cudaMemcpyHostToDevice, cs));
            CUDA_TRY(cudaMemcpyAsync(h->d_bts[b], times + q0, c * 4, cudaMemcpyHostToDevice, cs));
            eat_status e = enqueue_batch(h, h->d_bsrc[b], h->d_bts[b], c, h->d_bout[b], cs, h->d_bcounter + b, 1 + b);
            if (e != EAT_OK) return e;
            CUDA_TRY(cudaEventRecord(h->bev[b], cs));
            CUDA_TRY(cudaStreamWaitEvent(ks, h->bev[b], 0));
            CUDA_TRY(cudaMemcpyAsync(pinned ? out + q0 * n : h->h_stage[b], h->d_bout[b], c * n * 4,
                                     cudaMemcpyDeviceToHost, ks));
            CUDA_TRY(cudaEventRecord(h->bev[2 + b], ks));
        }
        if (i >= 1) {  // retire chunk i-1 (its stage is reused by chunk i+1)
            const int b = int((i - 1) & 1);
            const uint64_t q0 = (i - 1) * chunk, c = std::min(chunk, nq - q0);
            CUDA_TRY(cudaEventSynchronize(h->bev[2 + b]));
            if (!pinned) host_copy(out + q0 * n, h->h_stage[b], c * n * 4);
        }
    }
    return EAT_OK;
}

}  // namespace

extern "C" {

eat_status eat_query_many(eat_handle *h, const uint32_t *sources, const uint32_t *times, uint64_t nq,
                          uint32_t *out) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    if (h->host_only) return fail(EAT_ESTATE, "handle was built with EAT_BUILD_HOST_ONLY");
    if (nq == 0) return EAT_OK;
    if (!sources || !times || !out) return fail(EAT_EINVAL, "NULL argument");
    if (h->mode == EAT_MODE_EDGE_PARTITIONED)
        return fail(EAT_ESTATE, "batched queries need a replicated handle (query-parallel sharding)");
    for (uint64_t q = 0; q < nq; ++q) {
        if (sources[q] >= h->hx.n) return fail(EAT_EINVAL, "invalid source vertex id at index " + std::to_string(q));
        if (times[q] >= EAT_INF) return fail(EAT_ERANGE, "t_s >= EAT_INF at index " + std::to_string(q));
    }
    const uint64_t n = h->hx.n;
    return shard_queries(h, nq, [&](eat_handle *hh, uint64_t q0, uint64_t c) {
        return query_many_impl(hh, sources + q0, times + q0, c, out + q0 * n);
    });
}

eat_status eat_lookup_device(eat_handle *h, const uint32_t *d_type, const uint32_t *d_bound, uint64_t n,
                             uint32_t *d_out, void *cuda_stream) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    if (h->host_only) return fail(EAT_ESTATE, "handle was built with EAT_BUILD_HOST_ONLY");
    if (n && (!d_type || !d_bound || !d_out)) return fail(EAT_EINVAL, "NULL argument");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    CUDA_TRY(eat::launch_lookup(h->ix, d_type, d_bound, n, d_out, static_cast<cudaStream_t>(cuda_stream)));
    return EAT_OK;
}

eat_status eat_index_export(const eat_handle *h, uint32_t *perm, uint32_t *type_ptr, uint32_t *type_rec,
                            uint32_t *crec, uint32_t *pool) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    const eat::HostIndex &x = h->hx;
    if (perm) std::copy(x.perm.begin(), x.perm.end(), perm);
    if (type_ptr) std::copy(x.type_ptr.begin(), x.type_ptr.end(), type_ptr);
    if (type_rec) std::copy(x.type_rec.begin(), x.type_rec.end(), type_rec);
    if (crec) std::copy(x.crec.begin(), x.crec.end(), crec);
    if (pool) std::copy(x.pool.begin(), x.pool.end(), pool);
    return EAT_OK;
}

eat_status eat_peer_export(eat_handle *h, void *handle_out) {
    if (!h || !handle_out) return fail(EAT_EINVAL, "NULL argument");
    if (h->mode != EAT_MODE_EDGE_PARTITIONED || h->exchange != EAT_EXCHANGE_PEER || h->loopback || h->peer_own.empty())
        return fail(EAT_ESTATE, "eat_peer_export needs a multi-process EAT_EXCHANGE_PEER handle");
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    cudaIpcMemHandle_t ipc;
    CUDA_TRY(cudaIpcGetMemHandle(&ipc, h->peer_own[0]));
    static_assert(sizeof(ipc) == EAT_PEER_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle_out, &ipc, sizeof(ipc));
    return EAT_OK;
}

eat_status eat_peer_connect(eat_handle *h, const void *handles, uint32_t count) {
    if (!h || !handles) return fail(EAT_EINVAL, "NULL argument");
    if (h->mode != EAT_MODE_EDGE_PARTITIONED || h->exchange != EAT_EXCHANGE_PEER || h->loopback)
        return fail(EAT_ESTATE, "eat_peer_connect needs a multi-process EAT_EXCHANGE_PEER handle");
    if (count != h->part_count) return fail(EAT_EINVAL, "eat_peer_connect: count must equal part_count");
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->peer_ready) return fail(EAT_ESTATE, "eat_peer_connect: already connected");
    CUDA_TRY(cudaSetDevice(h->device));
    const uint32_t n = h->hx.n;
    eat::PeerCtx &c = h->peer_ctx;
    for (uint32_t p = 0; p < count; ++p) {
        if (p == h->part_rank) continue;
        cudaIpcMemHandle_t ipc;
        std::memcpy(&ipc, static_cast<const char *>(handles) + size_t(p) * EAT_PEER_HANDLE_BYTES, sizeof(ipc));
        void *ptr = nullptr;
        CUDA_TRY(cudaIpcOpenMemHandle(&ptr, ipc, cudaIpcMemLazyEnablePeerAccess));
        h->peer_mapped.push_back(ptr);
        uint32_t lo = 0, hi = 0;
        eat::partition_range(h->hx, p, count, lo, hi);
        c.part[p] = eat::peer_part_view(ptr, n, lo, hi);
        if (p == 0) c.gctl = eat::peer_gctl(ptr, n, hi - lo);
    }
    eat_status e = peer_publish(h);
    if (e != EAT_OK) return e;
    h->peer_ready = true;
    return EAT_OK;
}

eat_status eat_selftest(const eat_handle *hc, uint64_t *failures) {
    if (!hc || !failures) return fail(EAT_EINVAL, "NULL argument");
    if (hc->host_only) return fail(EAT_ESTATE, "handle was built with EAT_BUILD_HOST_ONLY");
    eat_handle *h = const_cast<eat_handle *>(hc);
    std::lock_guard<std::mutex> lk(h->mu);
    CUDA_TRY(cudaSetDevice(h->device));
    unsigned long long *d = nullptr;
    CUDA_TRY(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
    cudaError_t e = eat::launch_selftest(h->ix, d, h->stream);
    unsigned long long f[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(f, d, sizeof(f), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    cudaFree(d);
    CUDA_TRY(e);
    failures[0] = f[0];
    failures[1] = f[1];
    return EAT_OK;
}

eat_status eat_probe_read(const void *d_buf, uint64_t bytes, uint32_t reps, void *cuda_stream) {
    if (!d_buf || (reinterpret_cast<uintptr_t>(d_buf) & 15u) || (bytes & 15u))
        return fail(EAT_EINVAL, "eat_probe_read: NULL or misaligned buffer");
    CUDA_TRY(eat::launch_read_probe(static_cast<const uint4 *>(d_buf), bytes / 16, reps,
                                    static_cast<cudaStream_t>(cuda_stream)));
    return EAT_OK;
}

eat_status eat_partition_range(const eat_handle *h, uint32_t rank, uint32_t count, uint32_t *lo, uint32_t *hi) {
    if (!h || !lo || !hi || count == 0 || rank >= count) return fail(EAT_EINVAL, "bad partition arguments");
    eat::partition_range(h->hx, rank, count, *lo, *hi);
    return EAT_OK;
}

eat_status eat_index_sizes(const eat_handle *h, uint64_t *num_types, uint64_t *num_cluster_records,
                           uint64_t *num_pool_items) {
    if (!h) return fail(EAT_EINVAL, "NULL handle");
    if (num_types) *num_types = h->hx.num_types;
    if (num_cluster_records) *num_cluster_records = h->hx.num_crec;
    if (num_pool_items) *num_pool_items = h->hx.pool.size();
    return EAT_OK;
}

}  // extern "C"
