// partition.cuh -- edge-partitioned single query (north star: "a single huge
// query is edge-partitioned with one NCCL allreduce(min) on the arrival
// array per sweep over NVLink").  Each rank owns the out-types of a
// contiguous internal vertex range [lo, hi) and a full e[] replica.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "eat.h"
#include "kernels.cuh"

namespace eat {

struct PartWork {
    uint32_t *arr = nullptr;     // [n+1]: e[] replica + exchange flag word at [n]
    uint32_t *prev = nullptr;    // [n]: e[] as contributed to the last exchange
    uint32_t *q0 = nullptr, *q1 = nullptr, *stamp = nullptr;  // [n] local worklists + dedup stamps
    uint32_t *ctl = nullptr;     // [kCtlWords] counters / sweeps / stamp base, kBarWord grid barrier
    uint32_t *h_flag = nullptr;  // pinned: flag word after exchange
    uint32_t n = 0;
    uint32_t h_sweeps = 0;       // sweeps of the last query (host copy)
    uint32_t local_sweeps_per_round = 0;  // 0 = to local quiescence; k = at most k sweeps per round
                                          // (eat_build_opts.local_sweeps; 1 = one allreduce per sweep)
    bool comm_dead = false;      // the communicator was aborted after an asynchronous NCCL error
};

cudaError_t part_alloc(PartWork &w, uint32_t n);
void part_free(PartWork &w);

// One exchange round's local phase (persistent cooperative kernel).
cudaError_t launch_part_round(const DevIndex &ix, const PartWork &w, uint32_t lo, uint32_t hi, int subwarp,
                              bool first, uint32_t s, uint32_t t_s, cudaStream_t st);

// Elementwise min of `count` u32 words of src into dst (loopback exchange).
cudaError_t launch_min_merge(uint32_t *dst, const uint32_t *src, uint64_t count, cudaStream_t st);

// Gather caller-ordered output out[i] = arr[perm[i]].
cudaError_t launch_gather(const DevIndex &ix, const uint32_t *arr, uint32_t *out, cudaStream_t st);

// Whole query: rounds of {local relax; ncclAllReduce(min) of e[] ++ flag} until
// no rank lowered a vertex it does not own.  comm may be NULL (one partition).
eat_status part_query(const DevIndex &ix, PartWork &w, ncclComm_t comm, uint32_t lo, uint32_t hi, int subwarp,
                      uint32_t s, uint32_t t_s, uint32_t *d_out, cudaStream_t st, uint32_t *rounds,
                      uint32_t *sweeps, std::string &err);

// All P partitions on one device (tests / single-GPU runs of the e2 path):
// the exchange is a device min-merge of the P e[] ++ flag buffers.
eat_status part_query_loopback(const std::vector<DevIndex> &ix, std::vector<PartWork *> &w,
                               const std::vector<uint32_t> &lo, const std::vector<uint32_t> &hi, int subwarp,
                               uint32_t s, uint32_t t_s, uint32_t *d_out, cudaStream_t st, uint32_t *rounds,
                               uint32_t *sweeps, std::string &err);

}  // namespace eat
