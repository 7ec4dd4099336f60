// async.cuh -- CTA-partitioned asynchronous single-query kernel (async.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace eat {

struct AsyncWork {
    uint32_t *garr = nullptr;       // [n] e[] mirror (the result), internal ids
    uint32_t *inflag = nullptr;     // [n] "message pending" flags
    uint32_t *inbox = nullptr;      // [2][n] per-round-parity inboxes; owner c's region starts at c*span
    uint32_t *inbox_cnt = nullptr;  // [2][P] inbox fill counts
    uint32_t *ctl = nullptr;        // [kCtlWords]: 0-2 message counters (rotating), 8 rounds, 9 sweeps, kBarWord grid barrier
};

cudaError_t async_alloc(AsyncWork &w, uint32_t n, uint32_t max_parts);
void async_free(AsyncWork &w);
size_t async_smem_bytes(uint32_t span);
// Number of CTAs (partitions) the async kernel uses for n vertices; 0 if a slice does not fit shared memory.
int async_parts(uint32_t n);
cudaError_t launch_query_async(const DevIndex &ix, const AsyncWork &w, uint32_t s, uint32_t t_s, uint32_t *d_out,
                               cudaStream_t st);

}  // namespace eat
