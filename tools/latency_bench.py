"""Microbenchmarks for the single-query sweep floor on this B200: software
grid barrier cost per sweep (the one device_common.cuh uses) at 148/296/592
CTAs, and dependent-latency chains (L2-resident pointer chase, global
atomicMin / atomicExch on L2-resident words, HBM pointer chase)."""
import json
import torch
from torch.utils.cpp_extension import load_inline

src = r'''
#include <cuda/atomic>
#include <torch/extension.h>
__device__ __forceinline__ void grid_sync(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> cnt(bar[0]);
        cuda::atomic_ref<unsigned, cuda::thread_scope_device> gen(bar[1]);
        const unsigned g = gen.load(cuda::memory_order_relaxed);
        __threadfence();
        if (cnt.fetch_add(1u, cuda::memory_order_acq_rel) == gridDim.x - 1u) {
            cnt.store(0u, cuda::memory_order_relaxed);
            gen.fetch_add(1u, cuda::memory_order_release);
        } else {
            while (gen.load(cuda::memory_order_acquire) == g) {}
        }
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_bar(unsigned *bar, int iters) { for (int i = 0; i < iters; ++i) grid_sync(bar); }
// monotonic-counter barrier: red.release arrive, acquire-poll the same word
__device__ __forceinline__ void grid_sync_mono(unsigned *cnt, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(cnt) : "memory");
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(cnt) : "memory"); } while (v < target);
    }
    __syncthreads();
}
__global__ void k_bar_mono(unsigned *bar, int iters) {
    for (int i = 0; i < iters; ++i) grid_sync_mono(bar, (unsigned)(i + 1) * gridDim.x);
}
// same without acquire/release on the poll (relaxed + fences)
__device__ __forceinline__ void grid_sync_mono_f(unsigned *cnt, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(cnt, 1u);
        while (*(volatile unsigned *)cnt < target) {}
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_bar_mono_f(unsigned *bar, int iters) {
    for (int i = 0; i < iters; ++i) grid_sync_mono_f(bar, (unsigned)(i + 1) * gridDim.x);
}
__global__ void k_chase(const unsigned *next, int hops, unsigned *out) {
    unsigned x = 0;
    for (int i = 0; i < hops; ++i) x = __ldcg(next + x);
    out[0] = x;
}
__global__ void k_atom(unsigned *a, int hops, unsigned *out, int kind) {
    unsigned x = 0;
    for (int i = 0; i < hops; ++i) {
        unsigned idx = (x * 2654435761u + i * 97u) & ((1u << 18) - 1u);
        x = kind == 0 ? atomicMin(a + idx, 0xFFFFFFFFu - i) : atomicExch(a + idx, i);
        x &= 1023u;
    }
    out[0] = x;
}
double bar_us(int grid, int iters, int kind, int threads) {
    auto bar = torch::zeros({2}, torch::dtype(torch::kInt32).device(torch::kCUDA));
    unsigned *b = (unsigned *)bar.data_ptr();
    void *args[] = {&b, &iters};
    void *k = kind == 0 ? (void *)k_bar : (kind == 1 ? (void *)k_bar_mono : (void *)k_bar_mono_f);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchCooperativeKernel(k, dim3(grid), dim3(threads), args, 0, 0);
    cudaMemset(b, 0, 8);
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel(k, dim3(grid), dim3(threads), args, 0, 0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1000.0 / iters;
}
double chase_ns(torch::Tensor next, int hops) {
    auto out = torch::zeros({1}, next.options());
    k_chase<<<1, 1>>>((unsigned *)next.data_ptr(), 64, (unsigned *)out.data_ptr());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_chase<<<1, 1>>>((unsigned *)next.data_ptr(), hops, (unsigned *)out.data_ptr());
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e6 / hops;
}
double atom_ns(torch::Tensor a, int hops, int kind) {
    auto out = torch::zeros({1}, a.options());
    k_atom<<<1, 1>>>((unsigned *)a.data_ptr(), 64, (unsigned *)out.data_ptr(), kind);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_atom<<<1, 1>>>((unsigned *)a.data_ptr(), hops, (unsigned *)out.data_ptr(), kind);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e6 / hops;
}
'''
m = load_inline("latbench", cpp_sources="double bar_us(int, int, int, int); double chase_ns(torch::Tensor, int); double atom_ns(torch::Tensor, int, int);",
                cuda_sources=src, functions=["bar_us", "chase_ns", "atom_ns"],
                extra_cuda_cflags=["-gencode", "arch=compute_100a,code=sm_100a", "-O3"], verbose=False)
res = {}
for g in (148, 296, 592, 1184):
    res[f"grid_sync_us_{g}ctas"] = m.bar_us(g, 2000, 0, 256)
for kind, name in ((0, "gen"), (1, "mono_acqrel"), (2, "mono_fence")):
    res[f"grid_sync_{name}_us_148x1024"] = m.bar_us(148, 2000, kind, 1024)
for mb in (1, 64, 1024):
    n = mb * 1024 * 1024 // 4
    perm = torch.randperm(n, dtype=torch.int64)
    nxt = torch.empty(n, dtype=torch.int64)
    nxt[perm] = torch.roll(perm, -1)
    res[f"chase_ns_{mb}MiB"] = m.chase_ns(nxt.to(torch.int32).cuda(), 20000)
a = torch.zeros(1 << 18, dtype=torch.int32, device="cuda")
res["atomicMin_chain_ns"] = m.atom_ns(a, 20000, 0)
res["atomicExch_chain_ns"] = m.atom_ns(a, 20000, 1)
print(json.dumps(res))
