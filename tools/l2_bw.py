"""Microbenchmark: L2-resident and HBM read bandwidth on this B200 (context for
the batched kernel, whose index is L2-resident).  A plain grid-stride
uint4 read kernel (148 x 8 CTAs of 256 threads) over buffers of 16 MiB -
4 GiB, repeated; CUDA events.  Prints one JSON line (GB/s per size)."""
import json

import torch
from torch.utils.cpp_extension import load_inline

SRC = r"""
#include <torch/extension.h>
__global__ void rd(const uint4* __restrict__ p, size_t n, int reps, unsigned* out) {
  unsigned acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      uint4 v = __ldcg(p + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345678u) out[0] = acc;
}
void run(torch::Tensor buf, int reps, torch::Tensor out) {
  size_t n = buf.numel() * buf.element_size() / 16;
  rd<<<148 * 8, 256>>>((const uint4*)buf.data_ptr(), n, reps, (unsigned*)out.data_ptr());
}
"""
CPP = "void run(torch::Tensor buf, int reps, torch::Tensor out);"
mod = load_inline("l2bw", cpp_sources=CPP, cuda_sources=SRC, functions=["run"],
                  extra_cuda_cflags=["-O3", "-gencode", "arch=compute_100a,code=sm_100a"], verbose=False)
res = {}
out = torch.zeros(4, dtype=torch.int32, device="cuda")
for mib in (16, 32, 64, 96, 512, 4096):
    buf = torch.ones(mib * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    reps = max(1, 4096 // mib)
    mod.run(buf, 1, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    mod.run(buf, reps, out)
    b.record()
    b.synchronize()
    res[f"read_{mib}MiB_GBps"] = buf.numel() * 4 * reps / (a.elapsed_time(b) / 1e3) / 1e9
print(json.dumps(res))
