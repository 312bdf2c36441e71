"""The random-gather ceiling C4 runs against (development tool): 4-byte
reads at hashed positions of an L2-resident x (2^20 int32 = 4 MB), no other
traffic, so every read is one 32-byte L2 sector -- next to C4's own rate
(nnz / kernel time).  NVRTC-compiled here; not part of the product.

python tools/l2_gather_bench.py
"""

import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import jit  # noqa: E402

SRC = r"""
typedef unsigned long long u64;
__device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
extern "C" __global__ void __launch_bounds__(256) rand_gather(const int* __restrict__ x, int mask, long long n,
                                                               int* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  int acc = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride * 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const u64 h = mix64((u64)(i + u * stride));
      acc += __ldg(&x[(int)(h & (u64)mask)]);
    }
  }
  if (acc == 0x7fffffff) out[0] = acc;
}
"""


def main():
    dev = torch.device("cuda")
    kern = jit._Kernel(SRC, ("rand_gather",))
    from cuda.bindings import driver

    ncols = 1 << 20
    x = torch.randint(-(1 << 15), 1 << 15, (ncols,), dtype=torch.int32, device=dev)
    out = torch.zeros(1, dtype=torch.int32, device=dev)
    n = 1 << 28
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    grid = sms * 8

    def launch():
        vals = [ctypes.c_void_p(x.data_ptr()), ctypes.c_int(ncols - 1), ctypes.c_longlong(n),
                ctypes.c_void_p(out.data_ptr())]
        argv = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
        (err,) = driver.cuLaunchKernel(kern.fns["rand_gather"], grid, 1, 1, 256, 1, 1, 0,
                                       torch.cuda.current_stream().cuda_stream, ctypes.addressof(argv), 0)
        assert int(err) == 0

    for _ in range(3):
        launch()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        launch()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(json.dumps({"random_4B_gathers": n, "ms": ms, "Ggathers_per_s": n / ms / 1e6,
                      "l2_sector_GBs": 32 * n / ms / 1e6, "x_bytes": 4 * ncols}))


if __name__ == "__main__":
    main()
