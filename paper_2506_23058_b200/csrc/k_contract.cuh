// k_contract.cuh -- device checks of an entry function's preconditions.
//
// The verifier proves a site's check unnecessary ASSUMING the function's
// parameter annotations (infer.py:231-338: Range / Inj / Bij / Mono are
// assumed, never checked).  The reference interpreter never looks at them
// (oracle.py:117-135), so a caller that violates them still gets the
// reference's own answer -- the drop-in executor therefore checks them on
// the device before it uses ELIDED variants (contract.py), and runs the
// CHECKED variants when one fails.  The checks restate the reference's own
// concrete predicates chk_range / chk_inj / chk_bij / chk_mono
// (oracle.py:478-520); each is one streaming pass over the annotated array.
#pragma once
#include "k_generic.cuh"

namespace ixg {

// out2 = [min, max] of xs (caller-initialised to [INT64_MAX, INT64_MIN]):
// 16-byte loads, warp shuffles, one 64-bit atomic pair per warp
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_minmax(const E* __restrict__ xs, long long n,
                                                       long long* __restrict__ out2) {
  constexpr int V = 16 / (int)sizeof(E);
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  const bool vec = (((uintptr_t)xs) & 15) == 0;
  const long long nv = vec ? n / V : 0;
  for (long long k = tid; k < nv; k += stride) {
    const int4 v = ld_stream_v4(xs + k * V);
    const E* e = reinterpret_cast<const E*>(&v);
#pragma unroll
    for (int q = 0; q < V; ++q) {
      const long long x = (long long)e[q];
      lo = x < lo ? x : lo;
      hi = x > hi ? x : hi;
    }
  }
  for (long long i = nv * V + tid; i < n; i += stride) {
    const long long x = (long long)xs[i];
    lo = x < lo ? x : lo;
    hi = x > hi ? x : hi;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    const long long a = __shfl_xor_sync(0xffffffffu, lo, d), b = __shfl_xor_sync(0xffffffffu, hi, d);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  if (lane_id() == 0 && lo <= hi) {
    atomicMin(&out2[0], lo);
    atomicMax(&out2[1], hi);
  }
}

// Mono xs op (chk_mono, oracle.py:483-487): *bad += number of adjacent pairs
// (xs[i], xs[i+1]) violating op (0 <=, 1 <, 2 >=, 3 >)
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_mono(const E* __restrict__ xs, long long n, int op,
                                                     unsigned long long* __restrict__ bad) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long cnt = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i + 1 < n; i += stride) {
    const long long a = (long long)xs[i], b = (long long)xs[i + 1];
    const bool ok = op == 0 ? a <= b : op == 1 ? a < b : op == 2 ? a >= b : a > b;
    cnt += ok ? 0 : 1;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
  if (lane_id() == 0 && cnt) atomicAdd(bad, cnt);
}

// Inj / Bij over the values in [lo, lo + nbits) (chk_inj / chk_bij,
// oracle.py:492-520): every in-range value claims bit v - lo of a zeroed
// bitmap; out3[0] += in-range count, out3[1] += second claims (duplicates),
// out3[2] += in-range values outside [img_lo, img_hi]
__global__ void __launch_bounds__(kGThreads) k_inj_claim(const long long* __restrict__ xs, long long n,
                                                          long long lo, unsigned long long nbits,
                                                          long long img_lo, long long img_hi,
                                                          uint32_t* __restrict__ bitmap,
                                                          unsigned long long* __restrict__ out3) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long in = 0, dup = 0, out_img = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long v = __ldcs(&xs[i]);
    const unsigned long long r = (unsigned long long)v - (unsigned long long)lo;
    if (r < nbits) {
      ++in;
      out_img += (v < img_lo || v > img_hi) ? 1 : 0;
      const uint32_t bit = 1u << (r & 31);
      if (atomicOr(&bitmap[r >> 5], bit) & bit) ++dup;
    }
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    in += __shfl_xor_sync(0xffffffffu, in, d);
    dup += __shfl_xor_sync(0xffffffffu, dup, d);
    out_img += __shfl_xor_sync(0xffffffffu, out_img, d);
  }
  if (lane_id() == 0) {
    if (in) atomicAdd(&out3[0], in);
    if (dup) atomicAdd(&out3[1], dup);
    if (out_img) atomicAdd(&out3[2], out_img);
  }
}

}  // namespace ixg
