// k_stream.cuh -- shared pieces of the streaming kernels: 256-bit
// streaming loads/stores, the decoded predicate (Selector: the comparison
// kinds as one interval test in the element's width), and the class-count
// pass of the CHECKED partition pipelines.  The ELIDED compaction kernels
// (filter / C2 / partition) are the big-tile kernels of k_big.cuh.
#pragma once
#include <type_traits>

#include "lookback.cuh"

namespace ixg {

constexpr int kSThreads = 256;  // non-tiled helper kernels
constexpr int kSItems = 16;
constexpr int kSWarps = kSThreads / 32;

IXG_DEV void ld256(const void* p, uint32_t (&r)[8]) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}
IXG_DEV void st256(void* p, const uint32_t (&r)[8]) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]),
               "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

IXG_DEV uint32_t valid_mask(long long i0, long long n) {
  const long long valid = n - i0;
  return valid <= 0 ? 0u : (valid >= kSItems ? 0xffffu : ((1u << valid) - 1u));
}

// The predicate of a kernel, decoded once per thread: the comparison kinds
// become an interval test (common.cuh PredRange), HASH keeps its seed.
// sign bits of 16 int32 (bit j set iff x[j] < 0): the four top bytes of a
// 16-byte piece gathered with two-level byte permutes, their sign bits packed
// into a nibble by one multiply (bits 7/15/23/31 -> 28..31, no carries)
template <typename T>
IXG_DEV uint32_t sign16(const T (&x)[kSItems]) {
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < kSItems / 4; ++k) {
    const uint32_t a = __byte_perm((uint32_t)x[4 * k], (uint32_t)x[4 * k + 1], 0x0073);
    const uint32_t b = __byte_perm((uint32_t)x[4 * k + 2], (uint32_t)x[4 * k + 3], 0x0073);
    const uint32_t w = __byte_perm(a, b, 0x5410);
    m |= (((w & 0x80808080u) * 0x00204081u) >> 28) << (4 * k);
  }
  return m;
}

#ifndef IXG_SIGN_SEL
#define IXG_SIGN_SEL 1
#endif
template <typename T, bool kSign = true>
struct Selector {
  int kind;  // IXG_PRED_LT..NE -> range test
  PredRange<T> r;
  uint64_t seed;
  int sgn;  // int32 half ranges [INT_MIN, -1] (1) / [0, INT_MAX] (2): a sign-bit test
  IXG_DEV explicit Selector(const ixg_pred& p) : kind(p.kind), r(pred_range<T>(p)), seed(p.seed) {
    sgn = (kSign && IXG_SIGN_SEL && sizeof(T) == 4 && kind <= IXG_PRED_NE && r.keep && (unsigned long long)r.span == 0x7fffffffull &&
           ((unsigned long long)r.lo == 0ull || (unsigned long long)r.lo == 0x80000000ull))
              ? ((unsigned long long)r.lo ? 1 : 2)
              : 0;
  }
  // selection mask of 16 elements; the kind is uniform, so no divergence
  IXG_DEV uint32_t mask(const T (&x)[kSItems]) const {
    uint32_t m = 0;
    if (kSign && sizeof(T) == 4 && sgn) {
      m = sign16(x);
      return (sgn == 1 ? m : (~m & 0xffffu)) ^ r.flip;
    }
    if (kind <= IXG_PRED_NE) {
#pragma unroll
      for (int j = 0; j < kSItems; ++j) m |= (uint32_t)r.test(x[j]) << j;
      return (m & r.keep) ^ r.flip;
    }
    if (kind == IXG_PRED_HASH) {
#pragma unroll
      for (int j = 0; j < kSItems; ++j) m |= (uint32_t)(mix64((uint64_t)(long long)x[j] ^ seed) >> 63) << j;
      return m;
    }
    return kind == IXG_PRED_TRUE ? 0xffffu : 0u;
  }
};

template <typename T>
IXG_DEV uint32_t select_mask(const ixg_pred& p, const T (&x)[kSItems]) {
  return Selector<T>(p).mask(x);
}

// ---------------------------------------------------------------------------
// partition2 / partition3 class counts (the CHECKED pipelines' pass 1).
// kClasses = 2: class 0 = p x, class 1 = !p x.
// kClasses = 3: class 0 = p x, class 1 = !p x && q x, class 2 = rest.
template <typename T, int kClasses>
IXG_DEV int classify(const ixg_pred& p, const ixg_pred& q, T x) {
  if (pred_eval(p, (long long)x)) return 0;
  if (kClasses == 3 && pred_eval(q, (long long)x)) return 1;
  return kClasses - 1;
}

// Pass 1: per-CTA class counts, the last CTA adds them up into d_tot
// (self-resetting through hdr->done).
template <typename T, int kClasses>
__global__ void __launch_bounds__(kSThreads) k_class_count(const T* __restrict__ xs, long long n, ixg_pred p,
                                                           ixg_pred q, long long* partials, LBHeader* hdr,
                                                           long long* d_tot) {
  constexpr int V = 32 / (int)sizeof(T);
  long long c0 = 0, c1 = 0;
  const long long nv = n / V;
  const long long stride = (long long)gridDim.x * kSThreads;
  for (long long i = (long long)blockIdx.x * kSThreads + threadIdx.x; i < nv; i += stride) {
    uint32_t r[8];
    ld256(xs + i * V, r);
    const T* x = reinterpret_cast<const T*>(r);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int c = classify<T, kClasses>(p, q, x[e]);
      c0 += (c == 0);
      if (kClasses == 3) c1 += (c == 1);
    }
  }
  if (blockIdx.x == 0)
    for (long long i = nv * V + threadIdx.x; i < n; i += kSThreads) {
      const int c = classify<T, kClasses>(p, q, xs[i]);
      c0 += (c == 0);
      if (kClasses == 3) c1 += (c == 1);
    }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    c0 += __shfl_xor_sync(0xffffffffu, c0, d);
    c1 += __shfl_xor_sync(0xffffffffu, c1, d);
  }
  __shared__ long long s0[kSWarps], s1[kSWarps];
  __shared__ bool s_last;
  if (lane_id() == 0) {
    s0[warp_id()] = c0;
    s1[warp_id()] = c1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0;
    for (int w = 0; w < kSWarps; ++w) {
      a += s0[w];
      b += s1[w];
    }
    __stcg(&partials[2 * blockIdx.x], a);
    __stcg(&partials[2 * blockIdx.x + 1], b);
    __threadfence();
    s_last = atomicAdd(&hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    long long a = 0, b = 0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kSThreads) {
      a += __ldcg(&partials[2 * i]);
      b += __ldcg(&partials[2 * i + 1]);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, d);
      b += __shfl_xor_sync(0xffffffffu, b, d);
    }
    if (lane_id() == 0) {
      s0[warp_id()] = a;
      s1[warp_id()] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long ta = 0, tb = 0;
      for (int w = 0; w < kSWarps; ++w) {
        ta += s0[w];
        tb += s1[w];
      }
      d_tot[0] = ta;
      if (kClasses == 3) d_tot[1] = tb;
      hdr->done = 0;
    }
  }
}

}  // namespace ixg
