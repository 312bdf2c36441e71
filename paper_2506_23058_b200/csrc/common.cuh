// common.cuh -- shared device helpers for the sm_100a index-array kernels.
//
// Everything on this path is HBM-bound integer work, so the
// helpers here are about moving bytes: 128-bit streaming loads/stores with
// cache hints, warp-ballot ranking, and the decoupled look-back tile state
// used by every single-pass scan (lookback.cuh).
#pragma once
#include <cuda_runtime.h>
#include <limits.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/ixgpu.h"

#define IXG_DEV __device__ __forceinline__

namespace ixg {

constexpr int kWarp = 32;

// ---------------------------------------------------------------- memory ops
// Streaming (read-once) 128-bit load: bypass L1 allocation, evict-first in L2.
IXG_DEV int4 ld_stream_v4(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
IXG_DEV void st_stream_v4(void* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
IXG_DEV uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
IXG_DEV void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
IXG_DEV long long ld_relaxed_s64(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
IXG_DEV void st_relaxed_s64(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

IXG_DEV uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// named barrier over the first `nthreads` threads (id 0 is __syncthreads)
IXG_DEV void bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
IXG_DEV void bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Programmatic dependent launch (sm_90+): a kernel launched with the
// programmatic-serialization attribute may start while its predecessor in
// the stream still runs; pdl_wait() blocks the calling thread until the
// predecessor grid has completed and its writes are visible (a no-op for a
// kernel launched without a programmatic dependency).  pdl_trigger() lets
// this grid's dependents launch once every CTA of this grid has issued it.
IXG_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
IXG_DEV void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

IXG_DEV int lane_id() { return threadIdx.x & 31; }
IXG_DEV int warp_id() { return threadIdx.x >> 5; }

// ----------------------------------------------- generator + predicate semantics
// Bit-identical to oracle/ixoracle.c (ixo_mix64 / ixo_rand / ixo_pred_eval)
// and to paper_2506_23058_b200/pred.py.
IXG_DEV uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
IXG_DEV uint64_t rand_at(uint64_t seed_mixed, uint64_t i) {
  return mix64(i * 0x9E3779B97F4A7C15ULL + seed_mixed);
}
__host__ __device__ inline uint64_t seed_mix_host(uint64_t seed) {
  uint64_t z = seed ^ 0x5851F42D4C957F2DULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// The predicate is passed by value; kind is warp-uniform so the switch does
// not diverge.  `p x` of the reference (oracle.py:327-329).
IXG_DEV bool pred_eval(const ixg_pred& p, long long x) {
  switch (p.kind) {
    case IXG_PRED_LT: return x < p.thr;
    case IXG_PRED_GT: return x > p.thr;
    case IXG_PRED_LE: return x <= p.thr;
    case IXG_PRED_GE: return x >= p.thr;
    case IXG_PRED_EQ: return x == p.thr;
    case IXG_PRED_NE: return x != p.thr;
    case IXG_PRED_HASH: return (mix64((uint64_t)x ^ p.seed) >> 63) != 0;
    case IXG_PRED_TRUE: return true;
    default: return false;
  }
}

// The six comparison kinds as one interval test in the element's own width:
// `p x` <=> ((U)(x - lo) <= span) xor inv, with [lo, lo + span] the set of
// T values satisfying the comparison (clamped to T's range; `none` = empty).
// One subtract + one unsigned compare per element instead of a sign-extended
// 64-bit compare; identical truth table to pred_eval for every T value.
template <typename T>
struct PredRange {
  using U = typename std::conditional<sizeof(T) == 4, uint32_t, unsigned long long>::type;
  U lo, span;
  uint32_t keep, flip;  // mask = (mask & keep) ^ flip over 16 bits
  IXG_DEV bool test(T x) const { return (U)((U)x - lo) <= span; }
};
template <typename T>
IXG_DEV PredRange<T> pred_range(const ixg_pred& p) {
  using U = typename PredRange<T>::U;
  constexpr long long TMIN = sizeof(T) == 4 ? (long long)INT32_MIN : LLONG_MIN;
  constexpr long long TMAX = sizeof(T) == 4 ? (long long)INT32_MAX : LLONG_MAX;
  long long lo = LLONG_MIN, hi = LLONG_MAX;
  const long long t = p.thr;
  bool none = false, inv = false;
  switch (p.kind) {
    case IXG_PRED_LT: none = (t == LLONG_MIN); hi = t - (none ? 0 : 1); break;
    case IXG_PRED_GT: none = (t == LLONG_MAX); lo = t + (none ? 0 : 1); break;
    case IXG_PRED_LE: hi = t; break;
    case IXG_PRED_GE: lo = t; break;
    case IXG_PRED_EQ: lo = hi = t; break;
    default: lo = hi = t; inv = true; break;  // NE
  }
  lo = lo < TMIN ? TMIN : lo;
  hi = hi > TMAX ? TMAX : hi;
  none = none || lo > hi;
  PredRange<T> r;
  r.lo = none ? (U)0 : (U)lo;
  r.span = none ? (U)0 : (U)((U)hi - (U)lo);
  r.keep = none ? 0u : 0xffffu;
  r.flip = inv ? 0xffffu : 0u;
  return r;
}

// ------------------------------------------------------------ status word
// First failure in the reference's sequential order: key =
// [stmt:8][elem:48][site:8]; the smallest key wins (atomicMin).  The host
// (errors.py) maps it back to OutOfBounds / NonIdempotentScatter.
IXG_DEV unsigned long long status_key(int stmt, long long elem, int site) {
  return ((unsigned long long)(stmt & 0xff) << 56) |
         (((unsigned long long)elem & 0xffffffffffffULL) << 8) | (unsigned long long)(site & 0xff);
}
IXG_DEV void status_fail(ixg_status* st, int code, int stmt, long long elem, int site) {
  if (!st) return;
  atomicMin(&st->first, status_key(stmt, elem, site));
  atomicOr(&st->codes, 1u << code);
}

// ------------------------------------------------------ checked int64 arithmetic
// The reference's ints are unbounded (oracle.py:214-240): each op returns the
// wrapped result and whether the exact one left int64.
IXG_DEV bool add_ovf(long long a, long long b, long long* r) {
  const long long s = (long long)((unsigned long long)a + (unsigned long long)b);
  *r = s;
  return ((a ^ s) & (b ^ s)) < 0;
}
IXG_DEV bool sub_ovf(long long a, long long b, long long* r) {
  const long long s = (long long)((unsigned long long)a - (unsigned long long)b);
  *r = s;
  return ((a ^ b) & (a ^ s)) < 0;
}
IXG_DEV bool mul_ovf(long long a, long long b, long long* r) {
  const long long lo = (long long)((unsigned long long)a * (unsigned long long)b);
  *r = lo;
  return __mul64hi(a, b) != (lo >> 63);
}
// Did the sequential step prev + x = cur (all wrapped) overflow?  Exact for
// a scan: at the first position whose true prefix leaves int64 every earlier
// wrapped prefix equals the true one (modular arithmetic is exact until
// then), so checking cur against cur - x at every position finds it.
IXG_DEV bool step_ovf(long long cur, long long x) {
  const long long prev = (long long)((unsigned long long)cur - (unsigned long long)x);
  return ((prev ^ cur) & (x ^ cur)) < 0;
}
IXG_DEV void status_overflow(ixg_status* st, int stmt, long long elem) {
  status_fail(st, IXG_OVERFLOW, stmt, elem, IXG_OVF_SITE);
}

// --------------------------------------------------------- vector helpers
template <typename T>
struct Vec;
template <>
struct Vec<int32_t> {
  static constexpr int N = 4;
  IXG_DEV static void unpack(int4 v, int32_t (&o)[4]) { o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
  IXG_DEV static int4 pack(const int32_t (&o)[4]) { return make_int4(o[0], o[1], o[2], o[3]); }
};
template <>
struct Vec<int64_t> {
  static constexpr int N = 2;
  IXG_DEV static void unpack(int4 v, int64_t (&o)[2]) {
    o[0] = (int64_t)(((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x);
    o[1] = (int64_t)(((uint64_t)(uint32_t)v.w << 32) | (uint32_t)v.z);
  }
  IXG_DEV static int4 pack(const int64_t (&o)[2]) {
    return make_int4((int)(uint32_t)o[0], (int)(uint32_t)((uint64_t)o[0] >> 32), (int)(uint32_t)o[1],
                     (int)(uint32_t)((uint64_t)o[1] >> 32));
  }
};

template <>
struct Vec<long long> {
  static constexpr int N = 2;
  IXG_DEV static void unpack(int4 v, long long (&o)[2]) {
    o[0] = (long long)(((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x);
    o[1] = (long long)(((uint64_t)(uint32_t)v.w << 32) | (uint32_t)v.z);
  }
  IXG_DEV static int4 pack(const long long (&o)[2]) {
    return make_int4((int)(uint32_t)o[0], (int)(uint32_t)((uint64_t)o[0] >> 32), (int)(uint32_t)o[1],
                     (int)(uint32_t)((uint64_t)o[1] >> 32));
  }
};

// ---------------------------------------------------------------- tracing
// Build with -DIXG_TRACE to record %globaltimer at fixed points of the
// compaction kernels (thread 0 of the first 2^17 CTAs); read with
// ixg_trace_read().  Compiled out otherwise.
#ifdef IXG_TRACE
#define IXG_TRS 20  // trace slots per CTA
#ifdef IXG_TRACE_CLK  // SM cycle counter: exact within a CTA, not across SMs
#define IXG_TR_NOW(t) asm volatile("mov.u64 %0, %%clock64;" : "=l"(t))
#else
#define IXG_TR_NOW(t) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t))
#endif
__device__ unsigned long long g_trace[(1 << 17) * IXG_TRS];
#define IXG_TR(slot)                                                        \
  do {                                                                      \
    if (threadIdx.x == 0 && blockIdx.x < (1u << 17)) {                      \
      unsigned long long t__;                                               \
      IXG_TR_NOW(t__);                                                      \
      g_trace[blockIdx.x * IXG_TRS + (slot)] = t__;                               \
    }                                                                       \
  } while (0)
#define IXG_TR_LANE0(slot)                                                  \
  do {                                                                      \
    if ((threadIdx.x & 31) == 0 && blockIdx.x < (1u << 17)) {               \
      unsigned long long t__;                                               \
      IXG_TR_NOW(t__);                                                      \
      g_trace[blockIdx.x * IXG_TRS + (slot)] = t__;                               \
    }                                                                       \
  } while (0)
#else
#define IXG_TR(slot) \
  do {               \
  } while (0)
#define IXG_TR_LANE0(slot) \
  do {                     \
  } while (0)
#endif

// SM count of the CURRENT device (cached per device ordinal)
inline int num_sms() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  dev &= 63;
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

inline int cuda_rc(cudaError_t e) { return e == cudaSuccess ? IXG_OK : IXG_CUDA_ERR + (int)e; }

}  // namespace ixg
