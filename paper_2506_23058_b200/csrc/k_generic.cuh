// k_generic.cuh -- the builtins one kernel each (scan, segmented scan,
// scatter with/without the idempotence check, gather with/without bounds
// checks, hist, replicate, iota) and the CHECKED forms of the corpus
// pipelines, which materialise their index arrays exactly as the reference
// program does (the dynamic check needs the index array).
#pragma once
#include <type_traits>

#include "k_stream.cuh"
#include "lookback.cuh"

namespace ixg {

constexpr int kGThreads = 256;
constexpr int kGItems = 16;
constexpr int kGTile = kGThreads * kGItems;

// ---------------------------------------------------------------- loads
// 16 consecutive elements of E[] from i0 as int64: 256-bit (u8: 128-bit)
// vector loads when the 16 are in range and the address is aligned, else
// bounded scalar loads (out-of-range elements read as 0)
template <typename E>
IXG_DEV void load16_i64(const E* __restrict__ xs, long long i0, long long n, long long (&v)[kGItems]) {
  const E* p = xs + i0;
  if (i0 + kGItems <= n) {
    if constexpr (sizeof(E) == 1) {
      if ((((uintptr_t)p) & 15) == 0) {
        const int4 r = ld_stream_v4(p);
        const uint8_t* b = reinterpret_cast<const uint8_t*>(&r);
#pragma unroll
        for (int q = 0; q < kGItems; ++q) v[q] = (long long)b[q];
        return;
      }
    } else {
      if ((((uintptr_t)p) & 31) == 0) {
        constexpr int PER = 32 / (int)sizeof(E);
#pragma unroll
        for (int k = 0; k < kGItems / PER; ++k) {
          uint32_t r[8];
          ld256(p + k * PER, r);
          const E* e = reinterpret_cast<const E*>(r);
#pragma unroll
          for (int q = 0; q < PER; ++q) v[k * PER + q] = (long long)e[q];
        }
        return;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kGItems; ++q) v[q] = (i0 + q < n) ? (long long)p[q] : 0LL;
}

// 16 consecutive int64 (or int32) outputs from i0: four (two) 256-bit
// stores when all 16 are in range and 32-byte aligned
IXG_DEV void store16_i64(long long* __restrict__ out, long long i0, long long n, const long long (&o)[kGItems]) {
  long long* p = out + i0;
  if (i0 + kGItems <= n && (((uintptr_t)p) & 31) == 0) {
#pragma unroll
    for (int k = 0; k < kGItems / 4; ++k) {
      uint32_t r[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        r[2 * q] = (uint32_t)(unsigned long long)o[4 * k + q];
        r[2 * q + 1] = (uint32_t)((unsigned long long)o[4 * k + q] >> 32);
      }
      st256(p + 4 * k, r);
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < kGItems; ++q)
    if (i0 + q < n) p[q] = o[q];
}
IXG_DEV void store16_i32(int32_t* __restrict__ out, long long i0, long long n, const long long (&o)[kGItems]) {
  int32_t* p = out + i0;
  if (i0 + kGItems <= n && (((uintptr_t)p) & 31) == 0) {
#pragma unroll
    for (int k = 0; k < kGItems / 8; ++k) {
      uint32_t r[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = (uint32_t)o[8 * k + q];
      st256(p + 8 * k, r);
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < kGItems; ++q)
    if (i0 + q < n) p[q] = (int32_t)o[q];
}

// ---------------------------------------------------------------- sources
// A source gives thread t its 16 consecutive scan elements (load16); every
// source is typed at compile time (no per-element width switch) and loads
// with 256-bit vectors.
template <typename E>
struct SrcArrT {  // scan (+) over E[]
  const E* xs;
  IXG_DEV void load16(long long i0, long long n, SumOp::T (&v)[kGItems]) const {
    long long x[kGItems];
    load16_i64<E>(xs, i0, n, x);
#pragma unroll
    for (int q = 0; q < kGItems; ++q) v[q] = SumOp::T{x[q]};
  }
};
template <typename E>
struct SrcPredT {  // map (\x -> if p x then 1 else 0) xs, fused into the scan
  const E* xs;
  const uint8_t* cs;  // filter_by: the bool array instead of p
  ixg_pred p;
  IXG_DEV void load16(long long i0, long long n, SumOp::T (&v)[kGItems]) const {
    uint32_t m;
    if (cs) {
      long long c[kGItems];
      load16_i64<uint8_t>(cs, i0, n, c);
      m = 0;
#pragma unroll
      for (int q = 0; q < kGItems; ++q) m |= (uint32_t)(c[q] != 0) << q;
    } else {
      using TE = typename std::conditional<sizeof(E) == 4, int32_t, long long>::type;
      long long x[kGItems];
      load16_i64<E>(xs, i0, n, x);
      TE xe[kGItems];
#pragma unroll
      for (int q = 0; q < kGItems; ++q) xe[q] = (TE)x[q];
      m = Selector<TE>(p).mask(xe);
    }
    m &= valid_mask(i0, n);
#pragma unroll
    for (int q = 0; q < kGItems; ++q) v[q] = SumOp::T{(long long)((m >> q) & 1u)};
  }
};
template <typename E>
struct SrcClass3T {  // partition3: (flags1, flags2)
  const E* xs;
  ixg_pred p, q;
  IXG_DEV void load16(long long i0, long long n, Sum2Op::T (&v)[kGItems]) const {
    using TE = typename std::conditional<sizeof(E) == 4, int32_t, long long>::type;
    long long x[kGItems];
    load16_i64<E>(xs, i0, n, x);
    TE xe[kGItems];
#pragma unroll
    for (int k = 0; k < kGItems; ++k) xe[k] = (TE)x[k];
    const uint32_t vm = valid_mask(i0, n);
    const uint32_t m1 = Selector<TE>(p).mask(xe) & vm;
    const uint32_t m2 = Selector<TE>(q).mask(xe) & ~m1 & vm;
#pragma unroll
    for (int k = 0; k < kGItems; ++k) v[k] = Sum2Op::T{(long long)((m1 >> k) & 1u), (long long)((m2 >> k) & 1u)};
  }
};
template <typename EF, typename EX>
struct SrcSegT {  // (flags, xs) of the segmented scan
  const EF* flags;
  const EX* xs;
  IXG_DEV void load16(long long i0, long long n, SegOp::T (&v)[kGItems]) const {
    long long f[kGItems], x[kGItems];
    load16_i64<EF>(flags, i0, n, f);
    load16_i64<EX>(xs, i0, n, x);
#pragma unroll
    for (int q = 0; q < kGItems; ++q) v[q] = SegOp::T{x[q], f[q] != 0};
  }
};

// ---------------------------------------------------------------- epilogues
// An epilogue receives a thread's 16 inclusive prefixes at once (int64
// outputs leave as 256-bit stores).  The elements themselves are recovered
// from consecutive prefixes (xstep: wrapped differences, exact in modular
// arithmetic; SegOp's flags come as a bit mask), which keeps one array of
// 16 values live instead of two.
IXG_DEV SumOp::T xstep(const SumOp::T& prev, const SumOp::T& cur, uint32_t) {
  return SumOp::T{(long long)((unsigned long long)cur.v - (unsigned long long)prev.v)};
}
IXG_DEV Sum2Op::T xstep(const Sum2Op::T& prev, const Sum2Op::T& cur, uint32_t) {
  return Sum2Op::T{cur.a - prev.a, cur.b - prev.b};
}
IXG_DEV SegOp::T xstep(const SegOp::T& prev, const SegOp::T& cur, uint32_t f) {
  return SegOp::T{f ? cur.v : (long long)((unsigned long long)cur.v - (unsigned long long)prev.v), (int)f};
}
template <class T>
struct Run16 {  // incl[q] and the element x(q) = xstep(incl[q-1], incl[q])
  const T (&incl)[kGItems];
  const T& prev0;
  uint32_t fm;
  IXG_DEV T x(int q) const { return xstep(q ? incl[q - 1] : prev0, incl[q], (fm >> q) & 1u); }
};

struct EpiScanOut {  // out[i] = ne + inclusive (or exclusive) sum
  long long ne;
  int exclusive;
  long long* out;
  ixg_status* st;  // nullable: IXG_OVERFLOW at the first sum leaving int64
  IXG_DEV void operator()(long long i0, long long n, const Run16<SumOp::T>& r) const {
    long long o[kGItems];
    long long ovf = -1;
#pragma unroll
    for (int q = 0; q < kGItems; ++q) {
      const long long x = r.x(q).v;
      const long long cur = (long long)((unsigned long long)ne + (unsigned long long)r.incl[q].v);
      if (ovf < 0 && i0 + q < n && step_ovf(cur, x)) ovf = i0 + q;  // the reference's left fold, exactly
      o[q] = exclusive ? (long long)((unsigned long long)cur - (unsigned long long)x) : cur;
    }
    if (ovf >= 0) status_overflow(st, 0, ovf);
    store16_i64(out, i0, n, o);
  }
};
struct EpiFilterInds {  // filter.ixl:10-12: inds[i] = if c then offs[i]-1 else -1; count = offs[n-1]
  long long* inds;
  long long* d_count;
  IXG_DEV void operator()(long long i0, long long n, const Run16<SumOp::T>& r) const {
    long long o[kGItems];
#pragma unroll
    for (int q = 0; q < kGItems; ++q) o[q] = r.x(q).v ? r.incl[q].v - 1 : -1;
    store16_i64(inds, i0, n, o);
#pragma unroll
    for (int q = 0; q < kGItems; ++q)  // static indices: incl stays in registers
      if (i0 + q == n - 1) *d_count = r.incl[q].v;
  }
};
struct EpiPart2Inds {  // partition2.ixl:11-16 with num_true from the count pass
  const long long* d_nt;
  long long* inds;
  IXG_DEV void operator()(long long i0, long long n, const Run16<SumOp::T>& r) const {
    const long long nt = *d_nt;
    long long o[kGItems];
#pragma unroll
    for (int q = 0; q < kGItems; ++q) {
      const long long t = r.incl[q].v;               // indicesT[i]
      const long long f = (i0 + q + 1 - t) + nt;     // indicesF[i] = tmp[i] + num_true
      o[q] = r.x(q).v ? t - 1 : f - 1;
    }
    store16_i64(inds, i0, n, o);
  }
};
struct EpiPart3Inds {  // partition3.ixl:14-24 with (m1, m2) from the count pass
  const long long* d_m;
  long long* inds;
  IXG_DEV void operator()(long long i0, long long n, const Run16<Sum2Op::T>& r) const {
    const long long m1 = d_m[0], m2 = d_m[1];
    long long o[kGItems];
#pragma unroll
    for (int q = 0; q < kGItems; ++q) {
      const Sum2Op::T x = r.x(q);
      const long long inds1 = r.incl[q].a - 1, inds2 = m1 + r.incl[q].b - 1;
      const long long inds3 = m1 + m2 + (i0 + q) - (r.incl[q].a + r.incl[q].b);
      o[q] = x.a ? inds1 : (x.b ? inds2 : inds3);
    }
    store16_i64(inds, i0, n, o);
  }
};
struct EpiSegOut {  // sgmSum value (and flag) components
  int dt_out;
  void* out_v;
  uint8_t* out_f;
  ixg_status* st;
  IXG_DEV void operator()(long long i0, long long n, const Run16<SegOp::T>& r) const {
    long long o[kGItems];
    long long ovf = -1;
    bool narrow = false;
#pragma unroll
    for (int q = 0; q < kGItems; ++q) {
      const SegOp::T x = r.x(q);
      o[q] = r.incl[q].v;
      // within a segment: the step prev + x of the reference's left fold
      if (ovf < 0 && i0 + q < n && !x.f && step_ovf(o[q], x.v)) ovf = i0 + q;
      narrow |= i0 + q < n && o[q] != (long long)(int)o[q];
    }
    if (ovf >= 0) status_overflow(st, 0, ovf);
    if (dt_out == IXG_I32) {
      if (narrow && st) atomicOr(&st->flags, IXG_F_NARROW);
      store16_i32(reinterpret_cast<int32_t*>(out_v), i0, n, o);
    } else {
      store16_i64(reinterpret_cast<long long*>(out_v), i0, n, o);
    }
    if (out_f) {
#pragma unroll
      for (int q = 0; q < kGItems; ++q)
        if (i0 + q < n) out_f[i0 + q] = (uint8_t)r.incl[q].f;
    }
  }
};
struct EpiSegStarts {  // mkSgmDescr / mkFlags: ind[i] = if shape[i] <= 0 then -1 else scn[i]
  long long m;
  const long long* shape;
  long long* ind;        // nullable
  uint32_t* bits;        // nullable: set bit scn[i] (flag array as a bitmap)
  long long nbits;
  const long long* d_nbits;  // nullable: nbits on the device
  long long* d_total;    // nullable: scn[m-1] + shape[m-1]
  ixg_status* st = nullptr;  // nullable: IXG_OVERFLOW at the first prefix leaving int64 (§2.2)
  const long long* d_lo = nullptr;  // nullable: bitmap window [*d_lo, *d_lo + nb) (a shard's outputs)
  IXG_DEV void operator()(long long i0, long long n, const Run16<SumOp::T>& r) const {
    const long long nb = d_nbits ? *d_nbits : nbits;
    const long long lo = d_lo ? *d_lo : 0;
    long long o[kGItems];
    long long ovf = -1;
#pragma unroll
    for (int q = 0; q < kGItems; ++q) {
      const long long s = r.x(q).v, start = r.incl[q].v - s;
      if (ovf < 0 && i0 + q < n && step_ovf(r.incl[q].v, s)) ovf = i0 + q;
      o[q] = s <= 0 ? -1 : start;
      if (bits && i0 + q < n && s > 0 && start >= lo && start - lo < nb)
        atomicOr(&bits[(start - lo) >> 5], 1u << ((start - lo) & 31));
    }
    if (ovf >= 0) status_overflow(st, 0, ovf);
    if (ind) store16_i64(ind, i0, n, o);
    if (d_total) {
#pragma unroll
      for (int q = 0; q < kGItems; ++q)
        if (i0 + q == m - 1) *d_total = r.incl[q].v;
    }
  }
};

template <class T>
IXG_DEV uint32_t flag_mask(const T (&)[kGItems]) {
  return 0u;
}
IXG_DEV uint32_t flag_mask(const SegOp::T (&v)[kGItems]) {
  uint32_t m = 0;
#pragma unroll
  for (int q = 0; q < kGItems; ++q) m |= (uint32_t)(v[q].f != 0) << q;
  return m;
}

// Single-pass blocked scan: 16 consecutive elements per thread (vector
// loads), tiles of 4096 with decoupled look-back (lookback.cuh).  Tiles are
// numbered in the order CTAs START (an atomicAdd ticket on the channel
// header), so a tile only ever waits on tiles whose CTAs are already
// resident -- forward progress without relying on in-order block dispatch;
// the last CTA to retire resets the ticket for the next launch.  `d_n`
// (nullable): the element count known only on the device (a count pass
// before it) -- the grid covers the capacity, surplus tiles retire at once.
// resident CTAs per SM the registers must allow: 4 for the one-word monoid
// (64 registers), 3 for the two-word ones
#ifndef IXG_SCAN_MINB
#define IXG_SCAN_MINB 4
#endif
template <class M>
constexpr int scan_min_blocks() {
  return std::is_same<M, SumOp>::value ? IXG_SCAN_MINB : 3;
}

template <class M, class Src, class Epi>
__global__ void __launch_bounds__(kGThreads, scan_min_blocks<M>()) k_scan(long long n, const long long* __restrict__ d_n, Src src, Epi epi,
                                                    LBChan ch, uint32_t nonce) {
  using T = typename M::T;
  __shared__ T s_w[kGThreads / 32];
  __shared__ T s_carry;
  __shared__ long long s_tile;
  pdl_trigger();  // a PDL dependent (C2's fused kernel) may start its own loads now
  pdl_wait();     // launched as a PDL dependent (C2's mkFlags scan): the predecessor is done
  if (threadIdx.x == 0) s_tile = (long long)atomicAdd(&ch.hdr->ticket, 1u);
  if (d_n) n = *d_n;
  __syncthreads();
  const long long tile = s_tile;
  if (tile * kGTile < n) {
    const long long i0 = tile * kGTile + (long long)threadIdx.x * kGItems;
    T v[kGItems];
    src.load16(i0, n, v);
    T a = M::identity();
#pragma unroll
    for (int j = 0; j < kGItems; ++j) {
      if (i0 + j >= n) v[j] = M::identity();
      a = M::op(a, v[j]);
    }
    T inc = warp_inclusive<M>(a);
    T lex = M::shfl_up(inc, 1);
    if (lane_id() == 0) lex = M::identity();
    if (lane_id() == 31) s_w[warp_id()] = inc;
    __syncthreads();
    T wpre = M::identity(), tagg = M::identity();
#pragma unroll
    for (int w = 0; w < kGThreads / 32; ++w) {
      if (w < warp_id()) wpre = M::op(wpre, s_w[w]);
      tagg = M::op(tagg, s_w[w]);
    }
    if (threadIdx.x == 0) lb_publish<M>(ch, nonce, tile, tagg, tile == 0);
    if (warp_id() == 0) {
      T c = M::identity();
      if (tile > 0) c = lb_lookback<M>(ch, nonce, tile);
      if (lane_id() == 0) {
        s_carry = c;
        if (tile > 0) lb_publish<M>(ch, nonce, tile, M::op(c, tagg), true);
      }
    }
    __syncthreads();
    const T prev0 = M::op(M::op(s_carry, wpre), lex);
    const uint32_t fm = flag_mask(v);
    T run = prev0;
#pragma unroll
    for (int j = 0; j < kGItems; ++j) {  // v becomes the inclusive prefixes in place
      run = M::op(run, v[j]);
      v[j] = run;
    }
    epi(i0, n, Run16<T>{v, prev0, fm});
  }
  if (threadIdx.x == 0) {  // retire: the last CTA out resets the ticket
    __threadfence();
    if (atomicAdd(&ch.hdr->done, 1u) == gridDim.x - 1) {
      atomicExch(&ch.hdr->ticket, 0u);
      atomicExch(&ch.hdr->done, 0u);
    }
  }
}

// ---------------------------------------------------------------- scatter
// scatter (oracle.py:294-305).  Out-of-range indices are skipped (the
// reference semantics, both forms).  With `check`, each in-range
// destination is claimed in a bitmap (ndst/8 bytes: 64 MB at 2^29, resident
// in the 126 MB L2); a second claim raises the `dup` flag and only then
// does k_scatter_verify re-read (is, vs) and compare every value with the
// value that landed -- equal-valued duplicates are legal (oracle.py:301).
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_scatter(E* __restrict__ out, long long ndst,
                                                        const long long* __restrict__ d_ndst,
                                                        const long long* __restrict__ is,
                                                        const E* __restrict__ vs, long long m, int check,
                                                        uint32_t* __restrict__ claim, LBHeader* hdr) {
  if (d_ndst) ndst = *d_ndst;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool dup = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const long long d = __ldcs(&is[i]);
    if ((unsigned long long)d < (unsigned long long)ndst) {
      const E v = __ldcs(&vs[i]);
      if (check) {
        const uint32_t bit = 1u << (d & 31);
        if (atomicOr(&claim[d >> 5], bit) & bit) dup = true;
      }
      out[d] = v;
    }
  }
  if (__any_sync(0xffffffffu, dup) && lane_id() == 0) atomicExch(&hdr->dup, 1u);
}

template <typename E>
__global__ void __launch_bounds__(kGThreads) k_scatter_verify(const E* __restrict__ out, long long ndst,
                                                               const long long* __restrict__ d_ndst,
                                                               const long long* __restrict__ is,
                                                               const E* __restrict__ vs, long long m,
                                                               LBHeader* hdr, ixg_status* st, int stmt,
                                                               int site) {
  __shared__ bool s_last;
  if (((volatile LBHeader*)hdr)->dup == 0u) return;  // no destination claimed twice
  if (d_ndst) ndst = *d_ndst;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const long long d = is[i];
    if ((unsigned long long)d < (unsigned long long)ndst && out[d] != vs[i]) bad = true;
  }
  if (bad) status_fail(st, IXG_CONFLICT, stmt, 0, site);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    hdr->done = 0;
    hdr->dup = 0;
  }
}

// ---------------------------------------------------------------- gather
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_gather(const E* __restrict__ arr, long long len,
                                                       const long long* __restrict__ idx, long long n,
                                                       E* __restrict__ out, int check, ixg_status* st,
                                                       int stmt, int site) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long c = __ldcs(&idx[i]);
    if (check) {
      if ((unsigned long long)c >= (unsigned long long)len) {
        status_fail(st, IXG_OOB, stmt, i, site);
        out[i] = E(0);
        continue;
      }
    }
    out[i] = __ldg(&arr[c]);
  }
}

// CSR flat gather, corpus/c4_csr_gather.ixl: out[i] = values[i] * x[indices[i]].
// 4 elements per thread-iteration: values/out as 16-byte vectors (i32),
// indices as two 16-byte vectors; x (4 MB at C4) stays in L2.
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_csr_gather(const E* __restrict__ x, long long num_cols,
                                                           const E* __restrict__ values,
                                                           const long long* __restrict__ indices,
                                                           long long nnz, E* __restrict__ out, int check,
                                                           ixg_status* st) {
  constexpr int V = 16 / (int)sizeof(E);
  const long long nv = nnz / V;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool narrow = false;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nv; k += stride) {
    E v[V], o[V];
    Vec<E>::unpack(ld_stream_v4(values + k * V), v);
    long long c[V];
#pragma unroll
    for (int h = 0; h < V / 2; ++h) {
      int64_t cc[2];
      Vec<int64_t>::unpack(ld_stream_v4(indices + k * V + 2 * h), cc);
      c[2 * h] = cc[0];
      c[2 * h + 1] = cc[1];
    }
#pragma unroll
    for (int e = 0; e < V; ++e) {
      if (check && (unsigned long long)c[e] >= (unsigned long long)num_cols) {
        status_fail(st, IXG_OOB, 0, k * V + e, 0);
        o[e] = E(0);
        continue;
      }
      long long prod;
      if constexpr (sizeof(E) == 8) {  // int64 x int64: checked (int32 x int32 always fits)
        if (mul_ovf((long long)v[e], (long long)__ldg(&x[c[e]]), &prod)) status_overflow(st, 0, k * V + e);
      } else {
        prod = (long long)v[e] * (long long)__ldg(&x[c[e]]);
      }
      if (sizeof(E) == 4 && prod != (long long)(int)prod) narrow = true;
      o[e] = (E)prod;
    }
    st_stream_v4(out + k * V, Vec<E>::pack(o));
  }
  if (blockIdx.x == 0) {
    for (long long i = nv * V + threadIdx.x; i < nnz; i += blockDim.x) {
      const long long c = indices[i];
      if (check && (unsigned long long)c >= (unsigned long long)num_cols) {
        status_fail(st, IXG_OOB, 0, i, 0);
        out[i] = E(0);
        continue;
      }
      long long prod;
      if constexpr (sizeof(E) == 8) {
        if (mul_ovf((long long)values[i], (long long)x[c], &prod)) status_overflow(st, 0, i);
      } else {
        prod = (long long)values[i] * (long long)x[c];
      }
      if (sizeof(E) == 4 && prod != (long long)(int)prod) narrow = true;
      out[i] = (E)prod;
    }
  }
  if (narrow && st) atomicOr(&st->flags, IXG_F_NARROW);
}

// get_smallest_pairs' map (maxmatching.ixl:18): cs[i] = H[es[i]] == is[i]
__global__ void __launch_bounds__(kGThreads) k_eq_gather(const long long* __restrict__ H, long long hlen,
                                                          const long long* __restrict__ es,
                                                          const long long* __restrict__ is, long long n,
                                                          uint8_t* __restrict__ cs, int check, ixg_status* st,
                                                          int stmt) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const long long e = es[i];
    if (check && (unsigned long long)e >= (unsigned long long)hlen) {
      status_fail(st, IXG_OOB, stmt, i, 0);
      cs[i] = 0;
      continue;
    }
    cs[i] = H[e] == is[i];
  }
}

// ---------------------------------------------------------------- reduce
// sum of xs into *out (int64, zeroed by the caller): 16-byte loads, warp
// shuffles, one atomic per warp (integer: order-independent, exact)
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_reduce_add(const E* __restrict__ xs, long long n,
                                                          unsigned long long* __restrict__ out) {
  constexpr int V = 16 / (int)sizeof(E);
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long s = 0;
  const bool vec = (((uintptr_t)xs) & 15) == 0;
  const long long nv = vec ? n / V : 0;
  for (long long k = tid; k < nv; k += stride) {
    const int4 v = ld_stream_v4(xs + k * V);
    const E* e = reinterpret_cast<const E*>(&v);
#pragma unroll
    for (int q = 0; q < V; ++q) s += (long long)e[q];
  }
  for (long long i = nv * V + tid; i < n; i += stride) s += (long long)xs[i];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if (lane_id() == 0 && s != 0) atomicAdd(out, (unsigned long long)s);
}

// ---------------------------------------------------------------- jagged
// partition2L's destinations (corpus/partition2l.ixl:41) for a jagged array
// whose row starts are the set bits of `bits` (mkFlags over n positions,
// sum shp == n): tb = the segmented inclusive count of cs per row.  A true
// element goes to its row start + the trues before it in its row, a false
// one to its own index + the trues after it in its row.
// Row start / end come from the nearest set bits (rows average tens of
// elements: a word or two of the bitmap).
__global__ void __launch_bounds__(kGThreads) k_jagged_dest(const uint32_t* __restrict__ bits, long long n,
                                                           const uint8_t* __restrict__ cs,
                                                           const long long* __restrict__ tb,
                                                           long long* __restrict__ dest) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    long long w = i >> 5;
    uint32_t m = bits[w] & (0xffffffffu >> (31 - (int)(i & 31)));  // starts <= i
    while (m == 0) m = bits[--w];  // position 0 starts the first non-empty row
    const long long rs = (w << 5) + (31 - __clz(m));
    long long re = n;  // one past the row's last element: the next start, or n
    const long long j = i + 1;
    if (j < n) {
      long long w2 = j >> 5;
      uint32_t m2 = bits[w2] & (0xffffffffu << (int)(j & 31));
      while (m2 == 0 && ((w2 + 1) << 5) < n) m2 = bits[++w2];
      if (m2) re = (w2 << 5) + (__ffs(m2) - 1);
      if (re > n) re = n;
    }
    const long long t = tb[i];
    dest[i] = cs[i] ? rs + t - 1 : i + (tb[re - 1] - t);
  }
}

// ---------------------------------------------------------------- hist
// (+): every bin is a 128-bit integer (hi:lo) -- lo = out[d], updated with
// one 64-bit atomicAdd whose returned old value gives the carry; the high
// word (hi[d], in the workspace) moves only when the carry and the sign
// extension of v do not cancel.  The bin's exact sum fits int64 iff hi is
// the sign extension of lo (k_hist_check).
__global__ void __launch_bounds__(kGThreads) k_hist(int op, long long dlen, const long long* __restrict__ is,
                                                     const long long* __restrict__ vs, long long m,
                                                     long long* __restrict__ out, long long* __restrict__ hi) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const long long d = is[i];
    if ((unsigned long long)d >= (unsigned long long)dlen) continue;  // oracle.py:314
    const long long v = vs[i];
    if (op == IXG_HIST_MIN) atomicMin(&out[d], v);
    else if (op == IXG_HIST_MAX) atomicMax(&out[d], v);
    else {
      const unsigned long long old = atomicAdd(reinterpret_cast<unsigned long long*>(&out[d]), (unsigned long long)v);
      const long long c = (v < 0 ? -1LL : 0LL) + ((old + (unsigned long long)v < old) ? 1LL : 0LL);
      if (c) atomicAdd(reinterpret_cast<unsigned long long*>(&hi[d]), (unsigned long long)c);
    }
  }
}

__global__ void __launch_bounds__(kGThreads) k_hist_check(const long long* __restrict__ out,
                                                           const long long* __restrict__ hi, long long dlen,
                                                           ixg_status* st) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long d = (long long)blockIdx.x * blockDim.x + threadIdx.x; d < dlen; d += stride)
    if (hi[d] != (out[d] >> 63)) status_overflow(st, 0, d);
}

// the words of a flag bitmap over *d_nbits positions (+ the readers' slack)
__global__ void __launch_bounds__(kGThreads) k_bitmap_clear(uint32_t* __restrict__ bits,
                                                             const long long* __restrict__ d_nbits) {
  const long long words = (*d_nbits + 31) / 32 + 2 + 512;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) bits[w] = 0u;
}

// the mkFlags bitmap's clear as the head of C2's programmatic-launch chain
// (clear -> mkFlags scan -> fused filter + sgmSum): words [0, words) (or the
// words of *d_nbits + the look-back slack) in 16-byte stores; the mkFlags
// scan starts at once and waits for this grid only before it sets bits
__global__ void __launch_bounds__(kGThreads) k_bitmap_zero(uint32_t* __restrict__ bits, long long words,
                                                            const long long* __restrict__ d_nbits) {
  pdl_trigger();
  if (d_nbits) words = (*d_nbits + 31) / 32 + 2 + 512;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long nv = words / 4;  // bits is 16-byte aligned
  for (long long k = tid; k < nv; k += stride) reinterpret_cast<int4*>(bits)[k] = make_int4(0, 0, 0, 0);
  for (long long w = nv * 4 + tid; w < words; w += stride) bits[w] = 0u;
}

// ---------------------------------------------------------------- fill / iota
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_fill(E* __restrict__ out, long long n,
                                                     const long long* __restrict__ d_n, E v) {
  if (d_n) n = *d_n;
  constexpr int V = 16 / (int)sizeof(E);
  const long long stride = (long long)gridDim.x * blockDim.x;
  E vv[V];
#pragma unroll
  for (int e = 0; e < V; ++e) vv[e] = v;
  const int4 pk = *reinterpret_cast<int4*>(vv);
  const long long nv = n / V;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nv; k += stride)
    st_stream_v4(out + k * V, pk);
  if (blockIdx.x == 0)
    for (long long i = nv * V + threadIdx.x; i < n; i += blockDim.x) out[i] = v;
}

__global__ void __launch_bounds__(kGThreads) k_iota(long long* __restrict__ out, long long n) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) out[i] = i;
}

// ---------------------------------------------------------------- kmeans_ker
// corpus/kmeans_ker.ixl, one thread per requested row; the for-loop runs in
// the reference's order with one rounding per operation (no FMA contraction).
__global__ void __launch_bounds__(128) k_kmeans(const long long* __restrict__ rows, long long nrows,
                                                 const long long* __restrict__ ptr, long long np1,
                                                 const double* __restrict__ cluster, long long num_cols,
                                                 const double* __restrict__ values,
                                                 const long long* __restrict__ indices, long long nnz,
                                                 double* __restrict__ out, uint32_t variant, ixg_status* st) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const long long row = rows[r];
  auto chk = [&](int site) { return (IXG_SITE_BITS(variant, site) & IXG_V_BOUNDS) != 0; };
  // stmt = r: rows are independent calls, ordered by request index
  if (chk(0) && (unsigned long long)row >= (unsigned long long)np1) {
    status_fail(st, IXG_OOB, 0, r, 0);
    return;
  }
  const long long start = ptr[row];
  if (chk(1) && (unsigned long long)(row + 1) >= (unsigned long long)np1) {
    status_fail(st, IXG_OOB, 0, r, 1);
    return;
  }
  const long long cnt = ptr[row + 1] - start;
  double corr = 0.0;
  for (long long j = 0; j < cnt; ++j) {
    const long long a = start + j;
    if (chk(2) && (unsigned long long)a >= (unsigned long long)nnz) {
      status_fail(st, IXG_OOB, 0, r, 2);
      return;
    }
    const double ev = values[a];
    if (chk(3) && (unsigned long long)a >= (unsigned long long)nnz) {
      status_fail(st, IXG_OOB, 0, r, 3);
      return;
    }
    const long long col = indices[a];
    if (chk(4) && (unsigned long long)col >= (unsigned long long)num_cols) {
      status_fail(st, IXG_OOB, 0, r, 4);
      return;
    }
    const double cv = cluster[col];
    const double diff = __dsub_rn(ev, __dmul_rn(2.0, cv));
    corr = __dadd_rn(corr, __dmul_rn(diff, ev));
  }
  out[r] = corr;
}

// ---------------------------------------------------------------- generator
// out[i] = lo + rand(seed, offset + i) mod (hi - lo + 1)   (ixo_rand)
template <typename E>
__global__ void __launch_bounds__(kGThreads) k_gen_uniform(E* __restrict__ out, long long n, long long lo,
                                                            unsigned long long span, uint64_t smix,
                                                            long long offset) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t u = rand_at(smix, (uint64_t)(offset + i));
    out[i] = (E)(span ? (long long)((unsigned long long)lo + u % span) : (long long)u);
  }
}

}  // namespace ixg
