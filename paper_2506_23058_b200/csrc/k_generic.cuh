// k_generic.cuh -- the builtins one kernel each (scan, segmented scan,
// scatter with/without the idempotence check, gather with/without bounds
// checks, hist, replicate, iota) and the CHECKED forms of the corpus
// pipelines, which materialise their index arrays exactly as the reference
// program does (the dynamic check needs the index array).
#pragma once
#include <type_traits>

#include "lookback.cuh"

namespace ixg {

constexpr int kGThreads = 256;
constexpr int kGItems = 16;
constexpr int kGTile = kGThreads * kGItems;

// ---------------------------------------------------------------- sources
template <typename E>
IXG_DEV long long load_as_i64(const void* p, long long i) {
  return (long long)reinterpret_cast<const E*>(p)[i];
}
IXG_DEV long long load_dt(int dt, const void* p, long long i) {
  switch (dt) {
    case IXG_I32: return load_as_i64<int32_t>(p, i);
    case IXG_U8: return load_as_i64<uint8_t>(p, i);
    default: return load_as_i64<int64_t>(p, i);
  }
}
IXG_DEV void store_dt(int dt, void* p, long long i, long long v) {
  if (dt == IXG_I32) reinterpret_cast<int32_t*>(p)[i] = (int32_t)v;
  else if (dt == IXG_U8) reinterpret_cast<uint8_t*>(p)[i] = (uint8_t)v;
  else reinterpret_cast<int64_t*>(p)[i] = v;
}

struct SrcArr {  // scan (+) over an integer array (any element width)
  int dt;
  const void* xs;
  IXG_DEV SumOp::T operator()(long long i) const { return SumOp::T{load_dt(dt, xs, i)}; }
};
template <typename E>
struct SrcArrT {  // scan (+) over E[], 16 elements per thread through 256-bit loads
  const E* xs;
  IXG_DEV SumOp::T operator()(long long i) const { return SumOp::T{(long long)xs[i]}; }
  IXG_DEV void load16(long long i0, long long n, SumOp::T (&v)[kGItems]) const {
    if (sizeof(E) >= 2 && i0 + kGItems <= n && (((uintptr_t)(xs + i0)) & 31) == 0) {
      constexpr int PER = 32 / (int)sizeof(E);
#pragma unroll
      for (int k = 0; k < kGItems / PER; ++k) {
        uint32_t r[8];
        asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                       "=r"(r[7])
                     : "l"(xs + i0 + k * PER));
        const E* e = reinterpret_cast<const E*>(r);
#pragma unroll
        for (int q = 0; q < PER; ++q) v[k * PER + q] = SumOp::T{(long long)e[q]};
      }
    } else {
#pragma unroll
      for (int j = 0; j < kGItems; ++j) v[j] = SumOp::T{(i0 + j < n) ? (long long)xs[i0 + j] : 0};
    }
  }
};
struct SrcPred {  // map (\x -> if p x then 1 else 0) xs, fused into the scan
  int dt;
  const void* xs;
  const uint8_t* cs;  // filter_by: the bool array instead of p
  ixg_pred p;
  IXG_DEV SumOp::T operator()(long long i) const {
    if (cs) return SumOp::T{cs[i] != 0};
    return SumOp::T{pred_eval(p, load_dt(dt, xs, i)) ? 1 : 0};
  }
};
struct SrcClass3 {  // partition3: (flags1, flags2)
  int dt;
  const void* xs;
  ixg_pred p, q;
  IXG_DEV Sum2Op::T operator()(long long i) const {
    const long long x = load_dt(dt, xs, i);
    const bool c1 = pred_eval(p, x);
    const bool c2 = !c1 && pred_eval(q, x);
    return Sum2Op::T{c1 ? 1 : 0, c2 ? 1 : 0};
  }
};
struct SrcSeg {  // (flags, xs) of the segmented scan
  int dt_f, dt_x;
  const void* flags;
  const void* xs;
  IXG_DEV SegOp::T operator()(long long i) const {
    return SegOp::T{load_dt(dt_x, xs, i), load_dt(dt_f, flags, i) != 0};
  }
};

// ---------------------------------------------------------------- epilogues
struct EpiScanOut {  // out[i] = ne + inclusive (or exclusive) sum
  long long ne;
  int exclusive;
  long long* out;
  IXG_DEV void operator()(long long i, SumOp::T incl, SumOp::T x) const {
    out[i] = ne + (exclusive ? incl.v - x.v : incl.v);
  }
};
struct EpiFilterInds {  // filter.ixl:10-12: inds[i] = if c then offs[i]-1 else -1; count = offs[n-1]
  long long n;
  long long* inds;
  long long* d_count;
  IXG_DEV void operator()(long long i, SumOp::T incl, SumOp::T x) const {
    inds[i] = x.v ? incl.v - 1 : -1;
    if (i == n - 1) *d_count = incl.v;
  }
};
struct EpiPart2Inds {  // partition2.ixl:11-16 with num_true from the count pass
  const long long* d_nt;
  long long* inds;
  IXG_DEV void operator()(long long i, SumOp::T incl, SumOp::T x) const {
    const long long t = incl.v;             // indicesT[i]
    const long long f = (i + 1 - t) + *d_nt;  // indicesF[i] = tmp[i] + num_true
    inds[i] = x.v ? t - 1 : f - 1;
  }
};
struct EpiPart3Inds {  // partition3.ixl:14-24 with (m1, m2) from the count pass
  const long long* d_m;
  long long* inds;
  IXG_DEV void operator()(long long i, Sum2Op::T incl, Sum2Op::T x) const {
    const long long m1 = d_m[0], m2 = d_m[1];
    const long long inds1 = incl.a - 1, inds2 = m1 + incl.b - 1;
    const long long inds3 = m1 + m2 + i - (incl.a + incl.b);
    inds[i] = x.a ? inds1 : (x.b ? inds2 : inds3);
  }
};
struct EpiSegOut {  // sgmSum value (and flag) components
  int dt_out;
  void* out_v;
  uint8_t* out_f;
  ixg_status* st;
  IXG_DEV void operator()(long long i, SegOp::T incl, SegOp::T) const {
    if (dt_out == IXG_I32) {
      if (incl.v != (long long)(int)incl.v && st) atomicOr(&st->flags, IXG_F_NARROW);
      reinterpret_cast<int32_t*>(out_v)[i] = (int32_t)incl.v;
    } else {
      reinterpret_cast<int64_t*>(out_v)[i] = incl.v;
    }
    if (out_f) out_f[i] = (uint8_t)incl.f;
  }
};
struct EpiSegStarts {  // mkSgmDescr / mkFlags: ind[i] = if shape[i] <= 0 then -1 else scn[i]
  long long m;
  const long long* shape;
  long long* ind;        // nullable
  uint32_t* bits;        // nullable: set bit scn[i] (flag array as a bitmap)
  long long nbits;
  long long* d_total;    // nullable: scn[m-1] + shape[m-1]
  IXG_DEV void operator()(long long i, SumOp::T incl, SumOp::T x) const {
    const long long s = x.v, start = incl.v - s;
    if (ind) ind[i] = s <= 0 ? -1 : start;
    if (bits && s > 0 && start >= 0 && start < nbits) atomicOr(&bits[start >> 5], 1u << (start & 31));
    if (d_total && i == m - 1) *d_total = incl.v;
  }
};

// Single-pass blocked scan with a source functor and an epilogue functor.
// tile = blockIdx.x (see lookback.cuh / k_stream.cuh for the protocol); a
// source may provide load16() with 256-bit loads of its 16 elements.
template <class Src, class T>
IXG_DEV auto src_load16(const Src& src, long long i0, long long n, T (&v)[kGItems], int)
    -> decltype(src.load16(i0, n, v), void()) {
  src.load16(i0, n, v);
}
template <class Src, class T>
IXG_DEV void src_load16(const Src& src, long long i0, long long n, T (&v)[kGItems], long) {
#pragma unroll
  for (int j = 0; j < kGItems; ++j) v[j] = (i0 + j < n) ? src(i0 + j) : T{};
}

template <class M, class Src, class Epi>
__global__ void __launch_bounds__(kGThreads) k_scan(long long n, Src src, Epi epi, LBChan ch, uint32_t nonce) {
  using T = typename M::T;
  __shared__ T s_w[kGThreads / 32];
  __shared__ T s_carry;
  const long long tile = blockIdx.x;
  const long long i0 = tile * kGTile + (long long)threadIdx.x * kGItems;
  T v[kGItems];
  src_load16(src, i0, n, v, 0);
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
  T run = M::op(M::op(s_carry, wpre), lex);
#pragma unroll
  for (int j = 0; j < kGItems; ++j) {
    if (i0 + j < n) {
      run = M::op(run, v[j]);
      epi(i0 + j, run, v[j]);
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
      const long long prod = (long long)v[e] * (long long)__ldg(&x[c[e]]);
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
      const long long prod = (long long)values[i] * (long long)x[c];
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
__global__ void __launch_bounds__(kGThreads) k_hist(int op, long long dlen, const long long* __restrict__ is,
                                                     const long long* __restrict__ vs, long long m,
                                                     long long* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const long long d = is[i];
    if ((unsigned long long)d >= (unsigned long long)dlen) continue;  // oracle.py:314
    const long long v = vs[i];
    if (op == IXG_HIST_MIN) atomicMin(&out[d], v);
    else if (op == IXG_HIST_MAX) atomicMax(&out[d], v);
    else atomicAdd(reinterpret_cast<unsigned long long*>(&out[d]), (unsigned long long)v);
  }
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
