// k_stream.cuh -- single-pass stream compaction for sm_100a: filter /
// filter_by (+ the flag-array segmented sum of BASELINE C2) and the stable
// 2-/3-way partition placement.
//
// Why these can be fused at all: the verifier proved the final scatter of
// each program safe AND bijective onto its destination (Sc1, SURVEY.md App. B:
// filter (14,12), partition2 (18,12), partition3 (26,12)), so the destination
// needs no initialisation, no OOB test and no duplicate check, and every
// element's destination is determined by the running count alone.  The
// scatter collapses into a stable compaction inside the scan tile: xs is read
// once, ys (and zs) written once.
//
// Shape of the kernels (chosen by measurement):
//   * one CTA per tile of NT x 16 elements, tile = blockIdx.x (CTAs are
//     dispatched in index order, so a CTA only waits on tiles already
//     resident or done -- the forward-progress argument CUB's single-pass
//     scan relies on); no ticket/retire atomics, and the look-back slots are
//     tagged with a per-launch nonce from the host so the workspace never
//     needs a reset.  A persistent ticket-driven variant with register
//     prefetch measured 2-3x slower (all CTAs reach their look-back in
//     lock-step).  The look-back resolves ~32 tiles per L2 round trip, so
//     throughput scales with the tile size: NT = 512 (8192 elements).
//   * blocked layout: 16 consecutive elements per thread via 256-bit loads
//     (LDG.E.256); a thread's selected elements are consecutive in the
//     output, so ranks are one popc + a warp/CTA prefix of per-thread counts
//     and the segmented sum of C2 is a per-thread fold plus one warp scan.
//   * the compacted run is staged in shared memory at its global 32-byte
//     phase and written with aligned 256-bit stores (scalar only at the two
//     run ends).
//   * C2 needs only the count look-back: the segmented sum is computed with a
//     tile-local carry and each tile's aggregate is written out; a fix-up
//     pass (k_seg_tile_scan + k_seg_fixup) adds the carry of the preceding
//     tiles to the tile's output prefix before its first segment start
//     (segments average 128 elements at C2: a few % of zs).
#pragma once
#include <type_traits>

#include "lookback.cuh"

namespace ixg {

constexpr int kSThreads = 256;  // non-tiled helper kernels
constexpr int kSItems = 16;
constexpr int kSWarps = kSThreads / 32;
#ifndef IXG_STREAM_THREADS
#define IXG_STREAM_THREADS 512
#endif
constexpr int kNT = IXG_STREAM_THREADS;  // threads of the compaction kernels
constexpr int kSTile = kNT * kSItems;    // elements per tile

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

// 16 consecutive elements of type T per thread
template <typename T>
struct Blk16 {
  T x[kSItems];
  IXG_DEV void load(const T* __restrict__ xs, long long i0, long long n) {
    if (i0 + kSItems <= n) {
      constexpr int NV = kSItems * (int)sizeof(T) / 32;  // 256-bit loads
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        uint32_t r[8];
        ld256(xs + i0 + v * (32 / (int)sizeof(T)), r);
#pragma unroll
        for (int e = 0; e < 32 / (int)sizeof(T); ++e) {
          if constexpr (sizeof(T) == 4) x[v * 8 + e] = (T)r[e];
          else x[v * 4 + e] = (T)(((unsigned long long)r[2 * e + 1] << 32) | r[2 * e]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < kSItems; ++j) x[j] = (i0 + j < n) ? xs[i0 + j] : T(0);
    }
  }
};

IXG_DEV uint32_t valid_mask(long long i0, long long n) {
  const long long valid = n - i0;
  return valid <= 0 ? 0u : (valid >= kSItems ? 0xffffu : ((1u << valid) - 1u));
}

// The predicate of a kernel, decoded once per thread: the comparison kinds
// become an interval test (common.cuh PredRange), HASH keeps its seed.
template <typename T>
struct Selector {
  int kind;  // IXG_PRED_LT..NE -> range test
  PredRange<T> r;
  uint64_t seed;
  IXG_DEV explicit Selector(const ixg_pred& p) : kind(p.kind), r(pred_range<T>(p)), seed(p.seed) {}
  // selection mask of 16 elements; the kind is uniform, so no divergence
  IXG_DEV uint32_t mask(const T (&x)[kSItems]) const {
    uint32_t m = 0;
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

// CTA-wide exclusive prefix of per-thread counts; returns the thread's
// exclusive prefix, *total = the CTA total.  Contains one named barrier (id 1) over the NT worker threads.
template <int NT>
IXG_DEV int cta_exclusive(int c, int* s_w, int* total) {
  const int lane = lane_id(), w = warp_id();
  int inc = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += o;
  }
  if (lane == 31) s_w[w] = inc;
  bar_sync(1, NT);
  int pre = 0, tot = 0;
#pragma unroll
  for (int k = 0; k < NT / 32; ++k) {
    const int v = s_w[k];
    pre += (k < w) ? v : 0;
    tot += v;
  }
  *total = tot;
  return pre + inc - c;
}

// store the run staged at stage[shift .. shift+cnt) (shift = base % VS, i.e.
// stage index = (g - base) + shift for global position g) to out[base ..]
template <typename E, int NT>
IXG_DEV void store_aligned(E* __restrict__ out, long long base, int cnt, const E* stage) {
  constexpr int VS = 32 / (int)sizeof(E);
  if (cnt <= 0) return;
  const long long c0 = base / VS, c1 = (base + cnt - 1) / VS;
  const int shift = (int)(base - c0 * VS);
  for (long long c = c0 + threadIdx.x; c <= c1; c += NT) {
    const int q0 = (int)(c - c0) * VS;
    const long long g0 = c * VS;
    if (g0 >= base && g0 + VS <= base + cnt) {
      uint32_t r[8];
      const uint4 a = *reinterpret_cast<const uint4*>(stage + q0);
      const uint4 b = *reinterpret_cast<const uint4*>(stage + q0 + VS / 2);
      r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
      r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
      st256(out + g0, r);
    } else {
#pragma unroll
      for (int e = 0; e < VS; ++e) {
        const int q = q0 + e;
        if (q >= shift && q < shift + cnt) out[g0 + e] = stage[q];
      }
    }
  }
}

// Per-tile output of the segmented fused kernel, for the fix-up pass.
struct SegTileMeta {
  long long v;     // tile aggregate value; after k_seg_tile_scan: the carry INTO the tile
  long long f;     // tile has a flag
  long long base;  // first output position of the tile
  long long cnt;   // outputs of the tile
};

// ---------------------------------------------------------------------------
// filter / filter_by [+ sgmSum over the output with flags from a bitmap]
template <typename T, typename Z, bool kByCs, bool kSeg>
__global__ void __launch_bounds__(kNT + 32, 2) k_filter_s(const T* __restrict__ xs, const uint8_t* __restrict__ cs,
                                                           long long n, ixg_pred p, T* __restrict__ ys,
                                                           Z* __restrict__ zs, const uint32_t* __restrict__ segbits,
                                                           long long out_base, LBChan ch, uint32_t nonce,
                                                           long long* d_count, SegTileMeta* __restrict__ meta,
                                                           ixg_status* st) {
  constexpr int NT = kNT;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int VS = 32 / (int)sizeof(T);
  constexpr int VZ = 32 / (int)sizeof(Z);
  T* stage = reinterpret_cast<T*>(smem_raw);
  Z* stage_z = reinterpret_cast<Z*>(smem_raw + (kSTile + VS) * sizeof(T));
  __shared__ int s_w[NT / 32];
  __shared__ int s_cnt;
  __shared__ long long s_excl;
  __shared__ SegOp::T s_seg[NT / 32];

  const long long tile = blockIdx.x;
  if (warp_id() == NT / 32) {
    // look-back warp: resolves the tile's exclusive prefix while the worker
    // warps' loads are in flight (it needs only the predecessors' slots)
    long long ex = 0;
    if (tile > 0) ex = lb_lookback<SumOp>(ch, nonce, tile).v;
    if (lane_id() == 0) s_excl = ex;
    IXG_TR_LANE0(3);
    bar_sync(2, NT + 32);  // the workers have published the aggregate
    if (lane_id() == 0) {
      const int cnt = s_cnt;
      if (tile > 0) lb_publish<SumOp>(ch, nonce, tile, SumOp::T{ex + cnt}, true);
      if (tile == (long long)gridDim.x - 1) *d_count = ex + cnt;
    }
    return;
  }
  const long long i0 = tile * kSTile + threadIdx.x * kSItems;
  Blk16<T> cur;
  IXG_TR(0);
  cur.load(xs, i0, n);
  uint32_t mask;
  if (kByCs) {
    mask = 0;
#pragma unroll
    for (int j = 0; j < kSItems; ++j) mask |= (uint32_t)((i0 + j < n) && cs[i0 + j] != 0) << j;
  } else {
    mask = select_mask<T>(p, cur.x) & valid_mask(i0, n);
  }
  const int c = __popc(mask);
  IXG_TR(1);
  int cnt;
  const int rank = cta_exclusive<NT>(c, s_w, &cnt);
  IXG_TR(2);
  if (threadIdx.x == 0) {
    s_cnt = cnt;
    lb_publish<SumOp>(ch, nonce, tile, SumOp::T{cnt}, tile == 0);
  }
  bar_sync(2, NT + 32);
  IXG_TR(4);
  const long long base = s_excl;
  const int shift = (int)(base % VS);
  int idx = shift + rank;
#pragma unroll
  for (int j = 0; j < kSItems; ++j) {
    if ((mask >> j) & 1u) stage[idx] = cur.x[j];
    idx += (mask >> j) & 1u;
  }
  if (kSeg) {
    // Flags of the thread's c output positions [pos0, pos0 + c) are bits of
    // the mkFlags bitmap (L2-resident).  Their load depends on `base`, so it
    // is issued first and the ys run is written while it is in flight.
    const long long pos0 = out_base + base + rank;
    const long long wd = pos0 >> 5;
    uint32_t bw0 = 0, bw1 = 0;
    if (c) {
      bw0 = __ldg(&segbits[wd]);
      bw1 = __ldg(&segbits[wd + 1]);
    }
    bar_sync(1, NT);
    IXG_TR(5);
    store_aligned<T, NT>(ys, base, cnt, stage);
    uint32_t fb = (uint32_t)((((uint64_t)bw1 << 32) | (uint64_t)bw0) >> (pos0 & 31));
    fb &= (c >= 32) ? 0xffffffffu : ((1u << c) - 1u);
    // segments average ~128 outputs, so a thread rarely holds a segment
    // start: expand the (sparse) flag bits to input slots
    uint32_t fm = 0;
    while (fb) {
      const int b = __ffs(fb) - 1;
      fb &= fb - 1;
      fm |= 1u << __fns(mask, 0, b + 1);
    }
    // thread aggregate: (has flag, sum of the selected values from its last flag on)
    const uint32_t tail = fm ? (mask & ~((1u << (31 - __clz(fm))) - 1u)) : mask;
    long long s64;
    if constexpr (sizeof(T) == 4) {
      int s32 = 0, ovf = 0;
#pragma unroll
      for (int j = 0; j < kSItems; ++j) {
        const int xv = ((tail >> j) & 1u) ? (int)cur.x[j] : 0;
        const int r = s32 + xv;
        ovf |= (s32 ^ r) & (xv ^ r);
        s32 = r;
      }
      if (ovf < 0) {  // rare: redo in 64 bits
        s64 = 0;
#pragma unroll
        for (int j = 0; j < kSItems; ++j) s64 += ((tail >> j) & 1u) ? (long long)cur.x[j] : 0LL;
      } else {
        s64 = s32;
      }
    } else {
      s64 = 0;
#pragma unroll
      for (int j = 0; j < kSItems; ++j) s64 += ((tail >> j) & 1u) ? (long long)cur.x[j] : 0LL;
    }
    const SegOp::T a{s64, fm != 0};
    SegOp::T inc = warp_inclusive<SegOp>(a);
    SegOp::T lex = SegOp::shfl_up(inc, 1);
    if (lane_id() == 0) lex = SegOp::identity();
    if (lane_id() == 31) s_seg[warp_id()] = inc;
    bar_sync(1, NT);
    SegOp::T pre = SegOp::identity(), tagg = SegOp::identity();
#pragma unroll
    for (int w = 0; w < NT / 32; ++w) {
      if (w < warp_id()) pre = SegOp::op(pre, s_seg[w]);
      tagg = SegOp::op(tagg, s_seg[w]);
    }
    const long long start = SegOp::op(pre, lex).v;
    const int iz0 = (int)(base % VZ) + rank;
    bool narrow = false;
    if constexpr (sizeof(T) == 4 && sizeof(Z) == 4) {
      // every run value is a zs value, so 32-bit arithmetic with an
      // overflow check is exact whenever zs fits its int32 storage
      int run = (int)start, ovf = 0, iz = iz0;
      narrow = start != (long long)run;
#pragma unroll
      for (int j = 0; j < kSItems; ++j) {
        const uint32_t sel = (mask >> j) & 1u;
        const int b = ((fm >> j) & 1u) ? 0 : run;
        const int r = b + (int)cur.x[j];
        if (sel) {
          ovf |= (b ^ r) & ((int)cur.x[j] ^ r);
          run = r;
          stage_z[iz] = (Z)r;
        }
        iz += sel;
      }
      narrow |= ovf < 0;
    } else {
      long long run = start, hi = 0;
      int iz = iz0;
#pragma unroll
      for (int j = 0; j < kSItems; ++j) {
        const uint32_t sel = (mask >> j) & 1u;
        const long long nv = (((fm >> j) & 1u) ? 0LL : run) + (long long)cur.x[j];
        run = sel ? nv : run;
        if (sel) stage_z[iz] = (Z)run;
        iz += sel;
        if (sizeof(Z) == 4) hi |= (run >> 31) ^ (run >> 63);  // nonzero iff run leaves int32
      }
      narrow = hi != 0;
    }
    if (narrow && st) atomicOr(&st->flags, IXG_F_NARROW);
    if (threadIdx.x == 0) meta[tile] = SegTileMeta{tagg.v, (long long)tagg.f, base, (long long)cnt};
    bar_sync(1, NT);
    store_aligned<Z, NT>(zs, base, cnt, stage_z);
    IXG_TR(6);
  } else {
    bar_sync(1, NT);
    IXG_TR(5);
    store_aligned<T, NT>(ys, base, cnt, stage);
    IXG_TR(6);
  }
}

// ---------------------------------------------------------------------------
// partition2 / partition3: class counts (pass 1), stable placement (pass 2).
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

// Pass 2: placement.  Class c of a tile is one contiguous run of the output
// at (totals of the classes before c) + (class-c elements in earlier
// tiles), and a thread's class-c elements are consecutive inside it.  The
// look-back carries the class-0 (and class-1) prefix; the last class's
// prefix is the tile start minus the others.
template <typename T, int kClasses>
__global__ void __launch_bounds__(kNT + 32, 2) k_place_s(const T* __restrict__ xs, long long n, ixg_pred p,
                                                          ixg_pred q, T* __restrict__ ys,
                                                          const long long* __restrict__ d_tot, LBChan ch,
                                                          uint32_t nonce) {
  constexpr int NT = kNT;
  using M = typename std::conditional<kClasses == 2, SumOp, Sum2Op>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int VS = 32 / (int)sizeof(T);
  constexpr int SLOT = kSTile + VS;
  T* stage0 = reinterpret_cast<T*>(smem_raw);
  T* stage_last = stage0 + SLOT;
  T* stage1 = stage_last + SLOT;  // partition3 only
  __shared__ int s_w[NT / 32];
  __shared__ int s_w1[NT / 32];
  __shared__ long long s_ex[2];
  __shared__ typename std::conditional<kClasses == 2, SumOp, Sum2Op>::type::T s_agg;

  const long long tile = blockIdx.x;
  if (warp_id() == NT / 32) {  // look-back warp (see k_filter_s)
    typename M::T ex = M::identity();
    if (tile > 0) ex = lb_lookback<M>(ch, nonce, tile);
    if (lane_id() == 0) {
      if constexpr (kClasses == 2) {
        s_ex[0] = ex.v;
        s_ex[1] = 0;
      } else {
        s_ex[0] = ex.a;
        s_ex[1] = ex.b;
      }
    }
    bar_sync(2, NT + 32);
    if (lane_id() == 0 && tile > 0) lb_publish<M>(ch, nonce, tile, M::op(ex, s_agg), true);
    return;
  }
  const long long tile_base = tile * kSTile;
  const long long i0 = tile_base + threadIdx.x * kSItems;
  Blk16<T> cur;
  cur.load(xs, i0, n);
  const int tile_len = (int)min((long long)kSTile, n - tile_base);
  const int before = min((int)threadIdx.x * kSItems, tile_len);  // elements of earlier threads
  const uint32_t vm = valid_mask(i0, n);
  const uint32_t m0 = select_mask<T>(p, cur.x) & vm;
  uint32_t m1 = 0;
  if (kClasses == 3) m1 = select_mask<T>(q, cur.x) & vm & ~m0;
  const uint32_t m2 = vm & ~m0 & ~m1;
  int cnt0, cnt1 = 0;
  const int r0 = cta_exclusive<NT>(__popc(m0), s_w, &cnt0);
  int r1 = 0;
  if (kClasses == 3) r1 = cta_exclusive<NT>(__popc(m1), s_w1, &cnt1);
  const int r2 = before - r0 - r1;
  typename M::T agg;
  if constexpr (kClasses == 2) agg = typename M::T{cnt0};
  else agg = typename M::T{cnt0, cnt1};
  if (threadIdx.x == 0) {
    s_agg = agg;
    lb_publish<M>(ch, nonce, tile, agg, tile == 0);
  }
  bar_sync(2, NT + 32);
  const long long t0 = d_tot[0];
  const long long t1 = kClasses == 3 ? d_tot[1] : 0;
  const long long e0 = s_ex[0], e1 = s_ex[1];
  const long long e2 = tile_base - e0 - e1;
  const long long b0 = e0, b1 = t0 + e1, b2 = t0 + t1 + e2;
  int k0 = (int)(b0 % VS) + r0, k1 = (int)(b1 % VS) + r1, k2 = (int)(b2 % VS) + r2;
#pragma unroll
  for (int j = 0; j < kSItems; ++j) {
    const uint32_t s0 = (m0 >> j) & 1u, s1 = (m1 >> j) & 1u, s2 = (m2 >> j) & 1u;
    if (s0) stage0[k0] = cur.x[j];
    if (kClasses == 3 && s1) stage1[k1] = cur.x[j];
    if (s2) stage_last[k2] = cur.x[j];
    k0 += s0;
    k1 += s1;
    k2 += s2;
  }
  bar_sync(1, NT);
  const int cnt2 = tile_len - cnt0 - cnt1;
  store_aligned<T, NT>(ys, b0, cnt0, stage0);
  if (kClasses == 3) store_aligned<T, NT>(ys, b1, cnt1, stage1);
  store_aligned<T, NT>(ys, b2, cnt2, stage_last);
}

// ---------------------------------------------------------------------------
// C2 fix-up: carry of the preceding tiles (and of preceding shards, `carry0`)
// added to each tile's outputs before its first segment start.
// Pass 1 (one CTA): exclusive segmented scan over the tile aggregates.
__global__ void __launch_bounds__(1024) k_seg_tile_scan(SegTileMeta* __restrict__ meta, long long ntiles,
                                                        long long carry_v, int carry_f) {
  __shared__ SegOp::T s_w[32];
  __shared__ SegOp::T s_carry;
  if (threadIdx.x == 0) s_carry = SegOp::T{carry_v, carry_f};
  __syncthreads();
  for (long long b = 0; b < ntiles; b += blockDim.x) {
    const long long t = b + threadIdx.x;
    SegOp::T x = SegOp::identity();
    if (t < ntiles) x = SegOp::T{meta[t].v, (int)(meta[t].f & 1)};
    SegOp::T inc = warp_inclusive<SegOp>(x);
    if (lane_id() == 31) s_w[warp_id()] = inc;
    __syncthreads();
    SegOp::T pre = s_carry;
    for (int w = 0; w < warp_id(); ++w) pre = SegOp::op(pre, s_w[w]);
    SegOp::T lex = SegOp::shfl_up(inc, 1);
    if (lane_id() == 0) lex = SegOp::identity();
    const SegOp::T ex = SegOp::op(pre, lex);
    __syncthreads();
    if (t < ntiles) meta[t].v = ex.v;  // carry INTO tile t (value since the last flag)
    if (threadIdx.x == blockDim.x - 1) s_carry = SegOp::op(ex, x);
    __syncthreads();
  }
}

// Pass 2: zs[q] += carry(tile) for q in [base, first flag of the tile).
// meta.f bit 1 (set by k_filter_b<kSeg>): a tile-local prefix value before
// the first flag left Z's range, so zs there holds it modulo 2^32 and the
// exact value carry + sum ys[base..q] is range-checked from ys instead.
template <typename Z, typename T>
__global__ void __launch_bounds__(256) k_seg_fixup(const SegTileMeta* __restrict__ meta, long long ntiles,
                                                   const uint32_t* __restrict__ segbits, long long out_base,
                                                   Z* __restrict__ zs, const T* __restrict__ ys, ixg_status* st) {
  __shared__ long long s_stop;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const long long c = meta[t].v;
    const long long base = meta[t].base, cnt = meta[t].cnt;
    const bool lovf = (meta[t].f & 2) != 0;
    if ((c == 0 && !lovf) || cnt == 0) continue;  // uniform per CTA
    if (warp_id() == 0) {  // first set flag bit in [base, base + cnt)
      long long stop = base + cnt;
      for (long long q = base; q < base + cnt; q += 32 * 32) {
        const long long ql = q + lane_id() * 32;
        uint32_t w = 0;
        if (ql < base + cnt) {
          const long long g = out_base + ql;
          const long long wd = g >> 5;
          w = (uint32_t)((((uint64_t)segbits[wd + 1] << 32) | segbits[wd]) >> (g & 31));
          const long long lim = base + cnt - ql;
          if (lim < 32) w &= (1u << lim) - 1u;
        }
        const uint32_t any = __ballot_sync(0xffffffffu, w != 0);
        if (any) {
          const int l = __ffs(any) - 1;
          const uint32_t wl = __shfl_sync(0xffffffffu, w, l);
          stop = q + l * 32 + (__ffs(wl) - 1);
          break;
        }
      }
      if (lane_id() == 0) s_stop = stop;
    }
    __syncthreads();
    const long long stop = s_stop;
    bool narrow = false;
    if (lovf && warp_id() == 0) {  // rare: exact values from ys, one warp
      long long run = c;
      for (long long q = base; q < stop; q += 32) {
        const bool in = q + lane_id() < stop;
        long long x = in ? (long long)ys[q + lane_id()] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const long long o = __shfl_up_sync(0xffffffffu, x, d);
          if (lane_id() >= d) x += o;
        }
        if (in && run + x != (long long)(int)(run + x)) narrow = true;
        run += __shfl_sync(0xffffffffu, x, 31);
      }
    }
    for (long long q = base + threadIdx.x; q < stop; q += blockDim.x) {
      const long long v = (long long)zs[q] + c;
      if (sizeof(Z) == 4 && !lovf && v != (long long)(int)v) narrow = true;
      zs[q] = (Z)v;
    }
    if (narrow && st) atomicOr(&st->flags, IXG_F_NARROW);
    __syncthreads();
  }
}

}  // namespace ixg
