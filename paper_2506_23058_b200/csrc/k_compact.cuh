// k_compact.cuh -- the fused ELIDED pipelines: filter (+ flag-array
// segmented sum = BASELINE C2) and partition2/3 placement.
//
// Why these can be fused at all: the verifier proved the final scatter of
// each program safe AND bijective onto its destination (Sc1, SURVEY.md App. B:
// filter (14,12), partition2 (18,12), partition3 (26,12)), so the destination
// needs no initialisation, no OOB test and no duplicate check, and every
// element's destination is determined by the running count alone.  The
// scatter therefore collapses into a stable compaction inside the scan tile:
// xs is read once, ys (and zs) written once -- the compulsory traffic.
//
// Tile layout (kThreads x kItems = 4096 elements):
//   load:   warp-striped 128-bit loads (warp w, row r, lane l holds the
//           16-byte chunk at w*512 + r*32*V + l*V), ranks from warp ballots;
//   stage:  compacted elements in shared memory, chunk-XOR-swizzled so that
//           both the scattered rank writes and the blocked per-thread reads
//           of the segmented phase are bank-conflict free;
//   store:  16-byte aligned vector stores of the tile's output run(s), with
//           scalar stores only for the two partial chunks at the run ends.
#pragma once
#include <type_traits>

#include "lookback.cuh"

namespace ixg {

constexpr int kThreads = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // 4096
constexpr int kWarps = kThreads / 32;

// physical index of element q in a stage of element type E
template <typename E>
IXG_DEV int swz(int q) {
  constexpr int V = 16 / (int)sizeof(E);
  constexpr int CPT = kItems / V;
  const int c = q / V;
  const int pc = c ^ ((c / CPT) & 7);
  return pc * V + (q % V);
}

// Store stage[off .. off+cnt) (logical, swizzled) to out[base .. base+cnt).
template <typename E>
IXG_DEV void store_run(E* __restrict__ out, long long base, int cnt, const E* stage, int off) {
  constexpr int V = 16 / (int)sizeof(E);
  if (cnt <= 0) return;
  const long long c0 = base / V, c1 = (base + cnt - 1) / V;
  for (long long c = c0 + threadIdx.x; c <= c1; c += kThreads) {
    const long long g0 = c * V;
    if (g0 >= base && g0 + V <= base + cnt) {
      E tmp[V];
      const int q0 = off + (int)(g0 - base);
#pragma unroll
      for (int e = 0; e < V; ++e) tmp[e] = stage[swz<E>(q0 + e)];
      st_stream_v4(out + g0, *reinterpret_cast<int4*>(tmp));
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const long long g = g0 + e;
        if (g >= base && g < base + cnt) out[g] = stage[swz<E>(off + (int)(g - base))];
      }
    }
  }
}

// Warp-striped tile load + selection.  kByCs: selection from a bool (u8)
// array (filter_by) instead of the predicate.
template <typename T, bool kByCs>
struct TileLoad {
  static constexpr int V = 16 / (int)sizeof(T);
  static constexpr int R = kItems / V;
  T x[R][V];
  bool s[R][V];

  IXG_DEV static long long index(long long tile_base, int r, int e) {
    return tile_base + warp_id() * (32 * kItems) + r * (32 * V) + lane_id() * V + e;
  }
  IXG_DEV static int local(int r, int e) { return warp_id() * (32 * kItems) + r * (32 * V) + lane_id() * V + e; }

  IXG_DEV void load(const T* __restrict__ xs, const uint8_t* __restrict__ cs, long long n, long long tile_base,
                    const ixg_pred& p) {
    const bool full = tile_base + kTile <= n;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const long long i0 = index(tile_base, r, 0);
      if (full) {
        int4 raw = ld_stream_v4(xs + i0);
        Vec<T>::unpack(raw, x[r]);
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e) x[r][e] = (i0 + e < n) ? xs[i0 + e] : T(0);
      }
      if (kByCs) {
#pragma unroll
        for (int e = 0; e < V; ++e) s[r][e] = (i0 + e < n) && cs[i0 + e] != 0;
      } else {
#pragma unroll
        for (int e = 0; e < V; ++e) s[r][e] = (i0 + e < n) && pred_eval(p, (long long)x[r][e]);
      }
    }
  }

  // rank of each selected element among the selected elements of its warp
  // slice; returns the warp's selected count.
  IXG_DEV int rank(int (&rk)[R][V]) const {
    const uint32_t lt = lanemask_lt();
    int running = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      int lane_prefix = 0, row_cnt = 0;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        const uint32_t b = __ballot_sync(0xffffffffu, s[r][e]);
        lane_prefix += __popc(b & lt);
        row_cnt += __popc(b);
      }
      int mine = 0;
#pragma unroll
      for (int e = 0; e < V; ++e) {
        rk[r][e] = running + lane_prefix + mine;
        mine += s[r][e] ? 1 : 0;
      }
      running += row_cnt;
    }
    return running;
  }
};

// ---------------------------------------------------------------------------
// filter / filter_by, optionally fused with mkFlags + sgmSum (C2).
//   ys[k] <- xs[i] for the k-th selected i          (filter.ixl:8-14, Sc1)
//   zs = sgmSum flags ys, flags[j] = bit (out_base + j) of segbits (mkFlags)
template <typename T, typename Z, bool kByCs, bool kSeg>
__global__ void __launch_bounds__(kThreads) k_filter(const T* __restrict__ xs, const uint8_t* __restrict__ cs,
                                                      long long n, ixg_pred p, T* __restrict__ ys,
                                                      Z* __restrict__ zs, const uint32_t* __restrict__ segbits,
                                                      long long out_base, LBChan cnt_ch, LBChan seg_ch,
                                                      long long* d_count, longlong2* d_seg_total,
                                                      ixg_status* st) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* stage = reinterpret_cast<T*>(smem_raw);
  Z* stage_z = reinterpret_cast<Z*>(smem_raw + kTile * sizeof(T));
  __shared__ int s_warp[kWarps];
  __shared__ long long s_tile;
  __shared__ uint32_t s_epoch[2];
  __shared__ long long s_excl;
  __shared__ SegOp::T s_seg[kWarps];
  __shared__ SegOp::T s_carry;

  if (threadIdx.x == 0) {
    long long t;
    uint32_t ep;
    lb_ticket(cnt_ch, &t, &ep);
    s_tile = t;
    s_epoch[0] = ep;
    if (kSeg) s_epoch[1] = ((volatile LBHeader*)seg_ch.hdr)->epoch & kEpochMask;
  }
  __syncthreads();
  const long long tile = s_tile;
  const uint32_t ep = s_epoch[0];
  const long long tile_base = tile * kTile;

  using L = TileLoad<T, kByCs>;
  L ld;
  ld.load(xs, cs, n, tile_base, p);
  int rk[L::R][L::V];
  const int wcnt = ld.rank(rk);
  if (lane_id() == 0) s_warp[warp_id()] = wcnt;
  __syncthreads();
  int wexcl = 0, cnt = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    wexcl += (w < warp_id()) ? s_warp[w] : 0;
    cnt += s_warp[w];
  }
  if (threadIdx.x == 0) lb_publish<SumOp>(cnt_ch, ep, tile, SumOp::T{cnt}, tile == 0);
  // stage the compacted elements while the look-back runs
#pragma unroll
  for (int r = 0; r < L::R; ++r)
#pragma unroll
    for (int e = 0; e < L::V; ++e)
      if (ld.s[r][e]) stage[swz<T>(wexcl + rk[r][e])] = ld.x[r][e];
  if (warp_id() == 0) {
    long long ex = 0;
    if (tile > 0) ex = lb_lookback<SumOp>(cnt_ch, ep, tile).v;
    if (lane_id() == 0) {
      s_excl = ex;
      if (tile > 0) lb_publish<SumOp>(cnt_ch, ep, tile, SumOp::T{ex + cnt}, true);
    }
  }
  __syncthreads();
  const long long base = s_excl;
  if (tile == (long long)gridDim.x - 1 && threadIdx.x == 0) *d_count = base + cnt;

  if (kSeg) {
    // blocked segmented sum over the tile's output run
    const int q0 = threadIdx.x * kItems;
    constexpr int VZ = 16 / (int)sizeof(T);
    T v[kItems];
#pragma unroll
    for (int c = 0; c < kItems / VZ; ++c) {
      const int4 raw = *reinterpret_cast<const int4*>(&stage[swz<T>(q0 + c * VZ)]);
      T tmp[VZ];
      Vec<T>::unpack(raw, tmp);
#pragma unroll
      for (int e = 0; e < VZ; ++e) v[c * VZ + e] = tmp[e];
    }
    const long long g0 = out_base + base + q0;
    const long long wd = g0 >> 5;
    uint64_t bits = 0;
    if (q0 < cnt)
      bits = (((uint64_t)__ldg(&segbits[wd + 1]) << 32) | (uint64_t)__ldg(&segbits[wd])) >> (g0 & 31);
    SegOp::T a = SegOp::identity();
#pragma unroll
    for (int j = 0; j < kItems; ++j)
      if (q0 + j < cnt) a = SegOp::op(a, SegOp::T{(long long)v[j], (int)((bits >> j) & 1)});
    SegOp::T inc = warp_inclusive<SegOp>(a);
    SegOp::T lex = SegOp::shfl_up(inc, 1);
    if (lane_id() == 0) lex = SegOp::identity();
    if (lane_id() == 31) s_seg[warp_id()] = inc;
    __syncthreads();
    SegOp::T wpre = SegOp::identity(), tagg = SegOp::identity();
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      if (w < warp_id()) wpre = SegOp::op(wpre, s_seg[w]);
      tagg = SegOp::op(tagg, s_seg[w]);
    }
    const uint32_t ep2 = s_epoch[1];
    if (threadIdx.x == 0) lb_publish<SegOp>(seg_ch, ep2, tile, tagg, tile == 0);
    if (warp_id() == 0) {
      SegOp::T carry = SegOp::identity();
      if (tile > 0) carry = lb_lookback<SegOp>(seg_ch, ep2, tile);
      if (lane_id() == 0) {
        s_carry = carry;
        SegOp::T incl = SegOp::op(carry, tagg);
        if (tile > 0) lb_publish<SegOp>(seg_ch, ep2, tile, incl, true);
        if (tile == (long long)gridDim.x - 1 && d_seg_total) *d_seg_total = make_longlong2(incl.v, incl.f);
      }
    }
    __syncthreads();
    SegOp::T run = SegOp::op(SegOp::op(s_carry, wpre), lex);
    bool narrow = false;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      if (q0 + j < cnt) {
        run = SegOp::op(run, SegOp::T{(long long)v[j], (int)((bits >> j) & 1)});
        if (sizeof(Z) == 4 && run.v != (long long)(int)run.v) narrow = true;
        stage_z[swz<Z>(q0 + j)] = (Z)run.v;
      }
    }
    if (narrow && st) atomicOr(&st->flags, IXG_F_NARROW);
    __syncthreads();
    store_run<Z>(zs, base, cnt, stage_z, 0);
  }
  store_run<T>(ys, base, cnt, stage, 0);
  if (threadIdx.x == 0) {
    lb_retire(cnt_ch, ep);
    if (kSeg) lb_retire(seg_ch, s_epoch[1]);
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
__global__ void __launch_bounds__(kThreads) k_class_count(const T* __restrict__ xs, long long n, ixg_pred p,
                                                           ixg_pred q, long long* partials, LBHeader* hdr,
                                                           long long* d_tot) {
  constexpr int V = 16 / (int)sizeof(T);
  long long c0 = 0, c1 = 0;
  const long long nv = n / V;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = (long long)blockIdx.x * kThreads + threadIdx.x; i < nv; i += stride) {
    T x[V];
    Vec<T>::unpack(ld_stream_v4(xs + i * V), x);
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int c = classify<T, kClasses>(p, q, x[e]);
      c0 += (c == 0);
      if (kClasses == 3) c1 += (c == 1);
    }
  }
  if (blockIdx.x == 0)
    for (long long i = nv * V + threadIdx.x; i < n; i += kThreads) {
      const int c = classify<T, kClasses>(p, q, xs[i]);
      c0 += (c == 0);
      if (kClasses == 3) c1 += (c == 1);
    }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    c0 += __shfl_xor_sync(0xffffffffu, c0, d);
    c1 += __shfl_xor_sync(0xffffffffu, c1, d);
  }
  __shared__ long long s0[kWarps], s1[kWarps];
  __shared__ bool s_last;
  if (lane_id() == 0) {
    s0[warp_id()] = c0;
    s1[warp_id()] = c1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0;
    for (int w = 0; w < kWarps; ++w) {
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
    for (int i = threadIdx.x; i < (int)gridDim.x; i += kThreads) {
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
      for (int w = 0; w < kWarps; ++w) {
        ta += s0[w];
        tb += s1[w];
      }
      d_tot[0] = ta;
      if (kClasses == 3) d_tot[1] = tb;
      hdr->done = 0;
    }
  }
}

// Pass 2: single-pass placement.  Class c of this tile is a contiguous run of
// the output starting at  start_c = (sum of smaller classes' totals)
// + (class-c elements before this tile); the look-back carries the class-0
// (and class-1) prefix, class kClasses-1's prefix is the rest.
template <typename T, int kClasses>
__global__ void __launch_bounds__(kThreads) k_place(const T* __restrict__ xs, long long n, ixg_pred p, ixg_pred q,
                                                     T* __restrict__ ys, const long long* __restrict__ d_tot,
                                                     LBChan ch) {
  using M = typename std::conditional<kClasses == 2, SumOp, Sum2Op>::type;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* stage = reinterpret_cast<T*>(smem_raw);
  __shared__ int s_warp[kWarps][2];
  __shared__ long long s_tile;
  __shared__ uint32_t s_epoch;
  __shared__ long long s_ex[2];

  if (threadIdx.x == 0) {
    long long t;
    uint32_t ep;
    lb_ticket(ch, &t, &ep);
    s_tile = t;
    s_epoch = ep;
  }
  __syncthreads();
  const long long tile = s_tile;
  const uint32_t ep = s_epoch;
  const long long tile_base = tile * kTile;
  const int tile_len = (int)min((long long)kTile, n - tile_base);

  constexpr int V = 16 / (int)sizeof(T);
  constexpr int R = kItems / V;
  T x[R][V];
  int cls[R][V];
  const bool full = tile_base + kTile <= n;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const long long i0 = tile_base + warp_id() * (32 * kItems) + r * (32 * V) + lane_id() * V;
    if (full) {
      Vec<T>::unpack(ld_stream_v4(xs + i0), x[r]);
    } else {
#pragma unroll
      for (int e = 0; e < V; ++e) x[r][e] = (i0 + e < n) ? xs[i0 + e] : T(0);
    }
#pragma unroll
    for (int e = 0; e < V; ++e) cls[r][e] = (i0 + e < n) ? classify<T, kClasses>(p, q, x[r][e]) : -1;
  }
  // ranks for class 0 and class 1 (class 2's rank is local index - r0 - r1)
  const uint32_t lt = lanemask_lt();
  int rk0[R][V], rk1[R][V];
  int run0 = 0, run1 = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    int lp0 = 0, rc0 = 0, lp1 = 0, rc1 = 0;
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const uint32_t b0 = __ballot_sync(0xffffffffu, cls[r][e] == 0);
      lp0 += __popc(b0 & lt);
      rc0 += __popc(b0);
      if (kClasses == 3) {
        const uint32_t b1 = __ballot_sync(0xffffffffu, cls[r][e] == 1);
        lp1 += __popc(b1 & lt);
        rc1 += __popc(b1);
      }
    }
    int m0 = 0, m1 = 0;
#pragma unroll
    for (int e = 0; e < V; ++e) {
      rk0[r][e] = run0 + lp0 + m0;
      rk1[r][e] = run1 + lp1 + m1;
      m0 += cls[r][e] == 0;
      m1 += cls[r][e] == 1;
    }
    run0 += rc0;
    run1 += rc1;
  }
  if (lane_id() == 0) {
    s_warp[warp_id()][0] = run0;
    s_warp[warp_id()][1] = run1;
  }
  __syncthreads();
  int we0 = 0, we1 = 0, c0 = 0, c1 = 0;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) {
    if (w < warp_id()) {
      we0 += s_warp[w][0];
      we1 += s_warp[w][1];
    }
    c0 += s_warp[w][0];
    c1 += s_warp[w][1];
  }
  typename M::T agg;
  if constexpr (kClasses == 2) agg = typename M::T{c0};
  else agg = typename M::T{c0, c1};
  if (threadIdx.x == 0) lb_publish<M>(ch, ep, tile, agg, tile == 0);
  // stage: class 0 run, then class 1 run, then class 2 run
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int c = cls[r][e];
      if (c < 0) continue;
      const int li = warp_id() * (32 * kItems) + r * (32 * V) + lane_id() * V + e;
      int pos;
      if (c == 0) pos = we0 + rk0[r][e];
      else if (kClasses == 3 && c == 1) pos = c0 + we1 + rk1[r][e];
      else pos = c0 + (kClasses == 3 ? c1 : 0) + (li - (we0 + rk0[r][e]) - (kClasses == 3 ? we1 + rk1[r][e] : 0));
      stage[swz<T>(pos)] = x[r][e];
    }
  if (warp_id() == 0) {
    typename M::T ex = M::identity();
    if (tile > 0) ex = lb_lookback<M>(ch, ep, tile);
    if (lane_id() == 0) {
      if constexpr (kClasses == 2) {
        s_ex[0] = ex.v;
        s_ex[1] = 0;
      } else {
        s_ex[0] = ex.a;
        s_ex[1] = ex.b;
      }
      if (tile > 0) lb_publish<M>(ch, ep, tile, M::op(ex, agg), true);
    }
  }
  __syncthreads();
  const long long e0 = s_ex[0], e1 = s_ex[1];
  const long long t0 = d_tot[0];
  const long long t1 = kClasses == 3 ? d_tot[1] : 0;
  store_run<T>(ys, e0, c0, stage, 0);
  if (kClasses == 3) store_run<T>(ys, t0 + e1, c1, stage, c0);
  const int c2 = tile_len - c0 - (kClasses == 3 ? c1 : 0);
  const long long e2 = tile_base - e0 - (kClasses == 3 ? e1 : 0);
  store_run<T>(ys, t0 + t1 + e2, c2, stage, c0 + (kClasses == 3 ? c1 : 0));
  if (threadIdx.x == 0) lb_retire(ch, ep);
}

}  // namespace ixg
