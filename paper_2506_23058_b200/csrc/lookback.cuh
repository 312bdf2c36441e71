// lookback.cuh -- decoupled look-back tile state for single-pass scans.
//
// Every scan on the hot path (scan (+) of oracle.py:281-293, the segmented
// scan of PAPER.md:399-402, the count/offset scans inside filter/partition)
// is ONE pass over HBM: tile t (= blockIdx.x) reduces its elements, publishes
// the aggregate, and its warp 0 walks back over the predecessors' published
// aggregates / inclusive prefixes, 32 x kPerLane tiles per L2 round trip,
// until it meets an inclusive prefix.
//
// Tile state = one 16-byte slot per tile, written with one 16-byte store and
// polled with one 16-byte L2 load:
//   w0 = payload (int64 sum / segmented value / two packed 32-bit counts)
//   w1 = [nonce:24][status:2][flag:1][pad:5][check:32]
// status 1 = aggregate, 2 = inclusive prefix.  A slot is first written with
// its aggregate and later overwritten with its inclusive prefix; `check`
// (a function of w0 and the nonce) lets a reader reject a torn read of the
// two 8-byte halves and retry.  The nonce is a per-launch value from the
// host, so slots left by earlier launches are never mistaken for current
// ones and the workspace is never reset.
//
// Slots of consecutive tiles are kSlotStride x 16 B apart: every warp that
// is looking back polls the slots of the most recent tiles, and packed slots
// put all of that traffic on a handful of L2 lines (one LTS slice).
// Measured at 2^28 (tools/_ab2.sh): stride 8 + a 32-tile window is the best
// of {stride 1, 8, 16} x {32, 64, 128, 512}-tile windows -- wider windows
// cost more in polling traffic than they save in walk length.
#pragma once
#include "common.cuh"

namespace ixg {

struct LBHeader {  // scratch words of the non-scan kernels (scatter dup flag, count partials)
  unsigned int ticket;
  unsigned int done;
  unsigned int epoch;
  unsigned int dup;
};

struct LBChan {
  LBHeader* hdr;
  ulonglong2* slot;  // [tiles * kSlotStride]
};

constexpr uint32_t kStAgg = 1, kStIncl = 2;
constexpr uint32_t kNonceMask = 0xffffffu;

#ifndef IXG_SLOT_STRIDE
#define IXG_SLOT_STRIDE 8
#endif
#ifndef IXG_LB_PER_LANE
#define IXG_LB_PER_LANE 1
#endif
constexpr int kSlotStride = IXG_SLOT_STRIDE;
constexpr int kPerLane = IXG_LB_PER_LANE;
#ifndef IXG_LB_SLEEP
#define IXG_LB_SLEEP 0  // ns between re-polls of unready slots (0: 32 tight spins, then 16 ns)
#endif

IXG_DEV ulonglong2* slot_at(const LBChan& ch, long long tile) { return ch.slot + tile * kSlotStride; }

// ------------------------------------------------------------ monoids
// payload(): value -> (w0, flag bit);  from(): (w0, flag) -> value
struct SumOp {  // int64 sums (counts, scan (+))
  struct T { long long v; };
  IXG_DEV static T identity() { return T{0}; }
  IXG_DEV static T op(T a, T b) { return T{a.v + b.v}; }  // a earlier, b later
  IXG_DEV static unsigned long long payload(T a, uint32_t* f) { *f = 0; return (unsigned long long)a.v; }
  IXG_DEV static T from(unsigned long long w, uint32_t) { return T{(long long)w}; }
  IXG_DEV static T shfl_down(T a, int d) { return T{__shfl_down_sync(0xffffffffu, a.v, d)}; }
  IXG_DEV static T shfl_up(T a, int d) { return T{__shfl_up_sync(0xffffffffu, a.v, d)}; }
  IXG_DEV static T shfl(T a, int l) { return T{__shfl_sync(0xffffffffu, a.v, l)}; }
};

// Pair of counts (partition3's two class counts); each < 2^32 in the slot.
struct Sum2Op {
  struct T { long long a, b; };
  IXG_DEV static T identity() { return T{0, 0}; }
  IXG_DEV static T op(T x, T y) { return T{x.a + y.a, x.b + y.b}; }
  IXG_DEV static unsigned long long payload(T x, uint32_t* f) {
    *f = 0;
    return (unsigned long long)(uint32_t)x.a | ((unsigned long long)(uint32_t)x.b << 32);
  }
  IXG_DEV static T from(unsigned long long w, uint32_t) { return T{(long long)(w & 0xffffffffull), (long long)(w >> 32)}; }
  IXG_DEV static T shfl_down(T x, int d) {
    return T{__shfl_down_sync(0xffffffffu, x.a, d), __shfl_down_sync(0xffffffffu, x.b, d)};
  }
  IXG_DEV static T shfl_up(T x, int d) {
    return T{__shfl_up_sync(0xffffffffu, x.a, d), __shfl_up_sync(0xffffffffu, x.b, d)};
  }
  IXG_DEV static T shfl(T x, int l) {
    return T{__shfl_sync(0xffffffffu, x.a, l), __shfl_sync(0xffffffffu, x.b, l)};
  }
};

// Segmented sum: the lifted operator of sgmSum
//   (f1, v1) (+) (f2, v2) = (f1 || f2, if f2 then v2 else v1 + v2)
// Associative, not commutative: op(a, b) with a EARLIER than b.
struct SegOp {
  struct T { long long v; int f; };
  IXG_DEV static T identity() { return T{0, 0}; }
  IXG_DEV static T op(T a, T b) { return T{b.f ? b.v : a.v + b.v, a.f | b.f}; }
  IXG_DEV static unsigned long long payload(T a, uint32_t* f) { *f = (uint32_t)(a.f != 0); return (unsigned long long)a.v; }
  IXG_DEV static T from(unsigned long long w, uint32_t f) { return T{(long long)w, (int)f}; }
  IXG_DEV static T shfl_down(T a, int d) {
    return T{__shfl_down_sync(0xffffffffu, a.v, d), __shfl_down_sync(0xffffffffu, a.f, d)};
  }
  IXG_DEV static T shfl_up(T a, int d) {
    return T{__shfl_up_sync(0xffffffffu, a.v, d), __shfl_up_sync(0xffffffffu, a.f, d)};
  }
  IXG_DEV static T shfl(T a, int l) {
    return T{__shfl_sync(0xffffffffu, a.v, l), __shfl_sync(0xffffffffu, a.f, l)};
  }
};

// ------------------------------------------------------------ slot codec
IXG_DEV uint32_t slot_check(unsigned long long w0, uint32_t nonce) {
  return (uint32_t)w0 ^ (uint32_t)(w0 >> 32) ^ (nonce * 0x9E3779B1u) ^ 0x5bd1e995u;
}
IXG_DEV void slot_store(ulonglong2* p, unsigned long long w0, uint32_t nonce, uint32_t status, uint32_t flag) {
  const unsigned long long w1 = ((unsigned long long)((nonce << 8) | (status << 6) | (flag << 5)) << 32) |
                                (unsigned long long)slot_check(w0, nonce);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
// returns status (0 = not ready / stale / torn)
IXG_DEV uint32_t slot_load(const ulonglong2* p, uint32_t nonce, unsigned long long* w0, uint32_t* flag) {
  unsigned long long a, b;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  const uint32_t hi = (uint32_t)(b >> 32);
  if ((hi >> 8) != nonce || (uint32_t)b != slot_check(a, nonce)) return 0;
  *w0 = a;
  *flag = (hi >> 5) & 1u;
  return (hi >> 6) & 3u;
}

template <class M>
IXG_DEV void lb_publish(const LBChan& ch, uint32_t nonce, long long tile, typename M::T v, bool inclusive) {
  uint32_t f;
  const unsigned long long w = M::payload(v, &f);
  slot_store(slot_at(ch, tile), w, nonce, inclusive ? kStIncl : kStAgg, f);
}

// Warp-collective (all 32 lanes of one warp): exclusive prefix of `tile`
// (tile > 0) from its predecessors.
template <class M>
IXG_DEV typename M::T lb_lookback(const LBChan& ch, uint32_t nonce, long long tile) {
  using T = typename M::T;
  const int lane = lane_id();
  T excl = M::identity();
  long long pred = tile - 1;
#ifdef IXG_TRACE
  unsigned int tr_rounds = 0, tr_spins = 0;
#endif
  while (true) {
#ifdef IXG_TRACE
    ++tr_rounds;
#endif
    // lane l holds tiles pred - (l*kPerLane + j), j = 0 (newest) .. kPerLane-1
    unsigned long long w[kPerLane];
    uint32_t f[kPerLane], st[kPerLane];
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
      const long long idx = pred - (lane * kPerLane + j);
      st[j] = kStIncl;  // virtual inclusive identity before tile 0
      w[j] = 0;
      f[j] = 0;
      if (idx >= 0) st[j] = slot_load(slot_at(ch, idx), nonce, &w[j], &f[j]);
    }
    // re-poll only the slots that were not ready
    int spins = 0;
    while (true) {
      bool ready = true;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) ready &= st[j] != 0;
      if (ready) break;
#ifdef IXG_TRACE
      ++tr_spins;
#endif
      if (IXG_LB_SLEEP) {
        __nanosleep(IXG_LB_SLEEP);
      } else if (++spins > 32) {
        __nanosleep(16);
      }
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        const long long idx = pred - (lane * kPerLane + j);
        if (st[j] == 0) st[j] = slot_load(slot_at(ch, idx), nonce, &w[j], &f[j]);
      }
    }
    // this lane's newest inclusive slot (kPerLane = none)
    int jstop = kPerLane;
#pragma unroll
    for (int j = kPerLane - 1; j >= 0; --j)
      if (st[j] == kStIncl) jstop = j;
    const uint32_t incl_mask = __ballot_sync(0xffffffffu, jstop < kPerLane);
    const int stop = incl_mask ? (__ffs(incl_mask) - 1) : 32;
    // lane-local ordered fold, oldest -> newest, cut at the inclusive slot
    T v = M::identity();
    if (lane <= stop) {
      const int jmax = (lane == stop) ? jstop : kPerLane - 1;
#pragma unroll
      for (int j = kPerLane - 1; j >= 0; --j)
        if (j <= jmax) v = M::op(v, M::from(w[j], f[j]));
    }
    // ordered warp reduction: lane 0 holds the newest tiles
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T o = M::shfl_down(v, d);
      if (lane + d < 32) v = M::op(o, v);
    }
    excl = M::op(M::shfl(v, 0), excl);
    if (incl_mask) break;
    pred -= 32 * kPerLane;
  }
#ifdef IXG_TRACE
  if (lane == 0 && blockIdx.x < (1u << 17)) g_trace[blockIdx.x * IXG_TRS + (std::is_same<M, SegOp>::value ? 13 : 7)] =
      ((unsigned long long)tr_rounds << 32) | tr_spins;
#endif
  return excl;
}

// Warp inclusive scan (lanes in order).
template <class M>
IXG_DEV typename M::T warp_inclusive(typename M::T v) {
  const int lane = lane_id();
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    typename M::T o = M::shfl_up(v, d);
    if (lane >= d) v = M::op(o, v);
  }
  return v;
}

}  // namespace ixg
