// lookback.cuh -- decoupled look-back tile state for single-pass scans.
//
// Every scan on the hot path (scan (+) of oracle.py:281-293, the segmented
// scan of PAPER.md:399-402, the count/offset scans inside filter/partition)
// is ONE pass over HBM: a CTA takes a tile ticket, reduces its tile, publishes
// the aggregate, and warp 0 walks back over its predecessors' published
// aggregates/prefixes 32 tiles at a time until it meets an inclusive prefix.
//
// Tile state = one 16-byte slot per tile, written with one 16-byte store and
// polled with one 16-byte L2 load (one round trip per 32-tile window):
//   w0 = payload (int64 sum / segmented value / two packed 32-bit counts)
//   w1 = [epoch:24][status:2][flag:1][pad:5][check:32]
// status 1 = aggregate, 2 = inclusive prefix.  A slot is first written with
// its aggregate and later overwritten with its inclusive prefix; `check`
// (a function of w0 and the epoch) lets a reader reject a torn read of the
// two 8-byte halves and retry.
//
// Forward progress on sm_100a: tiles are handed out by an atomic ticket
// (not blockIdx), so a CTA only ever waits on tiles owned by CTAs that are
// already resident.
//
// The workspace is self-resetting: slots carry a 24-bit launch epoch, and
// the last CTA of a launch bumps the epoch and zeroes the ticket, so a
// zero-initialised workspace can be reused by any number of stream-ordered
// launches without a memset.
#pragma once
#include "common.cuh"

namespace ixg {

struct LBHeader {
  unsigned int ticket;
  unsigned int done;
  unsigned int epoch;
  unsigned int dup;  // scatter: "a destination was claimed twice" (self-reset by verify)
};

struct LBChan {
  LBHeader* hdr;
  ulonglong2* slot;  // [tiles]
};

constexpr uint32_t kStAgg = 1, kStIncl = 2;
constexpr uint32_t kEpochMask = 0xffffffu;

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
IXG_DEV uint32_t slot_check(unsigned long long w0, uint32_t epoch) {
  return (uint32_t)w0 ^ (uint32_t)(w0 >> 32) ^ (epoch * 0x9E3779B1u) ^ 0x5bd1e995u;
}
IXG_DEV void slot_store(ulonglong2* p, unsigned long long w0, uint32_t epoch, uint32_t status, uint32_t flag) {
  const unsigned long long w1 = ((unsigned long long)((epoch << 8) | (status << 6) | (flag << 5)) << 32) |
                                (unsigned long long)slot_check(w0, epoch);
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(w0), "l"(w1) : "memory");
}
// returns status (0 = not ready / stale / torn)
IXG_DEV uint32_t slot_load(const ulonglong2* p, uint32_t epoch, unsigned long long* w0, uint32_t* flag) {
  unsigned long long a, b;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
  const uint32_t hi = (uint32_t)(b >> 32);
  if ((hi >> 8) != epoch || (uint32_t)b != slot_check(a, epoch)) return 0;
  *w0 = a;
  *flag = (hi >> 5) & 1u;
  return (hi >> 6) & 3u;
}

// ------------------------------------------------------------ tile protocol
// Called by thread 0: take a ticket and read the launch epoch.
IXG_DEV void lb_ticket(const LBChan& ch, long long* tile, uint32_t* epoch) {
  volatile LBHeader* h = ch.hdr;
  *epoch = h->epoch & kEpochMask;
  *tile = (long long)atomicAdd(&ch.hdr->ticket, 1u);
}
IXG_DEV uint32_t lb_epoch(const LBChan& ch) { return ((volatile LBHeader*)ch.hdr)->epoch & kEpochMask; }

// Called by thread 0 at the very end of the CTA: the last CTA resets the header.
IXG_DEV void lb_retire(const LBChan& ch, uint32_t epoch) {
  __threadfence();
  unsigned int prev = atomicAdd(&ch.hdr->done, 1u);
  if (prev == gridDim.x - 1) {
    volatile LBHeader* h = ch.hdr;
    h->ticket = 0;
    h->done = 0;
    h->epoch = (epoch + 1) & kEpochMask;
    __threadfence();
  }
}

template <class M>
IXG_DEV void lb_publish(const LBChan& ch, uint32_t epoch, long long tile, typename M::T v, bool inclusive) {
  uint32_t f;
  const unsigned long long w = M::payload(v, &f);
  slot_store(&ch.slot[tile], w, epoch, inclusive ? kStIncl : kStAgg, f);
}

// Warp-collective (all 32 lanes of one warp): exclusive prefix of `tile`
// (tile > 0) from its predecessors.
//
// Window = 32 lanes x kPerLane tiles = 256 predecessors per L2 round trip.
// The window must cover every tile whose look-back is still in flight
// (aggregate published, inclusive prefix not yet): that lag is one round
// trip r (~0.5-1 us under load) / tile interval delta (~4 ns for a 4096
// x int32 tile at 6.5 TB/s) ~ 150-250 tiles.  A 32-tile window cannot
// cover it and the walk degenerates into many serial round trips.
#ifndef IXG_LB_PER_LANE
#define IXG_LB_PER_LANE 8
#endif
constexpr int kPerLane = IXG_LB_PER_LANE;

template <class M>
IXG_DEV typename M::T lb_lookback(const LBChan& ch, uint32_t epoch, long long tile) {
  using T = typename M::T;
  const int lane = lane_id();
  T excl = M::identity();
  long long pred = tile - 1;
  while (true) {
    // lane l holds tiles pred - (l*kPerLane + j), j = 0 (newest) .. kPerLane-1
    unsigned long long w[kPerLane];
    uint32_t f[kPerLane], st[kPerLane];
#pragma unroll
    for (int j = 0; j < kPerLane; ++j) {
      const long long idx = pred - (lane * kPerLane + j);
      st[j] = kStIncl;  // virtual inclusive identity before tile 0
      w[j] = 0;
      f[j] = 0;
      if (idx >= 0) st[j] = slot_load(&ch.slot[idx], epoch, &w[j], &f[j]);
    }
    // re-poll only the slots that were not ready
    int spins = 0;
    while (true) {
      bool ready = true;
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) ready &= st[j] != 0;
      if (ready) break;
      if (++spins > 32) __nanosleep(16);
#pragma unroll
      for (int j = 0; j < kPerLane; ++j) {
        const long long idx = pred - (lane * kPerLane + j);
        if (st[j] == 0) st[j] = slot_load(&ch.slot[idx], epoch, &w[j], &f[j]);
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
