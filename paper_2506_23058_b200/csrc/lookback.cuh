// lookback.cuh -- decoupled look-back tile state for single-pass scans.
//
// Every scan on the hot path (scan (+) of oracle.py:281-293, the segmented
// scan of PAPER.md:399-402, the count/offset scans inside filter/partition)
// is ONE pass over HBM: a CTA takes a tile ticket, reduces its tile, publishes
// the aggregate, and warp 0 walks back over its predecessors' published
// aggregates/prefixes 32 tiles at a time until it meets an inclusive prefix.
//
// Forward progress on sm_100a: tiles are handed out by an atomic ticket
// (not blockIdx), so a CTA only ever waits on tiles owned by CTAs that are
// already resident.  Ordering: the payload is stored (st.global.cg) by the
// same thread that then releases the flag word (st.release.gpu); readers
// acquire the flag (ld.acquire.gpu) and read the payload through L2 (ld.cg).
//
// The workspace is self-resetting: flag words carry a 29-bit launch epoch,
// and the last CTA of a launch bumps the epoch and zeroes the ticket, so a
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
  uint32_t* flags;    // [tiles]  (epoch << 3) | (extra << 2) | status
  longlong2* agg;     // [tiles]
  longlong2* incl;    // [tiles]
};

constexpr uint32_t kStAgg = 1, kStIncl = 2;
constexpr uint32_t kEpochMask = 0x1fffffffu;

inline size_t lb_bytes(long long tiles) {
  size_t t = (size_t)(tiles > 0 ? tiles : 1);
  return 256 + ((t * 4 + 255) / 256) * 256 + 2 * t * sizeof(longlong2);
}
// carve one channel out of `ws`; returns bytes used
inline size_t lb_carve(void* ws, long long tiles, LBChan* ch) {
  size_t t = (size_t)(tiles > 0 ? tiles : 1);
  char* p = (char*)ws;
  ch->hdr = (LBHeader*)p;
  p += 256;
  ch->flags = (uint32_t*)p;
  p += ((t * 4 + 255) / 256) * 256;
  ch->agg = (longlong2*)p;
  p += t * sizeof(longlong2);
  ch->incl = (longlong2*)p;
  return lb_bytes(tiles);
}

// ------------------------------------------------------------ monoids
// Sum of int64 (counts, scan (+)).  Associative and commutative.
struct SumOp {
  struct T { long long v; };
  IXG_DEV static T identity() { return T{0}; }
  IXG_DEV static T op(T a, T b) { return T{a.v + b.v}; }  // a earlier, b later
  IXG_DEV static longlong2 store(T a, uint32_t* extra) { *extra = 0; return make_longlong2(a.v, 0); }
  IXG_DEV static T load(longlong2 p, uint32_t) { return T{p.x}; }
  IXG_DEV static T shfl_down(T a, int d) { return T{__shfl_down_sync(0xffffffffu, a.v, d)}; }
  IXG_DEV static T shfl_up(T a, int d) { return T{__shfl_up_sync(0xffffffffu, a.v, d)}; }
  IXG_DEV static T shfl(T a, int l) { return T{__shfl_sync(0xffffffffu, a.v, l)}; }
};

// Pair of int64 sums (partition3's two class counts).
struct Sum2Op {
  struct T { long long a, b; };
  IXG_DEV static T identity() { return T{0, 0}; }
  IXG_DEV static T op(T x, T y) { return T{x.a + y.a, x.b + y.b}; }
  IXG_DEV static longlong2 store(T x, uint32_t* extra) { *extra = 0; return make_longlong2(x.a, x.b); }
  IXG_DEV static T load(longlong2 p, uint32_t) { return T{p.x, p.y}; }
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
  IXG_DEV static longlong2 store(T a, uint32_t* extra) { *extra = (uint32_t)(a.f != 0); return make_longlong2(a.v, 0); }
  IXG_DEV static T load(longlong2 p, uint32_t extra) { return T{p.x, (int)extra}; }
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

// ------------------------------------------------------------ tile protocol
// Called by thread 0: take a ticket and read the launch epoch.
IXG_DEV void lb_ticket(const LBChan& ch, long long* tile, uint32_t* epoch) {
  volatile LBHeader* h = ch.hdr;
  *epoch = h->epoch & kEpochMask;
  *tile = (long long)atomicAdd(&ch.hdr->ticket, 1u);
}

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
  uint32_t extra;
  longlong2 p = M::store(v, &extra);
  __stcg(inclusive ? &ch.incl[tile] : &ch.agg[tile], p);
  st_release_u32(&ch.flags[tile], (epoch << 3) | (extra << 2) | (inclusive ? kStIncl : kStAgg));
}

// Warp-collective (all 32 lanes of one warp): exclusive prefix of `tile`
// (tile > 0) from its predecessors.
template <class M>
IXG_DEV typename M::T lb_lookback(const LBChan& ch, uint32_t epoch, long long tile) {
  using T = typename M::T;
  const int lane = lane_id();
  T excl = M::identity();
  long long pred = tile - 1;
  while (true) {
    long long idx = pred - lane;
    uint32_t f = (epoch << 3) | kStIncl;  // virtual inclusive identity before tile 0
    T v = M::identity();
    if (idx >= 0) {
      int spins = 0;
      while (true) {
        f = ld_acquire_u32(&ch.flags[idx]);
        if ((f >> 3) == epoch && (f & 3u) != 0u) break;
        if (++spins > 4) __nanosleep(32);
      }
      longlong2 p = __ldcg((f & 3u) == kStIncl ? &ch.incl[idx] : &ch.agg[idx]);
      v = M::load(p, (f >> 2) & 1u);
    }
    const uint32_t incl_mask = __ballot_sync(0xffffffffu, (f & 3u) == kStIncl);
    const int stop = incl_mask ? (__ffs(incl_mask) - 1) : 31;
    if (lane > stop) v = M::identity();
    // ordered reduction: lane 0 is the newest tile, lane 31 the oldest
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T o = M::shfl_down(v, d);
      if (lane + d < 32) v = M::op(o, v);
    }
    T window = M::shfl(v, 0);
    excl = M::op(window, excl);
    if (incl_mask) break;
    pred -= 32;
  }
  return excl;
}

// Warp inclusive scan (lanes in order), returns inclusive; *total = lane 31's.
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
