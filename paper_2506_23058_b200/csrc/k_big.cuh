// k_big.cuh -- big-tile streaming kernels: the tile is staged in shared
// memory by the TMA engine (cp.async.bulk on mbarriers; per-lane cp.async
// only for the ragged last tile), so a CTA keeps its whole tile of HBM reads
// in flight without spending registers on them.
//
// Why: a trace of the register-tiled kernels showed every CTA
// spending ~5 us alive for 32 KB of input, most of it behind the look-back
// (each L2 round trip ~1 us under full HBM load).  Throughput per SM =
// bytes-in-flight / CTA life, so the lever is bytes per CTA: 3 chunks of 4096
// int32 per tile (48 KB, 4 CTAs per SM) with ONE look-back per tile,
// resolved by a dedicated warp while the copies land.
//
//   k_filter_b   filter / filter_by / partition2/3 [+ C2's sgmSum]: "quad"
//                layout (below), count pass, warp-packed scans of per-piece
//                counts, stable compaction IN PLACE to tile-local slots (an
//                element's output slot never lies after its input slot)
//                while the look-back resolves the base, then the run leaves
//                with 16-byte stores (C2: phase-shifted to the base and
//                written by 1-D bulk stores while the sgmSum passes run).
//   k_segsum_b   sgmSum over an array (C2's zs = sgmSum flags ys): flags are
//                bits of the mkFlags bitmap at the element's own position, so
//                they are fetched together with the data; the segmented
//                aggregate of the tile takes the look-back; every thread
//                writes its 16 results with two 256-bit stores.
//
// k_segsum_b's shared-memory layout gives a thread 16 consecutive elements:
// int32 full tiles are TMA-loaded into a linear buffer and read with an XOR
// rotation of the piece order (lin_read_xor: a quarter-warp's LDS.128 hit 8
// distinct bank groups); int64 and ragged tiles use per-lane cp.async with
// the same swizzle applied on the copy side.
#pragma once
#include "k_stream.cuh"

namespace ixg {

// 8 worker warps + the look-back warp, 3 chunks of 4096 int32 per tile
// (48 KB), 4 CTAs per SM: measured 4-5 % faster than 16 warps / 96 KB
// tiles / 2 CTAs per SM on filter, C2 and partition (more CTAs overlap the
// load, scan and store phases).
#ifndef IXG_BW
#define IXG_BW 8
#endif
constexpr int kBW = IXG_BW;             // worker warps
constexpr int kBT = kBW * 32;           // worker threads
constexpr int kBChunk = kBT * kSItems;  // elements per chunk
#ifndef IXG_MINB
#define IXG_MINB (kBW >= 16 ? 2 : 4)
#endif
constexpr int kBMinBlocks = IXG_MINB;  // resident CTAs per SM the registers must allow
#ifndef IXG_CH32
#define IXG_CH32 3  // chunks per int32 tile (48 KB, 4 CTAs/SM)
#endif
#ifndef IXG_CH64
#define IXG_CH64 2  // chunks per int64 tile (64 KB, 3 CTAs/SM): filter i64 0.347 -> 0.290 ms at 2^27
#endif
// resident CTAs per SM of a big-tile kernel over T (shared memory: 4 x 48 KB
// for int32; int64 tiles of IXG_CH64 x 32 KB)
template <typename T>
constexpr int big_min_blocks() {
  return sizeof(T) == 4 ? (IXG_CH32 <= 3 ? kBMinBlocks : 3) : (IXG_CH64 == 1 ? kBMinBlocks : 3);
}
#ifndef IXG_BULK_ST
#define IXG_BULK_ST 1  // C2: ys / zs leave as bulk (TMA) stores of the phase-shifted run (0.502 -> 0.481 ms)
#endif
#ifndef IXG_BULK_ALL
#define IXG_BULK_ALL 0  // int32 filter / partition too (measured 1 % slower; int64 always: 1 % faster)
#endif
#ifndef IXG_P1_UNROLL
#define IXG_P1_UNROLL 4
#endif
#ifndef IXG_P2_UNROLL
#define IXG_P2_UNROLL 8  // measured 0.5 % faster than 4 on C2
#endif
constexpr int kP1Unroll = IXG_P1_UNROLL, kP2Unroll = IXG_P2_UNROLL;
#ifndef IXG_SEGSUM_TMA64
#define IXG_SEGSUM_TMA64 1  // k_segsum_b int64: TMA linear tiles + lin_read_xor64
#endif
#ifndef IXG_SCAN32_CH
#define IXG_SCAN32_CH 4  // k_segsum_b<int32, int64> (scan (+) of int32): 64 KB tiles, 0.606 -> 0.590 ms at 2^28
#endif
// chunks per tile of k_segsum_b<T, Z> (0 = Big's default)
template <typename T, typename Z>
constexpr int kSegsumCH = (sizeof(T) == 4 && sizeof(Z) == 8) ? IXG_SCAN32_CH : 0;
#ifndef IXG_LB_DEFER
#define IXG_LB_DEFER 1  // look-back polling deferred until it can succeed: C2 0.463 -> 0.458 ms, filter -0.7 %
#endif
#ifndef IXG_MKF_CH
#define IXG_MKF_CH 1  // mkFlags scan: chunks (4 K int64 shape values) per tile
#endif
#ifndef IXG_SEGSUM_RUN32
#define IXG_SEGSUM_RUN32 1  // k_segsum_b<int32, int32, SegOp>: the pass-2 run in 32 bits with an exact overflow test
#endif
#ifndef IXG_SEGSUM_BITS
#define IXG_SEGSUM_BITS 1  // k_segsum_b with a predicate-bit element (CHECKED index scans): popcount sums
#endif
#ifndef IXG_SEGSUM_WSCAN
#define IXG_SEGSUM_WSCAN 1  // k_segsum_b: the (chunk, warp) prefixes by one warp scan instead of a loop per thread
#endif
#ifndef IXG_SEGSUM_MINB
#define IXG_SEGSUM_MINB 3  // k_segsum_b: 72 registers; measured 0.313 ms vs 0.321 (4) / 0.351 (2) at k = 2^27
#endif

template <typename T, int CHO = 0>  // CHO: chunks per tile if not the default
struct Big {
  static constexpr int P = (int)sizeof(T);           // 16-byte pieces per thread block (16 elements)
  static constexpr int EP = 16 / (int)sizeof(T);     // elements per piece
  static constexpr int CH = CHO ? CHO : (sizeof(T) == 4 ? IXG_CH32 : IXG_CH64);  // chunks per tile
  static constexpr int PAD = 32 / (int)sizeof(T);    // >= the 32-byte store phase
  static constexpr int TILE = CH * kBChunk;
  static constexpr int SMEM = (PAD + TILE) * (int)sizeof(T);
  IXG_DEV static int swz(int t, int j) { return j ^ ((t * P / 8) & (P - 1)); }
  // element offset (within the buffer) of piece j of thread t in chunk c
  IXG_DEV static int piece(int c, int t, int j) { return PAD + c * kBChunk + kSItems * t + swz(t, j) * EP; }
};

IXG_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
IXG_DEV void cp_async16(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem)), "l"(gmem), "r"(src_bytes)
               : "memory");
}
IXG_DEV void cp_async16_full(uint32_t saddr, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(gmem) : "memory");
}
// mbarrier + 1-D bulk copy (TMA engine, SASS UBLKCP) helpers
IXG_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
IXG_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
IXG_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
IXG_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 1-D bulk store shared -> global (TMA engine): both addresses 16-byte
// aligned, size a multiple of 16.  The writing threads' generic-proxy smem
// stores must be fenced into the async proxy before the issuing barrier, and
// the issuer must wait for the engine's smem reads before the buffer is
// rewritten or the CTA exits.
IXG_DEV void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
IXG_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
IXG_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
IXG_DEV void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
IXG_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}
IXG_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
IXG_DEV void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// issue the copies of thread t's blocks for all chunks of the tile
template <typename T, int CHO = 0>
IXG_DEV void big_issue(T* buf, const T* __restrict__ xs, long long n, long long tile_base, int t) {
  using B = Big<T, CHO>;
  if (tile_base + B::TILE <= n) {  // full tile: no per-piece bounds
    const T* src = xs + tile_base + kSItems * t;
    const uint32_t s0 = smem_u32(buf + B::PAD + kSItems * t);
#pragma unroll
    for (int c = 0; c < B::CH; ++c)
#pragma unroll
      for (int j = 0; j < B::P; ++j)
        cp_async16_full(s0 + (uint32_t)((c * kBChunk + B::swz(t, j) * B::EP) * (int)sizeof(T)),
                        src + c * kBChunk + j * B::EP);
    cp_async_commit();
    return;
  }
#pragma unroll
  for (int c = 0; c < B::CH; ++c) {
#pragma unroll
    for (int j = 0; j < B::P; ++j) {
      const long long ge = tile_base + (long long)c * kBChunk + (long long)kSItems * t + j * B::EP;
      long long valid = (n - ge) * (long long)sizeof(T);
      valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
      cp_async16(buf + B::piece(c, t, j), valid ? (const void*)(xs + ge) : (const void*)xs, (int)valid);
    }
  }
  cp_async_commit();
}

template <typename T>
IXG_DEV void big_read(const T* buf, int c, int t, T (&x)[kSItems]) {
  using B = Big<T>;
#pragma unroll
  for (int j = 0; j < B::P; ++j) {
    const uint4 v = *reinterpret_cast<const uint4*>(buf + B::piece(c, t, j));
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int q = 0; q < B::EP; ++q) x[j * B::EP + q] = e[q];
  }
}

// Thread t's 16 consecutive int32 of chunk c from a LINEAR (TMA-loaded)
// buffer without bank conflicts: step j reads piece j ^ r, r = (t >> 1) & 3
// (the XOR swizzle of big_issue moved from the copy to the read address, so
// a quarter-warp's LDS.128 hit 8 distinct bank groups), then two conditional
// swap stages put piece k back at k.
IXG_DEV void lin_read_xor(const int32_t* buf, int c, int t, int32_t (&x)[kSItems]) {
  const int r = (t >> 1) & 3;
  const int32_t* b = buf + Big<int32_t>::PAD + c * kBChunk + kSItems * t;
  uint4 v[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = *reinterpret_cast<const uint4*>(b + 4 * (j ^ r));
  auto cswap = [](bool p, uint4& a, uint4& d) {
    const uint4 a0 = a, d0 = d;
    a = make_uint4(p ? d0.x : a0.x, p ? d0.y : a0.y, p ? d0.z : a0.z, p ? d0.w : a0.w);
    d = make_uint4(p ? a0.x : d0.x, p ? a0.y : d0.y, p ? a0.z : d0.z, p ? a0.w : d0.w);
  };
  cswap(r & 1, v[0], v[1]);
  cswap(r & 1, v[2], v[3]);
  cswap(r & 2, v[0], v[2]);
  cswap(r & 2, v[1], v[3]);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    x[4 * k] = (int32_t)v[k].x;
    x[4 * k + 1] = (int32_t)v[k].y;
    x[4 * k + 2] = (int32_t)v[k].z;
    x[4 * k + 3] = (int32_t)v[k].w;
  }
}

// The int64 twin: thread t's 16 consecutive int64 are 8 pieces; step j reads
// piece j ^ (t & 7) (a quarter-warp's LDS.128 hit 8 distinct bank groups),
// three conditional swap stages put piece k back at k.
IXG_DEV void lin_read_xor64(const long long* buf, int c, int t, long long (&x)[kSItems]) {
  const int r = t & 7;
  const long long* b = buf + Big<long long>::PAD + c * kBChunk + kSItems * t;
  uint4 v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = *reinterpret_cast<const uint4*>(b + 2 * (j ^ r));
  auto cswap = [](bool p, uint4& a, uint4& d) {
    const uint4 a0 = a, d0 = d;
    a = make_uint4(p ? d0.x : a0.x, p ? d0.y : a0.y, p ? d0.z : a0.z, p ? d0.w : a0.w);
    d = make_uint4(p ? a0.x : d0.x, p ? a0.y : d0.y, p ? a0.z : d0.z, p ? a0.w : d0.w);
  };
#pragma unroll
  for (int bit = 1; bit < 8; bit <<= 1)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (!(j & bit)) cswap(r & bit, v[j], v[j | bit]);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    x[2 * k] = (long long)(((unsigned long long)v[k].y << 32) | v[k].x);
    x[2 * k + 1] = (long long)(((unsigned long long)v[k].w << 32) | v[k].z);
  }
}

// ---------------------------------------------------------------------------
// "Quad" layout of a tile (k_filter_b): in chunk c, warp w owns elements
// [512w, 512w + 512); its lane l holds P = 16/EP pieces of EP = 16/sizeof(T)
// consecutive elements, piece k at 512w + k*32*EP + l*EP.  Every warp-wide
// cp.async / LDS.128 of piece k then covers 512 contiguous bytes: 16 full
// sectors from L2 and 4 shared-memory wavefronts, with no swizzle (the
// blocked 16-per-lane layout cost 7x the wavefronts on the copy side).  The
// compaction stores of a warp for one (piece, element) land ~EP/2 words
// apart instead of ~8, i.e. <= 2-way bank conflicts.
template <typename T>
struct Quad {
  static constexpr int EP = 16 / (int)sizeof(T);
  static constexpr int P = kSItems / EP;
  // per-piece counts, 8 bits each (a warp's piece total is <= 32*EP <= 128)
  using PK = typename std::conditional<(P <= 4), uint32_t, unsigned long long>::type;
  IXG_DEV static int off(int w, int k, int l) { return w * (32 * kSItems) + k * (32 * EP) + l * EP; }
  IXG_DEV static PK counts(uint32_t m) {
    PK v = 0;
#pragma unroll
    for (int k = 0; k < P; ++k) v |= (PK)__popc((m >> (k * EP)) & ((1u << EP) - 1u)) << (8 * k);
    return v;
  }
  IXG_DEV static int field(PK v, int k) { return (int)((v >> (8 * k)) & 0xff); }
  IXG_DEV static int field_sum(PK v) {
    int s = 0;
#pragma unroll
    for (int k = 0; k < P; ++k) s += field(v, k);
    return s;
  }
};

template <typename T, typename B = Big<T>>
IXG_DEV void quad_issue(T* buf, const T* __restrict__ xs, long long n, long long tile_base, int w, int l, bool full) {
  using Q = Quad<T>;
  const int o0 = Q::off(w, 0, l);
  if (full) {
    const T* src = xs + tile_base + o0;
    const uint32_t s0 = smem_u32(buf + B::PAD + o0);
#pragma unroll
    for (int c = 0; c < B::CH; ++c)
#pragma unroll
      for (int k = 0; k < Q::P; ++k)
        cp_async16_full(s0 + (uint32_t)((c * kBChunk + k * 32 * Q::EP) * (int)sizeof(T)),
                        src + c * kBChunk + k * 32 * Q::EP);
  } else {
#pragma unroll
    for (int c = 0; c < B::CH; ++c)
#pragma unroll
      for (int k = 0; k < Q::P; ++k) {
        const int o = c * kBChunk + o0 + k * 32 * Q::EP;
        long long valid = (n - (tile_base + o)) * (long long)sizeof(T);
        valid = valid < 0 ? 0 : (valid > 16 ? 16 : valid);
        cp_async16(buf + B::PAD + o, valid ? (const void*)(xs + tile_base + o) : (const void*)xs, (int)valid);
      }
  }
  cp_async_commit();
}

template <typename T, typename B = Big<T>>
IXG_DEV void quad_read(const T* buf, int c, int w, int l, T (&x)[kSItems]) {
  using Q = Quad<T>;
#pragma unroll
  for (int k = 0; k < Q::P; ++k) {
    const uint4 v = *reinterpret_cast<const uint4*>(buf + B::PAD + c * kBChunk + Q::off(w, k, l));
    const T* e = reinterpret_cast<const T*>(&v);
#pragma unroll
    for (int q = 0; q < Q::EP; ++q) x[k * Q::EP + q] = e[q];
  }
}

// valid bits of the lane's pieces (g0 = global index of its piece 0)
template <int EP>
IXG_DEV uint32_t quad_valid(long long n, long long g0) {
  uint32_t vm = 0;
#pragma unroll
  for (int k = 0; k < kSItems / EP; ++k) {
    const long long r = n - (g0 + k * 32 * EP);
    const int v = r <= 0 ? 0 : (r >= EP ? EP : (int)r);
    vm |= ((1u << v) - 1u) << (k * EP);
  }
  return vm;
}

// filter_by: bit k*EP + e = (cs[g0 + k*32*EP + e] != 0), bounds-checked
template <int EP>
IXG_DEV uint32_t quad_cs_mask(const uint8_t* __restrict__ cs, long long n, long long g0, bool full) {
  uint32_t mm = 0;
#pragma unroll
  for (int k = 0; k < kSItems / EP; ++k) {
    const long long g = g0 + k * 32 * EP;
    uint32_t b = 0;
    if (full && ((reinterpret_cast<uintptr_t>(cs + g) & (EP - 1)) == 0)) {
      b = EP == 4 ? *reinterpret_cast<const uint32_t*>(cs + g) : (uint32_t)*reinterpret_cast<const uint16_t*>(cs + g);
    } else {
#pragma unroll
      for (int e = 0; e < EP; ++e) b |= (g + e < n) ? (uint32_t)cs[g + e] << (8 * e) : 0u;
    }
#pragma unroll
    for (int e = 0; e < EP; ++e) mm |= (uint32_t)(((b >> (8 * e)) & 0xffu) != 0) << (k * EP + e);
  }
  return mm;
}

// Fused partition + exchange (sharded C5): the global output is sharded
// contiguously over `ranks` GPUs, `shard` elements each; dst[r] is rank r's
// shard (a peer pointer mapped over NVLink for r != this rank).  A class
// segment s of this rank's tiles starts at global seg_base[s]; seg_local[s]
// is its start on the local look-back chain.
template <typename T>
struct PeerOut {
  T* dst[8];
  long long shard;
  long long seg_base[3];
  long long seg_local[3];
  int ranks;
  // device-resident bases (no host round trip): every rank's true count,
  // all-gathered on the device; this rank's index; the input shard size
  const long long* d_counts;
  int rank;
  long long in_shard;
};

// global start of local chain position `base` of class segment `seg`:
// trues of rank r follow the trues of ranks < r, its falses follow every
// true and the falses of ranks < r
template <typename T>
IXG_DEV long long peer_gbase(const PeerOut<T>& po, int seg, long long base) {
  if (!po.d_counts) return po.seg_base[seg] + (base - po.seg_local[seg]);
  long long tb = 0, nt = 0;
  for (int r = 0; r < po.ranks; ++r) {
    const long long c = po.d_counts[r];
    nt += c;
    tb += r < po.rank ? c : 0;
  }
  if (seg == 0) return tb + base;
  return nt + ((long long)po.rank * po.in_shard - tb) + (base - po.d_counts[po.rank]);
}

// store_run to the global positions [gbase, gbase + cnt) of a sharded
// output: every 16-byte chunk lies in one shard (shard % EP == 0) and goes
// to dst[g / shard] + g % shard -- a peer store when another GPU owns it
template <typename E, int NT>
IXG_DEV void store_run_peer(const PeerOut<E>& po, long long gbase, int cnt, const E* buf) {
  constexpr int EP = 16 / (int)sizeof(E);
  if (cnt <= 0) return;
  const long long c0 = gbase / EP;
  const int s = (int)(gbase - c0 * EP);
  const int nch = (int)((gbase + cnt - 1) / EP - c0) + 1;
  const int sw = ((EP - s) % EP) * (int)sizeof(E) / 4;
  for (int j = threadIdx.x; j < nch; j += NT) {
    const int l = j * EP - s;
    const long long g = (c0 + j) * EP;
    const long long r = g / po.shard;
    E* dst = po.dst[r] + (g - r * po.shard);
    if (l >= 0 && l + EP <= cnt) {
      uint4 v;
      if (sw == 0) {
        v = *reinterpret_cast<const uint4*>(buf + l);
      } else {
        const uint4 a = *reinterpret_cast<const uint4*>(buf + l - (EP - s));
        const uint4 b = *reinterpret_cast<const uint4*>(buf + l + s);
        if (sw == 1) v = make_uint4(a.y, a.z, a.w, b.x);
        else if (sw == 2) v = make_uint4(a.z, a.w, b.x, b.y);
        else v = make_uint4(a.w, b.x, b.y, b.z);
      }
      asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(v.x), "r"(v.y),
                   "r"(v.z), "r"(v.w)
                   : "memory");
    } else {
#pragma unroll
      for (int e = 0; e < EP; ++e)
        if (l + e >= 0 && l + e < cnt) dst[e] = buf[l + e];
    }
  }
}

// One WARP stores one contiguous run of shared memory (starting at any
// element) to the global positions [gbase, gbase + cnt) of the sharded
// output: 16-byte pieces funnel-shifted from the two aligned 16-byte words
// each straddles (the shift is uniform over the run).  r0 = gbase / shard
// when the run is no longer than a shard (one shard edge at most: two
// precomputed bases), else -1 (a division per piece).
// One WARP stores one contiguous run of shared memory (starting at any
// element) to the global positions [gbase, gbase + cnt) of the sharded
// output: 16-byte pieces funnel-shifted from the two aligned 16-byte words
// each straddles (the shift is uniform over the run).  r0 = gbase / shard
// when the run is no longer than a shard (one shard edge at most: two
// precomputed bases), else -1 (a division per piece).  (Specialising the
// interior pieces of a single-shard run -- no per-piece shard or bounds
// logic -- cut the kernel's instructions by a quarter but not its time:
// past this point it waits on memory latency, and the extra registers
// spilled.)
template <typename E>
IXG_DEV void store_run_peer_w(const PeerOut<E>& po, long long gbase, int cnt, const E* run, long long r0) {
  constexpr int EP = 16 / (int)sizeof(E);
  if (cnt <= 0) return;
  const int lane = lane_id();
  const long long c0 = gbase / EP;
  const int s = (int)(gbase - c0 * EP);
  const int nch = (int)((gbase + cnt - 1) / EP - c0) + 1;
  const int o = (int)((smem_u32(run) & 15u) / sizeof(E));  // run's element offset in its 16-byte word
  const E* al = run - o;
  const int sw = ((o - s + EP) % EP) * (int)sizeof(E) / 4;
  E* p0 = nullptr;
  E* p1 = nullptr;
  long long edge = 0;
  if (r0 >= 0) {  // dst(g) = (g < edge ? p0 : p1) + g
    edge = (r0 + 1) * po.shard;
    p0 = po.dst[r0] - r0 * po.shard;
    p1 = r0 + 1 < po.ranks ? po.dst[r0 + 1] - edge : p0;
  }
  for (int j = lane; j < nch; j += 32) {
    const int l = j * EP - s;
    const long long g = (c0 + j) * EP;
    E* dst;
    if (r0 >= 0) {
      dst = (g < edge ? p0 : p1) + g;
    } else {
      const long long r = g / po.shard;
      dst = po.dst[r] + (g - r * po.shard);
    }
    if (l >= 0 && l + EP <= cnt) {
      const int a0 = (o + l) & ~(EP - 1);
      const uint4 a = *reinterpret_cast<const uint4*>(al + a0);
      uint4 v = a;
      if (sw) {
        const uint4 b = *reinterpret_cast<const uint4*>(al + a0 + EP);
        if (sw == 1) v = make_uint4(a.y, a.z, a.w, b.x);
        else if (sw == 2) v = make_uint4(a.z, a.w, b.x, b.y);
        else v = make_uint4(a.w, b.x, b.y, b.z);
      }
      asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(v.x), "r"(v.y),
                   "r"(v.z), "r"(v.w)
                   : "memory");
    } else {
#pragma unroll
      for (int e = 0; e < EP; ++e)
        if (l + e >= 0 && l + e < cnt) dst[e] = run[l + e];
    }
  }
}

// CTA-wide exclusive scan of warp-uniform packed counts (3 x 21 bits):
// returns the exclusive prefix of the calling warp, *total = CTA totals
IXG_DEV unsigned long long cta_warp_exclusive3(unsigned long long v, unsigned long long* s_w,
                                               unsigned long long* total) {
  const int lane = lane_id(), w = warp_id();
  if (lane == 0) s_w[w] = v;
  bar_sync(1, kBT);
  unsigned long long x = lane < kBW ? s_w[lane] : 0ull;
#pragma unroll
  for (int d = 1; d < kBW; d <<= 1) {
    const unsigned long long o = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += o;
  }
  const unsigned long long pre = __shfl_sync(0xffffffffu, x, (w + 31) & 31);
  *total = __shfl_sync(0xffffffffu, x, kBW - 1);
  return w ? pre : 0ull;
}

// Store the run buf[0 .. cnt) (tile-local slots, 16-byte aligned buffer) to
// out[base ..]: thread j writes the j-th 16-byte chunk of out the run
// touches.  With base not chunk-aligned the chunk's elements straddle two
// aligned chunks of buf; the word offset is CTA-uniform, so the funnel is a
// uniform switch.  Consecutive lanes read consecutive 16-byte chunks of buf
// (conflict-free) and write consecutive 16-byte chunks of out.
template <typename E, int NT>
IXG_DEV void store_run(E* __restrict__ out, long long base, int cnt, const E* buf) {
  constexpr int EP = 16 / (int)sizeof(E);
  if (cnt <= 0) return;
  const long long c0 = base / EP;
  const int s = (int)(base - c0 * EP);                    // misalignment in elements
  const int nch = (int)((base + cnt - 1) / EP - c0) + 1;  // chunks of out touched
  const int sw = ((EP - s) % EP) * (int)sizeof(E) / 4;    // word offset of l in its aligned chunk
  for (int j = threadIdx.x; j < nch; j += NT) {
    const int l = j * EP - s;  // local index of the chunk's first element
    E* dst = out + (c0 + j) * EP;
    if (l >= 0 && l + EP <= cnt) {
      uint4 v;
      if (sw == 0) {
        v = *reinterpret_cast<const uint4*>(buf + l);
      } else {
        const uint4 a = *reinterpret_cast<const uint4*>(buf + l - (EP - s));
        const uint4 b = *reinterpret_cast<const uint4*>(buf + l + s);
        if (sw == 1) v = make_uint4(a.y, a.z, a.w, b.x);
        else if (sw == 2) v = make_uint4(a.z, a.w, b.x, b.y);
        else v = make_uint4(a.w, b.x, b.y, b.z);
      }
      asm volatile("st.global.L1::no_allocate.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(dst), "r"(v.x), "r"(v.y),
                   "r"(v.z), "r"(v.w)
                   : "memory");
    } else {
#pragma unroll
      for (int e = 0; e < EP; ++e)
        if (l + e >= 0 && l + e < cnt) dst[e] = buf[l + e];
    }
  }
}

// Move the run buf[0 .. cnt) up by s < EP slots (s = the output base's
// misalignment in elements), so that run element j sits at buf + s + j and
// shares its 16-byte phase with out + base + j: the aligned middle of the run
// can then leave in one bulk store.  New 16-byte chunk c is old chunks c-1
// and c funnelled by s; rounds of 2 * NT chunks run from the top down, each
// reading (before its barrier) everything it overwrites and the old chunk
// below it, which the next round rewrites only after that barrier.
template <typename T, int NT>
IXG_DEV void shift_run_up(T* buf, int cnt, int s) {
  constexpr int EP = 16 / (int)sizeof(T);
  constexpr int PER = 2;
  const int nnew = (cnt + s + EP - 1) / EP;  // chunks of the moved run
  uint4* b4 = reinterpret_cast<uint4*>(buf);
  const int sw = s * (int)sizeof(T) / 4;  // word shift 1..3
  IXG_TR(16);
  for (int top = nnew; top > 0; top -= PER * NT) {
    uint4 v[PER];
    int cidx[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int c = top - PER * NT + i * NT + (int)threadIdx.x;
      cidx[i] = c;
      if (c >= 0) {
        const uint4 hi = b4[c];
        const uint4 lo = c > 0 ? b4[c - 1] : make_uint4(0u, 0u, 0u, 0u);
        if (sw == 1) v[i] = make_uint4(lo.w, hi.x, hi.y, hi.z);
        else if (sw == 2) v[i] = make_uint4(lo.z, lo.w, hi.x, hi.y);
        else v[i] = make_uint4(lo.y, lo.z, lo.w, hi.x);
      }
    }
    bar_sync(1, NT);
    IXG_TR(17);
#pragma unroll
    for (int i = 0; i < PER; ++i)
      if (cidx[i] >= 0) b4[cidx[i]] = v[i];
  }
}

// Store run[0 .. cnt) (run = buf + s, phase-matched to out + base) to
// out[base ..]: the aligned middle as one bulk store issued by thread 0
// (after every thread's fence + the caller's barrier), the <= EP-1 head and
// tail elements by plain stores.  Returns with the bulk store in flight.
template <typename E, int NT>
IXG_DEV void store_run_bulk(E* __restrict__ out, long long base, int cnt, const E* run) {
  constexpr int EP = 16 / (int)sizeof(E);
  if (cnt <= 0) return;
  const int a0 = min(cnt, (int)((EP - (base & (EP - 1))) & (EP - 1)));  // first aligned element
  const int a1 = max(a0, (int)(((base + cnt) & ~(long long)(EP - 1)) - base));  // end of the aligned part
  const int t = (int)threadIdx.x;
  if (t == 0 && a1 > a0) {
    bulk_s2g(out + base + a0, run + a0, (uint32_t)(a1 - a0) * (uint32_t)sizeof(E));
    bulk_commit();
  }
  if (t >= 32 && t < 32 + a0) out[base + (t - 32)] = run[t - 32];
  if (t >= 64 && t < 64 + (cnt - a1)) out[base + a1 + (t - 64)] = run[a1 + (t - 64)];
}

// CTA-wide exclusive scan over SegOp values (C2's tile-local segmented scan);
// one named barrier over the kBT workers, *total = the CTA aggregate
IXG_DEV SegOp::T cta_seg_exclusive(SegOp::T a, SegOp::T* s_seg, SegOp::T* total) {
  const int lane = lane_id(), w = warp_id();
  const SegOp::T inc = warp_inclusive<SegOp>(a);
  SegOp::T lex = SegOp::shfl_up(inc, 1);
  if (lane == 0) lex = SegOp::identity();
  if (lane == 31) s_seg[w] = inc;
  bar_sync(1, kBT);
  SegOp::T x = lane < kBW ? s_seg[lane] : SegOp::identity();
#pragma unroll
  for (int d = 1; d < kBW; d <<= 1) {
    const SegOp::T o = SegOp::shfl_up(x, d);
    if (lane >= d) x = SegOp::op(o, x);
  }
  SegOp::T pre = SegOp::shfl(x, (w + 31) & 31);
  if (w == 0) pre = SegOp::identity();
  *total = SegOp::shfl(x, kBW - 1);
  return SegOp::op(pre, lex);
}

// per-chunk counts packed into 64 bits: CH fields of 64 / CH bits (a chunk's
// CTA total is <= kBChunk = 4096 < 2^16)
template <int CH>
IXG_DEV int fieldc(unsigned long long v, int c) {
  constexpr int W = 64 / CH;
  return (int)((v >> (W * c)) & (W >= 64 ? ~0ull : ((1ull << W) - 1ull)));
}

// ---------------------------------------------------------------------------
// kSeg (C2, Z the width of zs == sizeof(T)): after ys is stored, the
// compacted run still in shared memory is scanned again for zs = sgmSum
// flags ys with flags at the output positions (bits out_base + base + q of
// the mkFlags bitmap), first with a TILE-LOCAL carry; the tile's segmented
// aggregate goes on a second look-back chain, whose result (the carry of
// the preceding tiles) is added to the values before the tile's first flag
// just before zs is stored.
//
// NS > 1 (partition2 / partition3, ELIDED): the grid is NS segments of
// seg_tiles tiles over the same xs, segment s selecting class s (p; not p
// [and q]; not p and not q), all on ONE look-back chain -- so the chain's
// prefix is the class's output position and the whole stable partition is
// a single pass writing each element once (d_count[s] = the prefix at the
// end of segment s, for s < NS - 1).
template <typename T, bool kByCs, bool kSeg = false, typename Z = T, int NS = 1, bool kPeer = false, int CHO = 0>
__global__ void __launch_bounds__(kBT + 32, big_min_blocks<T>()) k_filter_b(const T* __restrict__ xs, const uint8_t* __restrict__ cs,
                                                          long long n, ixg_pred p, T* __restrict__ ys, LBChan ch,
                                                          uint32_t nonce, long long* d_count,
                                                          Z* __restrict__ zs = nullptr,
                                                          const uint32_t* __restrict__ segbits = nullptr,
                                                          long long out_base = 0, LBChan ch2 = LBChan{nullptr, nullptr},
                                                          ixg_status* st = nullptr, ixg_pred q = ixg_pred{},
                                                          long long seg_tiles = 0, PeerOut<T> po = PeerOut<T>{}) {
  static_assert(!kSeg || sizeof(Z) == sizeof(T), "zs is computed in place of ys");
  constexpr bool kDual = kPeer && NS == 1;  // one pass placing both classes (the count is known)
  using B = Big<T, CHO>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw);
  __shared__ SegOp::T s_seg[kBW];
  __shared__ unsigned long long s_w[kBW];
  __shared__ int s_cnt;
  __shared__ long long s_excl;
  __shared__ SegOp::T s_tagg, s_carry;
  __shared__ __align__(8) uint64_t s_mbar[B::CH];
  // kSeg: the mkFlags bitmap words of the tile's output range, fetched by
  // the look-back warp the moment the base is known
  constexpr int kBitsW = kSeg ? ((B::TILE + 31) / 32 + 8 + 3) & ~3 : 4;
  __shared__ __align__(16) uint32_t s_bits[kBitsW];
  __shared__ __align__(8) uint64_t s_mbar_bits;
  __shared__ long long s_wbase;

  const long long tile = blockIdx.x;  // position on the look-back chain
  const int seg = NS > 1 ? (int)(tile / seg_tiles) : 0;
  const long long tile_base = (NS > 1 ? tile - seg * seg_tiles : tile) * B::TILE;
  const int t = threadIdx.x;
  // PDL (launch_filter_b): the next kernel of the stream may be scheduled
  // now; this one waits for its predecessor before touching anything the
  // predecessor writes -- the look-back slots (shared by consecutive
  // launches on one workspace) and outputs at once, except C2 (kSeg), whose
  // predecessor is the mkFlags scan: only the bitmap depends on it, so the
  // tile's load, count and compaction overlap the scan's tail
  pdl_trigger();
  if constexpr (!kSeg) pdl_wait();
  if (warp_id() == kBW) {  // look-back warp
    if (kSeg && lane_id() == 0) {
      mbar_init(&s_mbar_bits, 1);
      mbar_fence_init();
    }
    long long ex = 0;
    // IXG_LB_DEFER: start polling once this tile's own count is published
    // (its predecessors' are then mostly published too: fewer spins
    // stealing issue slots from the workers)
    if (IXG_LB_DEFER && sizeof(T) == 4) bar_sync(4, 64);  // int64: measured 0.5 % slower
    if (tile > 0) ex = lb_lookback<SumOp>(ch, nonce, tile).v;
    if (lane_id() == 0) {
      s_excl = ex;
      if constexpr (kSeg) {
        // bitmap words [wb, wb + kBitsW) cover flags out_base + ex .. + TILE
        // (bitmap_bytes() pads the bitmap past its last word)
        const long long wb = ((out_base + ex) >> 5) & ~3LL;
        s_wbase = wb;
        pdl_wait();  // the mkFlags scan (the predecessor) has written the bitmap
        mbar_expect_tx(&s_mbar_bits, kBitsW * 4u);
        bulk_g2s(s_bits, segbits + wb, kBitsW * 4u, &s_mbar_bits);
      }
    }
    __syncwarp();
#ifdef IXG_TRACE
    unsigned long long t5__;
    IXG_TR_NOW(t5__);  // every lane: a divergent trace store here would let the warp's other lanes
                       // complete the (per-warp counted) barrier early
#endif
    bar_sync(2, kBT + 32);
#ifdef IXG_TRACE
    if (lane_id() == 0 && blockIdx.x < (1u << 17)) g_trace[blockIdx.x * IXG_TRS + 5] = t5__;
#endif
    if (lane_id() == 0) {
      const int cnt = s_cnt;
      if (tile > 0) lb_publish<SumOp>(ch, nonce, tile, SumOp::T{ex + cnt}, true);
      if (NS == 1 ? tile == (long long)gridDim.x - 1 : (seg < NS - 1 && tile == (seg + 1) * seg_tiles - 1))
        d_count[seg] = ex + cnt;
    }
    if constexpr (kSeg) {
      // second chain: the sgmSum carry into the tile (SegOp over the tiles'
      // segmented aggregates), polled while the workers store ys and scan
      SegOp::T carry = SegOp::identity();
      if (IXG_LB_DEFER) bar_sync(5, kBT + 32);  // the workers' pass 1 is done
      if (tile > 0) carry = lb_lookback<SegOp>(ch2, nonce, tile);
      if (lane_id() == 0) s_carry = carry;
      IXG_TR_LANE0(12);
      bar_sync(3, kBT + 32);
      const SegOp::T a = s_tagg;
      if (lane_id() == 0 && tile > 0 && !a.f) lb_publish<SegOp>(ch2, nonce, tile, SegOp::op(carry, a), true);
    }
    return;
  }
  IXG_TR(0);
  using Q = Quad<T>;
  const int w = warp_id(), l = lane_id();
  const bool full = tile_base + B::TILE <= n;
  // full tiles: one bulk (TMA) copy per chunk issued by one thread, landing
  // on the chunk's mbarrier (no per-lane copies, no LSU wavefronts); the
  // ragged last tile uses per-lane cp.async with zero fill
  if (full) {
    if (t == 0) {
#pragma unroll
      for (int c = 0; c < B::CH; ++c) mbar_init(&s_mbar[c], 1);
      mbar_fence_init();
#pragma unroll
      for (int c = 0; c < B::CH; ++c) {
        mbar_expect_tx(&s_mbar[c], kBChunk * (uint32_t)sizeof(T));
        bulk_g2s(buf + B::PAD + c * kBChunk, xs + tile_base + c * kBChunk, kBChunk * (uint32_t)sizeof(T), &s_mbar[c]);
      }
    }
    bar_sync(1, kBT);  // the mbarriers are initialised
  } else {
    quad_issue<T, B>(buf, xs, n, tile_base, w, l, false);
  }
  // selection masks of the lane's pieces (bit k*EP + e), filter_by reads cs meanwhile
  uint32_t m[B::CH];
  if (kByCs) {
#pragma unroll
    for (int c = 0; c < B::CH; ++c) m[c] = quad_cs_mask<Q::EP>(cs, n, tile_base + c * kBChunk + Q::off(w, 0, l), full);
    if (!full) cp_async_wait_all();
  } else {
    const Selector<T, (NS < 3)> sel(p);  // partition3: the sign test measured 3 % slower
    if (!full) cp_async_wait_all();
#pragma unroll
    for (int c = 0; c < B::CH; ++c) {
      if (full) mbar_wait(&s_mbar[c], 0);
      T x[kSItems];
      quad_read<T, B>(buf, c, w, l, x);
      m[c] = sel.mask(x);
      if constexpr (NS == 2) {
        if (seg == 1) m[c] ^= 0xffffu;
      } else if constexpr (NS == 3) {
        if (seg > 0) {
          const uint32_t mq = Selector<T, false>(q).mask(x);
          m[c] = ~m[c] & (seg == 1 ? mq : ~mq) & 0xffffu;
        }
      }
      if (!full) m[c] &= quad_valid<Q::EP>(n, tile_base + c * kBChunk + Q::off(w, 0, l));
    }
  }
  IXG_TR(1);
  // per-piece counts packed 8 bits per piece, scanned across the warp:
  // order within a chunk is (warp, piece, lane)
  typename Q::PK ex[B::CH], wt[B::CH];
  unsigned long long packed = 0;
#pragma unroll
  for (int c = 0; c < B::CH; ++c) {
    const typename Q::PK v = Q::counts(m[c]);
    typename Q::PK inc = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const typename Q::PK o = __shfl_up_sync(0xffffffffu, inc, d);
      if (l >= d) inc += o;
    }
    wt[c] = __shfl_sync(0xffffffffu, inc, 31);
    ex[c] = inc - v;
    packed |= (unsigned long long)Q::field_sum(wt[c]) << ((64 / B::CH) * c);
  }
  unsigned long long tot;
  const unsigned long long exw = cta_warp_exclusive3(packed, s_w, &tot);
  IXG_TR(2);
  int cnt = 0, before[B::CH];
#pragma unroll
  for (int c = 0; c < B::CH; ++c) {
    before[c] = cnt + fieldc<B::CH>(exw, c);
    cnt += fieldc<B::CH>(tot, c);
  }
  if (t == 0) {
    s_cnt = cnt;
    lb_publish<SumOp>(ch, nonce, tile, SumOp::T{cnt}, tile == 0);
  }
  if (IXG_LB_DEFER && sizeof(T) == 4 && w == 0) {
    __syncwarp();
    bar_arrive(4, 64);
  }
  // in-place stable compaction to TILE-LOCAL slots, chunk by chunk, while
  // the look-back warp resolves the tile's global base: output slot r of an
  // element never exceeds its input slot PAD + i, and chunk c's outputs end
  // before chunk c+1's inputs begin
  // kDual (the sharded partition2, true counts of every rank known
  // beforehand): each chunk is partitioned IN PLACE within its own slots --
  // trues first, then falses, both stable -- after every worker has read it,
  // so the tile's xs is read once and both classes leave from shared memory
  // as 2 x CH runs (8 B per element instead of the two-segment form's 12)
  int bcc = 0;  // trues of the tile's earlier chunks
#pragma unroll
  for (int c = 0; c < B::CH; ++c) {
    if (kByCs && full) mbar_wait(&s_mbar[c], 0);
    T x[kSItems];
    quad_read<T, B>(buf, c, w, l, x);
    bar_sync(1, kBT);
    const uint32_t mc = m[c];
    int pre = before[c];  // + totals of the warp's earlier pieces
    if constexpr (kDual) {
      uint32_t vc = 0xffffu;
      if (!full) vc = quad_valid<Q::EP>(n, tile_base + c * kBChunk + Q::off(w, 0, l));
      T* const cb = buf + B::PAD + c * kBChunk;
      const int tc = fieldc<B::CH>(tot, c);
#pragma unroll
      for (int k = 0; k < Q::P; ++k) {
        int r = pre - bcc + Q::field(ex[c], k);  // chunk-local trues before the piece
        pre += Q::field(wt[c], k);
        const int i0 = Q::off(w, k, l);  // the piece's first chunk index
#pragma unroll
        for (int e = 0; e < Q::EP; ++e) {
          const uint32_t bit = 1u << (k * Q::EP + e);
          if (mc & bit) cb[r++] = x[k * Q::EP + e];
          else if (vc & bit) cb[tc + (i0 + e - r)] = x[k * Q::EP + e];
        }
      }
      bcc += tc;
    } else {
#pragma unroll
      for (int k = 0; k < Q::P; ++k) {
        const int tb0 = pre + Q::field(ex[c], k);  // trues before the piece
        T* dst = buf + tb0;
        pre += Q::field(wt[c], k);
#pragma unroll
        for (int e = 0; e < Q::EP; ++e)
          if (mc & (1u << (k * Q::EP + e))) *dst++ = x[k * Q::EP + e];
      }
    }
  }
  IXG_TR(3);
#ifdef IXG_TRACE
  __shared__ unsigned long long s_arr__[kBW];  // each worker warp's arrival at bar 2
  {
    unsigned long long ta__;
    IXG_TR_NOW(ta__);
    if (l == 0) s_arr__[w] = ta__;
  }
#endif
  bar_sync(2, kBT + 32);  // base resolved; every worker's compaction done
  IXG_TR(4);
#ifdef IXG_TRACE
  if (t == 0 && blockIdx.x < (1u << 17)) {
    unsigned long long mx = 0, mn = ~0ull;
    for (int q = 0; q < kBW; ++q) {
      mx = s_arr__[q] > mx ? s_arr__[q] : mx;
      mn = s_arr__[q] < mn ? s_arr__[q] : mn;
    }
    g_trace[blockIdx.x * IXG_TRS + 18] = mx;
    g_trace[blockIdx.x * IXG_TRS + 19] = mn;
  }
#endif
  const long long base = s_excl;
  // kSeg: thread t scans the output piece [q0, q1) of odd length L (L <= 49
  // outputs: its flags span <= 3 bitmap words); the L2 loads of those words
  // are issued now and land during the ys stores
  int L = 0, q0 = 0, q1 = 0;
  long long g0 = 0;
  if constexpr (kSeg) {
    L = ((cnt + kBT - 1) / kBT) | 1;
    q0 = min(t * L, cnt);
    q1 = min(q0 + L, cnt);
    g0 = out_base + base + q0;
  }
  // kSeg + IXG_BULK_ST: the ys run is phase-shifted to base and leaves as
  // one bulk (TMA) store that drains while the workers scan zs
  constexpr bool kBulk = (kSeg && IXG_BULK_ST) || (!kSeg && !kPeer && (IXG_BULK_ALL || sizeof(T) == 8));
  const bool bulk = kBulk && ((((uintptr_t)ys) | (kSeg ? (uintptr_t)zs : (uintptr_t)0)) & 15) == 0;  // 16-byte aligned outputs
  T* run = buf;
  if constexpr (kDual) {
    // 2 x CH sub-runs (chunk c's trues, then its falses), one worker warp
    // each: a warp's loop runs ~16 pieces per lane with its setup done once
    static_assert(2 * B::CH <= kBW, "one worker warp per sub-run");
    const int w = warp_id();
    if (w < 2 * B::CH) {
      const int c = w >> 1, cls = w & 1;
      int pre = 0, tc_c = 0, nv_c = 0;
#pragma unroll
      for (int q = 0; q < B::CH; ++q) {
        const long long left = n - tile_base - (long long)q * kBChunk;
        const int nv = left <= 0 ? 0 : (left >= kBChunk ? kBChunk : (int)left);
        const int tc = fieldc<B::CH>(tot, q);
        if (q < c) pre += cls ? nv - tc : tc;
        if (q == c) {
          tc_c = tc;
          nv_c = nv;
        }
      }
      const long long g0 =
          cls ? peer_gbase(po, 1, po.d_counts[po.rank] + (tile_base - base)) + pre  // the tile's falses
              : peer_gbase(po, 0, base) + pre;                                       // its trues
      const int len = cls ? nv_c - tc_c : tc_c;
      // a sub-run is <= a chunk: with shards of >= a chunk, one division per warp
      store_run_peer_w<T>(po, g0, len, buf + B::PAD + c * kBChunk + (cls ? tc_c : 0),
                          po.shard >= kBChunk ? g0 / po.shard : -1);
    }
  } else if constexpr (kPeer) {
    store_run_peer<T, kBT>(po, peer_gbase(po, seg, base), cnt, buf);
  } else if (bulk) {
    const int sh0 = (int)(base & (B::EP - 1));
    if (sh0) {
      shift_run_up<T, kBT>(buf, cnt, sh0);
      run = buf + sh0;
    }
    IXG_TR(14);
    fence_async_smem();
    bar_sync(1, kBT);
    IXG_TR(15);
    store_run_bulk<T, kBT>(ys, base, cnt, run);
    if (!kSeg && t == 0) bulk_wait_read0();  // before the CTA's smem is released
  } else {
    store_run<T, kBT>(ys, base, cnt, buf);
  }
  IXG_TR(6);
  if constexpr (kSeg) {
    // thread t scans the run piece [q0, q1) of odd length L (odd stride:
    // the scalar shared-memory reads of a warp hit 32 distinct banks)
    uint32_t bw0 = 0, bw1 = 0, bw2 = 0;
    mbar_wait(&s_mbar_bits, 0);  // the look-back warp's bitmap window has landed
    if (q1 > q0) {
      const int wd = (int)((g0 >> 5) - s_wbase);
      bw0 = s_bits[wd];
      bw1 = s_bits[wd + 1];
      bw2 = s_bits[wd + 2];
    }
    const int sh = (int)(g0 & 31);
    uint64_t fw = ((((uint64_t)bw1 << 32) | bw0) >> sh) | (sh ? ((uint64_t)bw2 << (64 - sh)) : 0ull);
    const int len = q1 - q0;
    const uint64_t lenmask = len >= 64 ? ~0ull : ((1ull << len) - 1ull);
    fw &= lenmask;
    // pass 1: the piece's segmented aggregate
    const int last = fw ? 63 - __clzll(fw) : 0;
    long long s = 0;
#pragma unroll kP1Unroll
    for (int j = last; j < len; ++j) s += (long long)run[q0 + j];
    // tile-local exclusive prefix of the piece (its barrier also orders
    // every thread's ys stores from buf -- and the bulk store's smem reads,
    // waited for by its issuer -- before zs overwrites it)
    if (bulk && t == 0) bulk_wait_read0();
    SegOp::T tagg;
    const SegOp::T init = cta_seg_exclusive(SegOp::T{s, fw != 0}, s_seg, &tagg);
    IXG_TR(8);
    if (t == 0) {  // a tile with a flag knows its inclusive value already
      s_tagg = tagg;
      lb_publish<SegOp>(ch2, nonce, tile, tagg, tile == 0 || tagg.f);
    }
    if (IXG_LB_DEFER) {
      __syncwarp();
      bar_arrive(5, kBT + 32);
    }
    // pass 2: zs in place of ys.  Values at or after the tile's first flag
    // are final; the earlier ones (j < jm) are tile-local until the carry of
    // the preceding tiles arrives, so they run exactly in 64 bits and keep
    // their range [lo, hi] for the check once the carry is known.
    Z* zbuf = reinterpret_cast<Z*>(run) + q0;
    const int jf = init.f ? 0 : (fw ? __ffsll((long long)fw) - 1 : len);
    const int jm = jf < len ? jf : len;
    uint64_t fb = fw >> jm;
    long long lo = LLONG_MAX, hi = LLONG_MIN;
    {
      long long r = init.v;
      for (int j = 0; j < jm; ++j) {  // no flags here
        r += (long long)zbuf[j];
        lo = r < lo ? r : lo;
        hi = r > hi ? r : hi;
        zbuf[j] = (Z)r;
      }
    }
    int j = jm;
    if constexpr (sizeof(Z) == 4) {
      // 32-bit modular run from the first flag on (or from an exact final
      // init): a value leaves int32 iff its add overflows
      int32_t r = (int32_t)init.v;
      uint32_t ov = 0;
#pragma unroll kP2Unroll
      for (; j < len; ++j, fb >>= 1) {
        const int32_t x = (int32_t)zbuf[j];
        const int32_t rr = (fb & 1ull) ? 0 : r;
        const int32_t nr = (int32_t)((uint32_t)rr + (uint32_t)x);
        ov |= (uint32_t)((rr ^ nr) & (x ^ nr));
        zbuf[j] = (Z)nr;
        r = nr;
      }
      if ((int32_t)ov < 0 && st) atomicOr(&st->flags, IXG_F_NARROW);
    } else {
      // 64-bit run from the first flag on: the exact check of each
      // sequential step (the reference's ints are unbounded)
      long long r = init.v;
      bool ov = false;
      int jo = len;
      for (; j < len; ++j, fb >>= 1) {
        const long long x = (long long)zbuf[j];
        const long long rr = (fb & 1ull) ? 0LL : r;
        r = (long long)((unsigned long long)rr + (unsigned long long)x);
        if (!ov && ((rr ^ r) & (x ^ r)) < 0) {
          ov = true;
          jo = j;
        }
        zbuf[j] = (Z)r;
      }
      if (ov) status_overflow(st, 0, base + q0 + jo);
    }
    IXG_TR(9);
    bar_sync(3, kBT + 32);  // carry of the preceding tiles
    IXG_TR(10);
    if (jm > 0) {
      const long long cv = s_carry.v;
      if (sizeof(Z) == 4 && st && (cv + lo < (long long)INT32_MIN || cv + hi > (long long)INT32_MAX))
        atomicOr(&st->flags, IXG_F_NARROW);
      if constexpr (sizeof(Z) == 8) {
        // the values before the piece's first flag get the carry now: check
        // each sequential step (x_j = local_j - local_{j-1}, all wrapped)
        long long prevl = init.v;
        for (int q = 0; q < jm; ++q) {
          const long long loc = (long long)zbuf[q];
          const long long x = (long long)((unsigned long long)loc - (unsigned long long)prevl);
          const long long fin = (long long)((unsigned long long)loc + (unsigned long long)cv);
          prevl = loc;
          zbuf[q] = (Z)fin;
          if (step_ovf(fin, x)) {
            status_overflow(st, 0, base + q0 + q);
            for (++q; q < jm; ++q) zbuf[q] = (Z)((unsigned long long)zbuf[q] + (unsigned long long)cv);
            break;
          }
        }
      } else {
        for (int q = 0; q < jm; ++q) zbuf[q] = (Z)((unsigned long long)zbuf[q] + (unsigned long long)cv);
      }
    }
    if (bulk) {
      fence_async_smem();
      bar_sync(1, kBT);
      store_run_bulk<Z, kBT>(zs, base, cnt, reinterpret_cast<Z*>(run));
      if (t == 0) bulk_wait_read0();  // the engine has read the run before the CTA's smem is released
    } else {
      bar_sync(1, kBT);
      store_run<Z, kBT>(zs, base, cnt, reinterpret_cast<Z*>(buf));
    }
    IXG_TR(11);
  }
}

// ---------------------------------------------------------------------------
// zs = sgmSum flags vs over n elements; flag of element i = bit (flag_base + i)
// of `bits` (mkFlags' bitmap over output positions).  Z: zs storage.
// k_segsum_b's monoid: SegOp for sgmSum, SumOp for a flag-free scan (+)
template <class M>
IXG_DEV typename M::T seg_mk(long long v, int f);
template <>
IXG_DEV SegOp::T seg_mk<SegOp>(long long v, int f) { return SegOp::T{v, f}; }
template <>
IXG_DEV SumOp::T seg_mk<SumOp>(long long v, int) { return SumOp::T{v}; }
template <class M>
IXG_DEV int seg_f(const typename M::T& a) {
  if constexpr (std::is_same<M, SegOp>::value) return a.f;
  else return 0;
}

// What the scan adds up and what it stores (k_segsum_b's F): ScanId is the
// plain scan / sgmSum (element = value, output = the running sum, int64
// overflow checked); the CHECKED pipelines' index scans fuse the predicate
// map in front and the index formula behind (filter.ixl:9-12,
// partition2.ixl:9-16), writing the materialised int64 index array at the
// big-tile kernel's bandwidth.
struct ScanId {
  static constexpr bool kOvf = true;
  static constexpr bool kFlagArr = false;
  static constexpr bool kStore = true;     // out() is stored to zs (else called for its effect only)
  static constexpr bool kBits = false;     // elem() is a 0 / 1 predicate bit (mask16 gives 16 of them)
  static constexpr bool kTrigger = false;  // PDL chain member: release the dependent at the top, wait for
                                           // the predecessor only before the outputs
  static constexpr int kCH = 0;            // chunks per tile if not the default
  IXG_DEV uint32_t flags16(long long, long long) const { return 0u; }
  IXG_DEV void init() {}
  template <typename T>
  IXG_DEV long long elem(T x) const { return (long long)x; }
  IXG_DEV long long out(long long run, long long, long long) const { return run; }
  IXG_DEV void last(long long) const {}
};
template <typename T>
struct PredBit {  // `p x` as 0 / 1 (pred_eval, with the comparison kinds as one interval test)
  ixg_pred p;
  PredRange<T> r;
  IXG_DEV void init() { r = pred_range<T>(p); }
  IXG_DEV long long bit(T x) const {
    if (p.kind <= IXG_PRED_NE) return (long long)(((r.test(x) ? 1u : 0u) & (r.keep & 1u)) ^ (r.flip & 1u));
    return pred_eval(p, (long long)x) ? 1 : 0;
  }
};
// sgmSum over values with the flags of a materialised int64 flag array (the
// CHECKED C2: mkFlags' scatter result): 16 flags of a
// thread per chunk through four 256-bit loads
struct SegFlagArr : ScanId {
  static constexpr bool kFlagArr = true;
  const long long* fa;
  IXG_DEV uint32_t flags16(long long g, long long n) const {
    uint32_t f = 0;
    if (g + kSItems <= n && (((uintptr_t)(fa + g)) & 31) == 0) {
#pragma unroll
      for (int k = 0; k < kSItems / 4; ++k) {
        uint32_t r[8];
        ld256(fa + g + 4 * k, r);
#pragma unroll
        for (int q = 0; q < 4; ++q) f |= (uint32_t)((r[2 * q] | r[2 * q + 1]) != 0u) << (4 * k + q);
      }
    } else {
      for (int q = 0; q < kSItems; ++q)
        if (g + q < n) f |= (uint32_t)(fa[g + q] != 0) << q;
    }
    return f;
  }
};

// mkFlags as a bitmap (the ELIDED C2, ixg_flag_bitmap): the exclusive scan
// of the segment shape; a nonempty segment sets the bit of its start
// (mkSgmDescr's `if shape[i] <= 0 then -1 else scn[i]`, PAPER.md:399-402,
// scattered under Ss2 with starts outside [0, nbits) skipped).  The C2 fused
// kernel is its programmatic dependent.
struct ScanSegStartBits : ScanId {
  static constexpr bool kOvf = true;  // a start past int64 is IXG_OVERFLOW, never a wrapped bit (§2.2)
  static constexpr bool kStore = false;
  static constexpr bool kTrigger = true;
  static constexpr int kCH = IXG_MKF_CH;  // 4 K-value tiles: 256 CTAs for C2's 2^20 segments
  uint32_t* bits;
  long long nb;
  const long long* d_nb;  // nullable: nbits on the device
  const long long* d_lo = nullptr;  // nullable: bitmap window [*d_lo, *d_lo + nb) (a shard's outputs)
  long long lo = 0;
  IXG_DEV void init() {
    if (d_nb) nb = *d_nb;
    if (d_lo) lo = *d_lo;
  }
  IXG_DEV long long out(long long run, long long xv, long long) const {
    const long long start = run - xv;
    if (xv > 0 && start >= lo && start - lo < nb) atomicOr(&bits[(start - lo) >> 5], 1u << ((start - lo) & 31));
    return 0;
  }
};

template <typename T>
struct ScanFilterInds {  // inds[i] = if p xs[i] then offs[i] - 1 else -1; *d_count = offs[n-1]
  static constexpr bool kOvf = false;
  static constexpr bool kFlagArr = false;
  static constexpr bool kStore = true;
  static constexpr bool kTrigger = false;
  static constexpr int kCH = 0;
  IXG_DEV uint32_t flags16(long long, long long) const { return 0u; }
  PredBit<T> pb;
  long long* d_count;
  IXG_DEV void init() { pb.init(); }
  static constexpr bool kBits = true;
  IXG_DEV uint32_t mask16(const T (&x)[kSItems]) const {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < kSItems; ++j) m |= (uint32_t)pb.bit(x[j]) << j;
    return m;
  }
  IXG_DEV long long elem(T x) const { return pb.bit(x); }
  IXG_DEV long long out(long long run, long long xv, long long) const { return xv ? run - 1 : -1; }
  IXG_DEV void last(long long run) const { *d_count = run; }
};
template <typename T>
struct ScanPart2Inds {  // indices[i] = if p x then indicesT[i] - 1 else i + 1 - indicesT[i] + num_true - 1
  static constexpr bool kOvf = false;
  static constexpr bool kFlagArr = false;
  static constexpr bool kStore = true;
  static constexpr bool kTrigger = false;
  static constexpr int kCH = 0;
  IXG_DEV uint32_t flags16(long long, long long) const { return 0u; }
  PredBit<T> pb;
  const long long* d_nt;
  long long nt;
  IXG_DEV void init() {
    pb.init();
    nt = *d_nt;
  }
  static constexpr bool kBits = true;
  IXG_DEV uint32_t mask16(const T (&x)[kSItems]) const {
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < kSItems; ++j) m |= (uint32_t)pb.bit(x[j]) << j;
    return m;
  }
  IXG_DEV long long elem(T x) const { return pb.bit(x); }
  IXG_DEV long long out(long long run, long long xv, long long g) const { return xv ? run - 1 : (g + 1 - run) + nt - 1; }
  IXG_DEV void last(long long) const {}
};

template <typename T, typename Z, class M = SegOp, class F = ScanId>
__global__ void __launch_bounds__(kBT + 32, IXG_SEGSUM_MINB) k_segsum_b(const T* __restrict__ vs, long long n,
                                                          const long long* __restrict__ d_n,
                                                          const uint32_t* __restrict__ bits, long long flag_base,
                                                          const long long* __restrict__ d_flag_base,
                                                          Z* __restrict__ zs, LBChan ch, uint32_t nonce,
                                                          long long carry_v, int carry_f, longlong2* d_total,
                                                          ixg_status* st, F fn = F{}) {
  constexpr int CHO = F::kCH ? F::kCH : kSegsumCH<T, Z>;
  using B = Big<T, CHO>;
  if constexpr (F::kTrigger) pdl_trigger();
  fn.init();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* buf = reinterpret_cast<T*>(smem_raw);
  __shared__ typename M::T s_w[B::CH][kBW];
  __shared__ typename M::T s_agg;
  __shared__ typename M::T s_carry;
  __shared__ __align__(8) uint64_t s_mbar[B::CH];

  if (d_n) n = *d_n;  // length known only on the device (C2: k = filter's count)
  if (d_flag_base) flag_base = *d_flag_base;  // sharded C2: this rank's first global output position
  const long long ntiles = (n + B::TILE - 1) / B::TILE;
  const long long tile = blockIdx.x;
  if (tile >= ntiles) return;  // capacity grid: tiles past the data do nothing
  const long long tile_base = tile * B::TILE;
  const int t = threadIdx.x;
  if (warp_id() == kBW) {  // look-back warp
    typename M::T ex = seg_mk<M>(carry_v, carry_f);  // carry into the first tile (earlier shards)
    if (tile > 0) ex = lb_lookback<M>(ch, nonce, tile);
    if (lane_id() == 0) s_carry = ex;
    bar_sync(2, kBT + 32);
    if (lane_id() == 0) {
      const typename M::T incl = M::op(ex, s_agg);
      if (tile > 0) lb_publish<M>(ch, nonce, tile, incl, true);
      if (tile == ntiles - 1 && d_total) *d_total = make_longlong2(incl.v, seg_f<M>(incl));
    }
    return;
  }
  // int32 full tiles: one TMA bulk copy per chunk into a linear buffer
  // (read back with lin_read_xor); otherwise swizzled per-lane cp.async
  const bool tma = (sizeof(T) == 4 || IXG_SEGSUM_TMA64) && tile_base + B::TILE <= n;
  if (tma) {
    if (t == 0) {
#pragma unroll
      for (int c = 0; c < B::CH; ++c) mbar_init(&s_mbar[c], 1);
      mbar_fence_init();
#pragma unroll
      for (int c = 0; c < B::CH; ++c) {
        mbar_expect_tx(&s_mbar[c], kBChunk * (uint32_t)sizeof(T));
        bulk_g2s(buf + B::PAD + c * kBChunk, vs + tile_base + c * kBChunk, kBChunk * (uint32_t)sizeof(T), &s_mbar[c]);
      }
    }
    bar_sync(1, kBT);  // the mbarriers are initialised
  } else {
    big_issue<T, CHO>(buf, vs, n, tile_base, t);
  }
  // the thread's 16 flag bits per chunk (positions are known up front)
  uint32_t fl[B::CH];
#pragma unroll
  for (int c = 0; c < B::CH; ++c) {
    const long long g = tile_base + (long long)c * kBChunk + (long long)kSItems * t;
    const long long pos = flag_base + g;
    const long long wd = pos >> 5;
    uint32_t f = 0;
    if constexpr (F::kFlagArr) {  // flags from a materialised int64 array (CHECKED sgmSum)
      if (g < n) f = fn.flags16(g, n);
    } else if (std::is_same<M, SegOp>::value && g < n && bits) {  // SumOp / no bits: a plain scan (ixg_scan_add)
      f = (uint32_t)((((uint64_t)__ldg(&bits[wd + 1]) << 32) | (uint64_t)__ldg(&bits[wd])) >> (pos & 31));
    }
    fl[c] = f & valid_mask(g, n);
  }
  if (!tma) cp_async_wait_all();
  typename M::T a[B::CH];
  uint32_t pm[B::CH];  // F::kBits: the chunk's 16 element bits
  (void)pm;
#pragma unroll
  for (int c = 0; c < B::CH; ++c) {
    T x[kSItems];
    if constexpr (sizeof(T) == 4) {
      if (tma) {
        mbar_wait(&s_mbar[c], 0);
        lin_read_xor(reinterpret_cast<const int32_t*>(buf), c, t, reinterpret_cast<int32_t(&)[kSItems]>(x));
      } else {
        big_read<T>(buf, c, t, x);
      }
    } else {
      if (tma) {
        mbar_wait(&s_mbar[c], 0);
        lin_read_xor64(reinterpret_cast<const long long*>(buf), c, t, reinterpret_cast<long long(&)[kSItems]>(x));
      } else {
        big_read<T>(buf, c, t, x);
      }
    }
    const long long g = tile_base + (long long)c * kBChunk + (long long)kSItems * t;
    const uint32_t vm = valid_mask(g, n);
    const uint32_t tail = fl[c] ? (vm & ~((1u << (31 - __clz(fl[c]))) - 1u)) : vm;
    long long s = 0;
    if constexpr (F::kBits && IXG_SEGSUM_BITS) {  // 0 / 1 elements: their sum is a popcount, the bits kept for pass 2
      pm[c] = fn.mask16(x);
      s = __popc(pm[c] & tail);
    } else {
#pragma unroll
      for (int j = 0; j < kSItems; ++j) s += ((tail >> j) & 1u) ? fn.elem(x[j]) : 0LL;
    }
    a[c] = seg_mk<M>(s, fl[c] != 0);
    typename M::T inc = warp_inclusive<M>(a[c]);
    if (lane_id() == 31) s_w[c][warp_id()] = inc;
    typename M::T lex = M::shfl_up(inc, 1);
    if (lane_id() == 0) lex = M::identity();
    a[c] = lex;  // the lane's exclusive prefix within its warp and chunk
  }
  bar_sync(1, kBT);
  // tile aggregate (chunk-major order) and each (chunk, warp) prefix
  typename M::T tagg = M::identity();
  typename M::T chunk_pre[B::CH];
  if constexpr (IXG_SEGSUM_WSCAN && B::CH * kBW <= 32) {
    // one warp-wide scan over the CH x kBW (chunk, warp) aggregates, in every
    // warp: lane l holds aggregate l (chunk l / kBW, warp l % kBW)
    const int l = lane_id();
    typename M::T ag = M::identity();
    if (l < B::CH * kBW) ag = s_w[l / kBW][l % kBW];
    const typename M::T inc = warp_inclusive<M>(ag);
    typename M::T exc = M::shfl_up(inc, 1);
    if (l == 0) exc = M::identity();
    tagg = M::shfl(inc, B::CH * kBW - 1);
#pragma unroll
    for (int c = 0; c < B::CH; ++c) chunk_pre[c] = M::op(M::shfl(exc, c * kBW + warp_id()), a[c]);
  } else {
#pragma unroll
    for (int c = 0; c < B::CH; ++c) {
      chunk_pre[c] = tagg;
      typename M::T wp = M::identity();
#pragma unroll
      for (int w = 0; w < kBW; ++w) {
        if (w < warp_id()) wp = M::op(wp, s_w[c][w]);
        tagg = M::op(tagg, s_w[c][w]);
      }
      chunk_pre[c] = M::op(M::op(chunk_pre[c], wp), a[c]);
    }
  }
  if (t == 0) {
    s_agg = tagg;
    if (tile == 0) lb_publish<M>(ch, nonce, tile, M::op(seg_mk<M>(carry_v, carry_f), tagg), true);
    else lb_publish<M>(ch, nonce, tile, tagg, false);
  }
  bar_sync(2, kBT + 32);
  if constexpr (F::kTrigger) pdl_wait();  // (mkFlags) the bitmap's clear has finished
  const typename M::T carry = s_carry;
  bool narrow = false;
  long long ovf_at = LLONG_MAX;  // first element whose int64 sum overflowed (Z = int64)
#pragma unroll
  for (int c = 0; c < B::CH; ++c) {
    T x[kSItems];
    if constexpr (sizeof(T) == 4) {
      if (tma) lin_read_xor(reinterpret_cast<const int32_t*>(buf), c, t, reinterpret_cast<int32_t(&)[kSItems]>(x));
      else big_read<T>(buf, c, t, x);
    } else {
      if (tma) lin_read_xor64(reinterpret_cast<const long long*>(buf), c, t, reinterpret_cast<long long(&)[kSItems]>(x));
      else big_read<T>(buf, c, t, x);
    }
    const long long g = tile_base + (long long)c * kBChunk + (long long)kSItems * t;
    long long run = M::op(carry, chunk_pre[c]).v;
    Z z[kSItems];
    // int32 sgmSum into int32 (C2's zs): from an exact start inside int32
    // the run is carried modulo 2^32 -- a result leaves int32 iff its signed
    // add overflows (before the first such add every start is exact), so
    // NARROW is the same as the 64-bit run's; a start outside int32 (only
    // a carry from earlier shards can be one) takes the 64-bit loop
    constexpr bool k32 = IXG_SEGSUM_RUN32 && sizeof(T) == 4 && sizeof(Z) == 4 && std::is_same<M, SegOp>::value &&
                         (std::is_same<F, ScanId>::value || std::is_same<F, SegFlagArr>::value);
    if (k32 && run == (long long)(int)run) {
      int32_t r = (int32_t)run;
      uint32_t ov = 0;
#pragma unroll
      for (int j = 0; j < kSItems; ++j) {
        const int32_t xv = (int32_t)x[j];
        const int32_t pr = ((fl[c] >> j) & 1u) ? 0 : r;
        const int32_t nr = (int32_t)((uint32_t)pr + (uint32_t)xv);
        ov |= (uint32_t)((pr ^ nr) & (xv ^ nr));
        z[j] = (Z)nr;
        r = nr;
      }
      if ((int32_t)ov < 0) narrow = true;
    } else {
      // exact: the sequential step prev + x in the reference's unbounded
      // ints -- the steps' signed-overflow bits are OR-ed, and the first
      // overflowing element is looked for only when one did (elements past
      // n are zero-filled: prev + 0 never overflows)
      const long long run0 = run;
      long long ovm = 0;
#pragma unroll
      for (int j = 0; j < kSItems; ++j) {
        const long long prev = ((fl[c] >> j) & 1u) ? 0LL : run;
        long long xv;
        if constexpr (F::kBits && IXG_SEGSUM_BITS) xv = (long long)((pm[c] >> j) & 1u);
        else xv = fn.elem(x[j]);
        run = (long long)((unsigned long long)prev + (unsigned long long)xv);
        if (sizeof(Z) == 4 && run != (long long)(int)run) narrow = true;
        if constexpr (F::kOvf && sizeof(Z) == 8) ovm |= (prev ^ run) & (xv ^ run);
        if (g + j == n - 1) fn.last(run);
        if constexpr (F::kStore) z[j] = (Z)fn.out(run, xv, g + j);
        else if (g + j < n) fn.out(run, xv, g + j);
      }
      if (F::kOvf && sizeof(Z) == 8 && ovm < 0 && ovf_at == LLONG_MAX) {
        long long r2 = run0;
        for (int j = 0; j < kSItems; ++j) {
          const long long prev = ((fl[c] >> j) & 1u) ? 0LL : r2;
          const long long xv = fn.elem(x[j]);
          r2 = (long long)((unsigned long long)prev + (unsigned long long)xv);
          if ((((prev ^ r2) & (xv ^ r2)) < 0) && g + j < n) {
            ovf_at = g + j;
            break;
          }
        }
      }
    }
    if constexpr (!F::kStore) {
    } else if (g + kSItems <= n) {
      constexpr int ZV = 32 / (int)sizeof(Z);  // elements per 256-bit store
#pragma unroll
      for (int v = 0; v < kSItems / ZV; ++v) {
        uint32_t r[8];
#pragma unroll
        for (int e = 0; e < ZV; ++e) {
          if constexpr (sizeof(Z) == 4) {
            r[e] = (uint32_t)z[v * ZV + e];
          } else {
            r[2 * e] = (uint32_t)(unsigned long long)z[v * ZV + e];
            r[2 * e + 1] = (uint32_t)((unsigned long long)z[v * ZV + e] >> 32);
          }
        }
        st256(zs + g + v * ZV, r);
      }
    } else {
#pragma unroll
      for (int j = 0; j < kSItems; ++j)
        if (g + j < n) zs[g + j] = z[j];
    }
  }
  if (narrow && st) atomicOr(&st->flags, IXG_F_NARROW);
  if (sizeof(Z) == 8 && ovf_at != LLONG_MAX) status_overflow(st, 0, ovf_at);
}

// ---------------------------------------------------------------------------
// Shard carry (multi-GPU C2): the first flag at or after `flag_base` within
// [flag_base, flag_base + n), then zs[0 .. first) += carry.
__global__ void __launch_bounds__(256) k_first_flag(const uint32_t* __restrict__ bits, long long flag_base,
                                                    const long long* __restrict__ d_flag_base, long long n,
                                                    const long long* __restrict__ d_n, unsigned long long* first) {
  if (d_n) n = *d_n;
  if (d_flag_base) flag_base = *d_flag_base;
  const long long nw = (n + 31) / 32 + 1;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < nw; k += stride) {
    const long long q0 = k * 32;  // local position of this window
    if (q0 >= n) break;
    const long long g = flag_base + q0;
    uint32_t w = (uint32_t)((((uint64_t)bits[(g >> 5) + 1] << 32) | bits[g >> 5]) >> (g & 31));
    const long long lim = n - q0;
    if (lim < 32) w &= (1u << lim) - 1u;
    if (w) atomicMin(first, (unsigned long long)(q0 + __ffs(w) - 1));
  }
}

// carry into `rank` from every rank's segmented aggregate (v, f) (an
// all-gathered device array [ranks][2]): the segmented combine of those of
// ranks < rank
IXG_DEV long long seg_carry_from(const long long* __restrict__ aggs, int rank) {
  long long v = 0;
  for (int r = 0; r < rank; ++r) v = aggs[2 * r + 1] ? aggs[2 * r] : (long long)((unsigned long long)v + (unsigned long long)aggs[2 * r]);
  return v;
}

template <typename Z>
__global__ void __launch_bounds__(256) k_add_prefix(Z* __restrict__ zs, const unsigned long long* __restrict__ first,
                                                    long long n, const long long* __restrict__ d_n, long long c,
                                                    const long long* __restrict__ d_aggs, int rank, ixg_status* st) {
  if (d_n) n = *d_n;
  if (d_aggs) c = seg_carry_from(d_aggs, rank);
  if (c == 0) return;
  long long stop = (long long)*first;
  if (stop > n) stop = n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool narrow = false;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < stop; q += stride) {
    const long long v = (long long)zs[q] + c;
    if (sizeof(Z) == 4 && v != (long long)(int)v) narrow = true;
    zs[q] = (Z)v;
  }
  if (narrow && st) atomicOr(&st->flags, IXG_F_NARROW);
}

// out2 = [sum of counts[r * stride] over r < rank, over all r] (a rank's
// exclusive offset and the global total from an all-gathered device array)
__global__ void k_rank_offsets(const long long* __restrict__ counts, int ranks, int rank, int stride,
                               long long* __restrict__ out2) {
  if (threadIdx.x == 0) {
    long long before = 0, total = 0;
    for (int r = 0; r < ranks; ++r) {
      const long long c = counts[(long long)r * stride];
      total += c;
      before += r < rank ? c : 0;
    }
    out2[0] = before;
    out2[1] = total;
  }
}

// partition3's single pass leaves the prefix at the end of segment 1 (m1 + m2)
__global__ void k_sub_first(long long* d_tot) { d_tot[1] -= d_tot[0]; }

// ---------------------------------------------------------------------------
// Vectorised scatter (C3 and every fused-away-free scatter site): 8 source
// elements per thread-iteration, indices and values as 256-bit streaming
// loads (96 B in flight per thread for i64 indices + i32 values), then 8
// independent stores; CHECKED adds the claim-bitmap atomics exactly as
// k_scatter (k_generic.cuh).  Needs 32-byte aligned is / vs.
template <typename E>
__global__ void __launch_bounds__(256) k_scatter_v(E* __restrict__ out, long long ndst,
                                                   const long long* __restrict__ d_ndst,
                                                   const long long* __restrict__ is, const E* __restrict__ vs,
                                                   long long m, int check, uint32_t* __restrict__ claim,
                                                   LBHeader* hdr) {
  if (d_ndst) ndst = *d_ndst;
  const long long nv = m >> 3;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  bool dup = false;
  for (long long k = tid; k < nv; k += stride) {
    uint32_t a[8], b[8];
    ld256(is + 8 * k, a);
    ld256(is + 8 * k + 4, b);
    E x[8];
    if constexpr (sizeof(E) == 4) {
      uint32_t c[8];
      ld256(vs + 8 * k, c);
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = (E)c[j];
    } else {
      uint32_t c[8], e[8];
      ld256(vs + 8 * k, c);
      ld256(vs + 8 * k + 4, e);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        x[j] = (E)(((unsigned long long)c[2 * j + 1] << 32) | c[2 * j]);
        x[4 + j] = (E)(((unsigned long long)e[2 * j + 1] << 32) | e[2 * j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t lo = j < 4 ? a[2 * j] : b[2 * (j - 4)];
      const uint32_t hi = j < 4 ? a[2 * j + 1] : b[2 * (j - 4) + 1];
      const long long d = (long long)(((unsigned long long)hi << 32) | lo);
      if ((unsigned long long)d < (unsigned long long)ndst) {
        if (check) {
          const uint32_t bit = 1u << (d & 31);
          if (atomicOr(&claim[d >> 5], bit) & bit) dup = true;
        }
        out[d] = x[j];
      }
    }
  }
  for (long long i = nv * 8 + tid; i < m; i += stride) {
    const long long d = is[i];
    if ((unsigned long long)d < (unsigned long long)ndst) {
      if (check) {
        const uint32_t bit = 1u << (d & 31);
        if (atomicOr(&claim[d >> 5], bit) & bit) dup = true;
      }
      out[d] = vs[i];
    }
  }
  if (__any_sync(0xffffffffu, dup) && lane_id() == 0) atomicExch(&hdr->dup, 1u);
}


// ---------------------------------------------------------------------------
// TMA-staged scatter: one CTA per 4096-element tile; thread 0 bulk-copies the
// tile's indices and values to shared memory (48 KB for i64 indices + i32
// values: 4 CTAs per SM keep ~190 KB of reads in flight without LSU work),
// then the warps walk the tile STRIPED -- lane l takes element 32k + l -- so
// each warp-wide store covers 32 consecutive sources, i.e. the few
// contiguous destination runs of an index-array permutation (C3: two
// streams) land in a handful of sectors.  CHECKED adds the claim-bitmap
// atomics exactly as k_scatter (k_generic.cuh).
constexpr int kScTile = 4096;
template <typename E>
struct ScSmem {
  static constexpr int BYTES = kScTile * (8 + (int)sizeof(E));
};

template <typename E>
__global__ void __launch_bounds__(256) k_scatter_t(E* __restrict__ out, long long ndst,
                                                   const long long* __restrict__ d_ndst,
                                                   const long long* __restrict__ is, const E* __restrict__ vs,
                                                   long long m, int check, uint32_t* __restrict__ claim,
                                                   LBHeader* hdr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  long long* s_is = reinterpret_cast<long long*>(smem_raw);
  E* s_vs = reinterpret_cast<E*>(smem_raw + kScTile * 8);
  __shared__ __align__(8) uint64_t s_mbar;
  if (d_ndst) ndst = *d_ndst;
  const long long base = (long long)blockIdx.x * kScTile;
  const int t = threadIdx.x;
  const bool full = base + kScTile <= m;
  bool dup = false;
  auto one = [&](long long d, E v) {
    if ((unsigned long long)d < (unsigned long long)ndst) {
      if (check) {
        const uint32_t bit = 1u << (d & 31);
        if (atomicOr(&claim[d >> 5], bit) & bit) dup = true;
      }
      out[d] = v;
    }
  };
  if (full) {
    if (t == 0) {
      mbar_init(&s_mbar, 1);
      mbar_fence_init();
      mbar_expect_tx(&s_mbar, (uint32_t)ScSmem<E>::BYTES);
      bulk_g2s(s_is, is + base, kScTile * 8u, &s_mbar);
      bulk_g2s(s_vs, vs + base, kScTile * (uint32_t)sizeof(E), &s_mbar);
    }
    __syncthreads();  // the mbarrier is initialised
    mbar_wait(&s_mbar, 0);
#pragma unroll 4
    for (int k = t; k < kScTile; k += 256) one(s_is[k], s_vs[k]);
  } else {
    for (long long i = base + t; i < m; i += 256) one(is[i], vs[i]);
  }
  if (__any_sync(0xffffffffu, dup) && lane_id() == 0) atomicExch(&hdr->dup, 1u);
}

}  // namespace ixg
