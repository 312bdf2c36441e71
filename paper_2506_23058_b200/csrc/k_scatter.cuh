// k_scatter.cuh -- the generic scatter (oracle.py:294-305) beyond the fused
// pipelines: the CHECKED form's duplicate detection as a shared-memory-
// privatised claim histogram, and destination-window binning for index
// arrays without locality.
//
// CHECKED scatter (k_scatter_pc).  The reference keeps a `written` dict
// (oracle.py:298-302); the device form claims every in-range destination in
// a bitmap (one bit per destination) and only if some destination was
// claimed twice re-reads the pairs to compare values (equal-valued
// duplicates are legal).  Instead of one global atomicOr per element, each
// 4096-pair tile claims into up to kWinSlots shared-memory windows of 4096
// destinations (a window is 128 words; shared atomics), then merges each
// touched window into the global bitmap with ONE coalesced atomicOr per
// non-zero word -- a collision inside the tile shows in the shared OR, one
// across tiles in the global OR's old value.  An index array with locality
// (C3's partition indices: two monotone streams, so a tile touches <= 4
// windows) does ~16x fewer global atomics; pairs whose window finds no free
// slot fall back to the global atomic.  The shared windows are stored
// transposed (destination b -> bit b >> 7 of word b & 127) so that a warp's
// consecutive destinations claim in 32 different banks.
//
// Binned scatter (k_bin_*).  A random permutation scatters one 4-byte store
// per 32-byte sector over a 2 GB destination: every store misses, and the
// sector is read back before it is written (partial-sector writes).  The
// binned form first partitions the (index, value) pairs by destination
// window (B <= 256 windows of 2M int32 destinations = 8 MB, L2-resident):
// each tile counts its pairs per window in shared memory, reserves room in
// each window's global run with one atomicAdd per (tile, window), stages the
// pairs window by window in shared memory and writes each window's run
// contiguously (indices narrowed to u32).  The second pass is the ordinary
// (ELIDED or CHECKED) scatter over the binned pairs: at any moment the
// resident tiles write into one or two 8 MB windows, which the L2 absorbs
// until their lines are complete.  Pairs outside [0, ndst) are dropped by the
// first pass (the reference ignores them, oracle.py:300).
#pragma once
#include "k_big.cuh"

namespace ixg {

constexpr int kWinBits = 12;                      // claim window: 4096 destinations
constexpr int kWinWords = (1 << kWinBits) / 32;  // 128 bitmap words
constexpr int kWinSlots = 8;                      // windows per tile in shared memory
constexpr int kBinMax = 256;                      // destination windows of the binned scatter
#ifndef IXG_BLOCKED_CLAIMS
#define IXG_BLOCKED_CLAIMS 1
#endif
constexpr bool kBlockedClaims = IXG_BLOCKED_CLAIMS;  // k_scatter_pc: register-combined claims (A/B)

template <typename I, typename E>
struct PcSmem {  // TMA-staged tile of (I index, E value) pairs
  static constexpr int BYTES = kScTile * ((int)sizeof(I) + (int)sizeof(E));
};

// shared-window atomics in the shared state space (a generic-address atomic
// re-derives the CTA's shared window -- S2R SR_CgaCtaId -- every time)
IXG_DEV uint32_t atom_or_shared(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cta.or.b32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}
IXG_DEV unsigned long long atom_cas_shared(unsigned long long* p, unsigned long long cmp, unsigned long long v) {
  unsigned long long old;
  asm volatile("atom.shared::cta.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "r"(smem_u32(p)), "l"(cmp), "l"(v) : "memory");
  return old;
}

// L2 policy for streamed-once inputs: evict first, so a binned scatter's
// destination window stays resident while its pairs stream through
IXG_DEV uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
IXG_DEV uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
template <typename E>
IXG_DEV void st_keep(E* p, E v, uint64_t pol) {
  if constexpr (sizeof(E) == 4)
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"((uint32_t)v), "l"(pol)
                 : "memory");
  else
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p),
                 "l"((unsigned long long)v), "l"(pol)
                 : "memory");
}
IXG_DEV void bulk_g2s_ef(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

// CHECKED scatter, claims privatised in shared-memory windows (kPriv) or
// straight into the global bitmap (binned pairs: no locality to exploit);
// I = index type (int64 for the language's arrays, u32 for binned pairs),
// the tile TMA-staged when full.  A warp looks each distinct window up once
// (match_any): C3's 32 consecutive sources fall into ~2 windows.
template <typename I, typename E, bool kPriv = true>
__global__ void __launch_bounds__(256) k_scatter_pc(E* __restrict__ out, long long ndst,
                                                    const long long* __restrict__ d_ndst,
                                                    const I* __restrict__ is, const E* __restrict__ vs, long long m,
                                                    const long long* __restrict__ d_m, uint32_t* __restrict__ claim,
                                                    LBHeader* hdr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  I* s_is = reinterpret_cast<I*>(smem_raw);
  E* s_vs = reinterpret_cast<E*>(smem_raw + kScTile * sizeof(I));
  __shared__ uint32_t s_bits[kWinSlots * kWinWords];
  __shared__ unsigned long long s_win[kWinSlots];
  __shared__ __align__(8) uint64_t s_mbar;
  if (d_ndst) ndst = *d_ndst;
  if (d_m) m = *d_m;
  const long long base = (long long)blockIdx.x * kScTile;
  if (base >= m) return;
  const int t = threadIdx.x;
  const bool full = base + kScTile <= m;
  for (int q = t; q < kWinSlots * kWinWords; q += 256) s_bits[q] = 0u;
  if (t < kWinSlots) s_win[t] = ~0ull;
  if (full && t == 0) {
    mbar_init(&s_mbar, 1);
    mbar_fence_init();
    mbar_expect_tx(&s_mbar, (uint32_t)PcSmem<I, E>::BYTES);
    bulk_g2s(s_is, is + base, kScTile * (uint32_t)sizeof(I), &s_mbar);
    bulk_g2s(s_vs, vs + base, kScTile * (uint32_t)sizeof(E), &s_mbar);
  }
  __syncthreads();
  if (full) mbar_wait(&s_mbar, 0);
  volatile unsigned long long* vw = s_win;
  bool dup = false;
  const int cnt = full ? kScTile : (int)(m - base);
  // the thread's last two windows and their slots (C3: a thread's sources,
  // 256 apart, go to one of two streams, each advancing ~128 destinations)
  // the thread's last two windows and their slots (C3: a thread's sources,
  // 256 apart, go to one of two streams, each advancing ~128 destinations)
  unsigned long long cw0 = ~0ull, cw1 = ~0ull;
  int cs0 = -1, cs1 = -1;
  auto one = [&](long long d, E v) {
    if ((unsigned long long)d >= (unsigned long long)ndst) return;  // oracle.py:300
    if constexpr (kPriv) {
      const unsigned long long w = (unsigned long long)d >> kWinBits;
      int slot;
      if (w == cw0) {
        slot = cs0;
      } else if (w == cw1) {
        slot = cs1;
      } else {
        slot = -1;
#pragma unroll 1
        for (int j = 0; j < kWinSlots; ++j) {
          unsigned long long cur = vw[j];
          if (cur == ~0ull) {  // a free slot: claim it for w (or learn who did)
            cur = atom_cas_shared(&s_win[j], ~0ull, w);
            if (cur == ~0ull) cur = w;
          }
          if (cur == w) {
            slot = j;
            break;
          }
        }
        cw1 = cw0;
        cs1 = cs0;
        cw0 = w;
        cs0 = slot;
      }
      if (slot >= 0) {
        const uint32_t bit = 1u << (d & 31);
        if (atom_or_shared(&s_bits[slot * kWinWords + (int)((d >> 5) & (kWinWords - 1))], bit) & bit) dup = true;
      } else {
        const uint32_t bit = 1u << (d & 31);
        if (atomicOr(&claim[d >> 5], bit) & bit) dup = true;
      }
    } else {
      // no locality to privatise: a fire-and-forget reduction (RED, no
      // return trip); duplicates show up as fewer distinct bits than pairs
      // (k_claim_count)
      atomicOr(&claim[d >> 5], 1u << (d & 31));
    }
    out[d] = v;
  };
  // striped: a warp's stores cover 32 consecutive sources.  Separate loops
  // for the staged and the ragged tile: a select between a shared and a
  // global pointer would make every access a generic one
  if (full && kPriv && kBlockedClaims) {
    // claims thread-blocked (16 consecutive sources, read in a per-thread
    // rotated order so a warp's shared loads spread over the banks): the
    // bits a thread claims in one shared word are combined in a register
    // first, one shared atomic per run of same-word destinations
    int key = -1;
    uint32_t acc = 0;
#pragma unroll 1
    for (int jj = 0; jj < kScTile / 256; ++jj) {
      const long long d = (long long)s_is[t * (kScTile / 256) + ((jj + t) & (kScTile / 256 - 1))];
      if ((unsigned long long)d >= (unsigned long long)ndst) continue;
      const unsigned long long w = (unsigned long long)d >> kWinBits;
      int slot;
      if (w == cw0) {
        slot = cs0;
      } else if (w == cw1) {
        slot = cs1;
      } else {
        slot = -1;
#pragma unroll 1
        for (int j = 0; j < kWinSlots; ++j) {
          unsigned long long cur = vw[j];
          if (cur == ~0ull) {
            cur = atom_cas_shared(&s_win[j], ~0ull, w);
            if (cur == ~0ull) cur = w;
          }
          if (cur == w) {
            slot = j;
            break;
          }
        }
        cw1 = cw0;
        cs1 = cs0;
        cw0 = w;
        cs0 = slot;
      }
      const uint32_t bit = 1u << (d & 31);
      if (slot < 0) {
        if (atomicOr(&claim[d >> 5], bit) & bit) dup = true;
        continue;
      }
      const int kk = slot * kWinWords + (int)((d >> 5) & (kWinWords - 1));
      if (kk != key) {
        if (key >= 0 && (atom_or_shared(&s_bits[key], acc) & acc)) dup = true;
        key = kk;
        acc = 0u;
      }
      if (acc & bit) dup = true;
      acc |= bit;
    }
    if (key >= 0 && (atom_or_shared(&s_bits[key], acc) & acc)) dup = true;
    for (int k = t; k < kScTile; k += 256) {  // the stores, striped
      const long long d = (long long)s_is[k];
      if ((unsigned long long)d < (unsigned long long)ndst) out[d] = s_vs[k];
    }
  } else if (full) {
    for (int k = t; k < kScTile; k += 256) one((long long)s_is[k], s_vs[k]);
  } else {
    for (int k = t; k < cnt; k += 256) one((long long)is[base + k], vs[base + k]);
  }
  if constexpr (!kPriv) {
    if (__any_sync(0xffffffffu, dup) && lane_id() == 0) atomicExch(&hdr->dup, 1u);
    return;
  }
  __syncthreads();
  // merge the touched windows: global word q of a window holds destinations
  // 32q .. 32q+31, i.e. bit q >> 2 of the shared words (32q + j) & 127 --
  // transposed back with 32 broadcast reads, then ONE coalesced atomicOr
  // per non-zero word
  for (int gq = t; gq < kWinSlots * kWinWords; gq += 256) {
    const int slot = gq / kWinWords, q = gq % kWinWords;
    const unsigned long long w = s_win[slot];
    if (w == ~0ull) continue;
    const uint32_t word = s_bits[gq];
    if (word && (atomicOr(&claim[w * kWinWords + q], word) & word)) dup = true;
  }
  if (__any_sync(0xffffffffu, dup) && lane_id() == 0) atomicExch(&hdr->dup, 1u);
}

// CHECKED scatter, claims in 2-way set-associative shared-memory windows:
// window w (4096 destinations) lives in set w & 3, one of its two ways, so a
// claim finds its slot with ONE 16-byte tag load and two compares -- no
// window search, no per-thread window cache, no divergent lookup loop.  Two
// interleaved monotone streams (C3: each touches <= 2 consecutive windows
// per tile, i.e. two consecutive sets) always fit; a window that finds its
// set full claims straight in the global bitmap.  Each thread claims 16
// consecutive sources (rotated reads, conflict-free), one shared atomic per
// in-range pair whose old value flags a duplicate inside the tile; the
// windows are then merged with one coalesced global atomicOr per non-zero
// word (the old value flags one across tiles).  Stores are striped.
template <typename E>
__global__ void __launch_bounds__(256) k_scatter_sa(E* __restrict__ out, long long ndst,
                                                    const long long* __restrict__ d_ndst,
                                                    const long long* __restrict__ is, const E* __restrict__ vs,
                                                    long long m, uint32_t* __restrict__ claim, LBHeader* hdr) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  long long* s_is = reinterpret_cast<long long*>(smem_raw);
  E* s_vs = reinterpret_cast<E*>(smem_raw + kScTile * sizeof(long long));
  __shared__ uint32_t s_bits[kWinSlots * kWinWords];
  __shared__ __align__(16) unsigned long long s_win[kWinSlots];  // set q: ways 2q, 2q + 1
  __shared__ __align__(8) uint64_t s_mbar;
  if (d_ndst) ndst = *d_ndst;
  const long long base = (long long)blockIdx.x * kScTile;
  if (base >= m) return;
  const int t = threadIdx.x;
  const bool full = base + kScTile <= m;
  for (int q = t; q < kWinSlots * kWinWords; q += 256) s_bits[q] = 0u;
  if (t < kWinSlots) s_win[t] = ~0ull;
  if (full && t == 0) {
    mbar_init(&s_mbar, 1);
    mbar_fence_init();
    mbar_expect_tx(&s_mbar, (uint32_t)PcSmem<long long, E>::BYTES);
    bulk_g2s(s_is, is + base, kScTile * (uint32_t)sizeof(long long), &s_mbar);
    bulk_g2s(s_vs, vs + base, kScTile * (uint32_t)sizeof(E), &s_mbar);
  }
  __syncthreads();
  bool dup = false;
  const uint32_t win_sa = smem_u32(s_win);  // (the shared address once, not per claim)
  auto claim_one = [&](long long d) {
    if ((unsigned long long)d >= (unsigned long long)ndst) return;  // oracle.py:300
    const unsigned long long w = (unsigned long long)d >> kWinBits;
    const int q = 2 * (int)(w & (kWinSlots / 2 - 1));
    unsigned long long t0, t1;  // both ways' tags, one 16-byte shared load
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(t0), "=l"(t1) : "r"(win_sa + 8u * q));
    int sl = t0 == w ? q : (t1 == w ? q + 1 : -1);
    if (sl < 0) {  // first touch of w in this tile, or its set is full
#pragma unroll 1
      for (int j = q; j < q + 2; ++j) {
        unsigned long long cur = reinterpret_cast<volatile unsigned long long*>(s_win)[j];
        if (cur == ~0ull) {
          cur = atom_cas_shared(&s_win[j], ~0ull, w);
          if (cur == ~0ull) cur = w;
        }
        if (cur == w) {
          sl = j;
          break;
        }
      }
    }
    const uint32_t bit = 1u << (d & 31);
    if (sl >= 0) {
      if (atom_or_shared(&s_bits[sl * kWinWords + (int)((d >> 5) & (kWinWords - 1))], bit) & bit) dup = true;
    } else if (atomicOr(&claim[d >> 5], bit) & bit) {
      dup = true;
    }
  };
  if (full) {
    mbar_wait(&s_mbar, 0);
#pragma unroll 4
    for (int jj = 0; jj < kScTile / 256; ++jj)
      claim_one(s_is[t * (kScTile / 256) + ((jj + t) & (kScTile / 256 - 1))]);
    __syncwarp();  // reconverged: the striped stores leave as whole-warp stores
    for (int k = t; k < kScTile; k += 256) {
      const long long d = s_is[k];
      if ((unsigned long long)d < (unsigned long long)ndst) out[d] = s_vs[k];
    }
  } else {
    for (long long i = base + t; i < m; i += 256) {
      const long long d = is[i];
      claim_one(d);
      if ((unsigned long long)d < (unsigned long long)ndst) out[d] = vs[i];
    }
  }
  __syncthreads();
  // merge the touched windows: ONE coalesced atomicOr per non-zero word
  for (int gq = t; gq < kWinSlots * kWinWords; gq += 256) {
    const unsigned long long w = s_win[gq / kWinWords];
    if (w == ~0ull) continue;
    const uint32_t word = s_bits[gq];
    if (word && (atomicOr(&claim[w * kWinWords + gq % kWinWords], word) & word)) dup = true;
  }
  if (__any_sync(0xffffffffu, dup) && lane_id() == 0) atomicExch(&hdr->dup, 1u);
}

// ELIDED scatter of TMA-staged tiles (k_scatter_t) for any index type, with
// the pair count optionally on the device (binned pairs)
template <typename I, typename E>
__global__ void __launch_bounds__(256) k_scatter_ti(E* __restrict__ out, long long ndst,
                                                    const long long* __restrict__ d_ndst,
                                                    const I* __restrict__ is, const E* __restrict__ vs, long long m,
                                                    const long long* __restrict__ d_m) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  I* s_is = reinterpret_cast<I*>(smem_raw);
  E* s_vs = reinterpret_cast<E*>(smem_raw + kScTile * sizeof(I));
  __shared__ __align__(8) uint64_t s_mbar;
  if (d_ndst) ndst = *d_ndst;
  if (d_m) m = *d_m;
  const long long base = (long long)blockIdx.x * kScTile;
  if (base >= m) return;
  const int t = threadIdx.x;
  if (base + kScTile <= m) {
    if (t == 0) {
      mbar_init(&s_mbar, 1);
      mbar_fence_init();
      mbar_expect_tx(&s_mbar, (uint32_t)PcSmem<I, E>::BYTES);
      const uint64_t pol = l2_evict_first_policy();
      bulk_g2s_ef(s_is, is + base, kScTile * (uint32_t)sizeof(I), &s_mbar, pol);
      bulk_g2s_ef(s_vs, vs + base, kScTile * (uint32_t)sizeof(E), &s_mbar, pol);
    }
    __syncthreads();
    mbar_wait(&s_mbar, 0);
    const uint64_t keep = l2_evict_last_policy();  // the window's partial lines stay until complete
#pragma unroll 4
    for (int k = t; k < kScTile; k += 256) {
      const long long d = (long long)s_is[k];
      if ((unsigned long long)d < (unsigned long long)ndst) st_keep(out + d, s_vs[k], keep);
    }
  } else {
    for (long long i = base + t; i < m; i += 256) {
      const long long d = (long long)is[i];
      if ((unsigned long long)d < (unsigned long long)ndst) out[d] = vs[i];
    }
  }
}

// the value check after a duplicate claim (k_scatter_verify for any index type)
template <typename I, typename E>
__global__ void __launch_bounds__(kGThreads) k_scatter_verify_i(const E* __restrict__ out, long long ndst,
                                                                 const long long* __restrict__ d_ndst,
                                                                 const I* __restrict__ is, const E* __restrict__ vs,
                                                                 long long m, const long long* __restrict__ d_m,
                                                                 LBHeader* hdr, ixg_status* st, int stmt, int site) {
  __shared__ bool s_last;
  if (((volatile LBHeader*)hdr)->dup == 0u) return;  // no destination claimed twice
  if (d_ndst) ndst = *d_ndst;
  if (d_m) m = *d_m;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const long long d = (long long)is[i];
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

// Duplicate detection by counting (the claims of k_scatter_pc<.., false>):
// the in-range pairs (*d_m, all of them in range after binning) claimed
// fewer distinct destinations than there are pairs iff some destination was
// claimed twice.  Grid-wide popcount of the bitmap; the last CTA decides.
__global__ void __launch_bounds__(kGThreads) k_claim_count(const uint32_t* __restrict__ claim, long long nwords,
                                                            const long long* __restrict__ d_m,
                                                            unsigned long long* __restrict__ acc, LBHeader* hdr) {
  __shared__ bool s_last;
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long c = 0;
  for (long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x; q < nwords; q += stride) c += __popc(claim[q]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) c += __shfl_xor_sync(0xffffffffu, c, d);
  if (lane_id() == 0 && c) atomicAdd(acc, c);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&hdr->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    const unsigned long long distinct = atomicAdd(acc, 0ull);
    if (distinct != (unsigned long long)*d_m) atomicExch(&hdr->dup, 1u);
    *acc = 0;
    hdr->done = 0;
  }
}

// ------------------------------------------------------------------ binning
// Locality probe: 64 sample runs of 256 consecutive indices; each warp
// counts the distinct 4096-destination windows among its 32 (match_any
// leaders).  Indices with locality -- C3's two interleaved monotone streams
// -- touch 2-4 windows per warp, a random permutation ~32.  *flag = 1 (bin)
// when the samples average more than 8 distinct windows per warp.
__global__ void __launch_bounds__(256) k_scatter_probe(const long long* __restrict__ is, long long m,
                                                       int* __restrict__ flag) {
  __shared__ int s_distinct;
  if (threadIdx.x == 0) s_distinct = 0;
  __syncthreads();
  int distinct = 0;
  for (int sIdx = 0; sIdx < 64; ++sIdx) {
    const long long start = (m - 256) * sIdx / 63;
    const long long w = is[start + threadIdx.x] >> kWinBits;
    const unsigned peers = __match_any_sync(0xffffffffu, w);
    distinct += (__ffs(peers) - 1 == lane_id()) ? 1 : 0;  // one leader per distinct window
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) distinct += __shfl_xor_sync(0xffffffffu, distinct, d);
  if (lane_id() == 0) atomicAdd(&s_distinct, distinct);
  __syncthreads();
  if (threadIdx.x == 0) *flag = s_distinct > 64 * 8 * 8 ? 1 : 0;  // 64 samples x 8 warps x 8 windows
}

// pass 0 (CHECKED / unknown counts): pairs per destination window
__global__ void __launch_bounds__(256) k_bin_count(const long long* __restrict__ is, long long m, long long ndst,
                                                   int shift, unsigned long long* __restrict__ counts) {
  __shared__ unsigned int s_cnt[kBinMax];
  for (int b = threadIdx.x; b < kBinMax; b += 256) s_cnt[b] = 0u;
  __syncthreads();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const long long d = __ldcs(&is[i]);
    if ((unsigned long long)d < (unsigned long long)ndst) atomicAdd(&s_cnt[d >> shift], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kBinMax; b += 256)
    if (s_cnt[b]) atomicAdd(&counts[b], (unsigned long long)s_cnt[b]);
}

// run starts (cursor[b]), ends (end[b]) and the in-range total (*d_m) of the
// B windows: from counts (exclusive scan) or, without counts, the window
// sizes of a bijection onto [0, ndst) (the Sc1 contract: window b receives
// exactly its own destinations)
__global__ void k_bin_layout(const unsigned long long* __restrict__ counts, int nb, long long ndst, int shift,
                             unsigned long long* __restrict__ cursor, unsigned long long* __restrict__ end,
                             long long* __restrict__ d_m) {
  if (threadIdx.x != 0) return;
  unsigned long long acc = 0;
  for (int b = 0; b < nb; ++b) {
    cursor[b] = acc;
    const unsigned long long w0 = (unsigned long long)b << shift;
    const unsigned long long sz = counts ? counts[b]
                                         : ((unsigned long long)ndst - w0 < (1ull << shift) ? (unsigned long long)ndst - w0
                                                                                            : (1ull << shift));
    acc += sz;
    end[b] = acc;
  }
  *d_m = (long long)acc;
}

// pass 1: partition the pairs by destination window (see the file comment);
// one CTA per 4096-pair tile, indices narrowed to u32 (ndst <= 2^32)
template <typename E>
struct BinSmem {  // staged pairs of one tile, window by window
  static constexpr int BYTES = kScTile * (4 + (int)sizeof(E) + 1);
};
template <typename E>
__global__ void __launch_bounds__(256) k_bin_partition(const long long* __restrict__ is, const E* __restrict__ vs,
                                                       long long m, long long ndst, int shift, int nb,
                                                       unsigned long long* __restrict__ cursor,
                                                       const unsigned long long* __restrict__ end,
                                                       uint32_t* __restrict__ bis, E* __restrict__ bvs) {
  constexpr int PER = kScTile / 256;  // 16 pairs per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  E* s_vs = reinterpret_cast<E*>(smem_raw);
  uint32_t* s_is = reinterpret_cast<uint32_t*>(smem_raw + kScTile * sizeof(E));
  uint8_t* s_b = smem_raw + kScTile * (sizeof(E) + 4);
  __shared__ unsigned int s_cnt[kBinMax];
  __shared__ unsigned int s_off[kBinMax];
  __shared__ unsigned long long s_base[kBinMax];
  __shared__ unsigned int s_wsum[8];
  const long long base = (long long)blockIdx.x * kScTile;
  const int t = threadIdx.x;
  for (int b = t; b < kBinMax; b += 256) s_cnt[b] = 0u;
  __syncthreads();
  long long d[PER];
  E v[PER];
  int slot[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {  // striped: coalesced loads
    const long long i = base + q * 256 + t;
    d[q] = i < m ? __ldcs(&is[i]) : -1;
    v[q] = i < m ? __ldcs(&vs[i]) : E(0);
    slot[q] = -1;
    if ((unsigned long long)d[q] < (unsigned long long)ndst) slot[q] = (int)atomicAdd(&s_cnt[d[q] >> shift], 1u);
  }
  __syncthreads();
  // exclusive scan of the window counts (nb <= 256: one per thread)
  const unsigned int c = t < nb ? s_cnt[t] : 0u;
  unsigned int inc = c;
#pragma unroll
  for (int k = 1; k < 32; k <<= 1) {
    const unsigned int o = __shfl_up_sync(0xffffffffu, inc, k);
    if (lane_id() >= k) inc += o;
  }
  if (lane_id() == 31) s_wsum[warp_id()] = inc;
  __syncthreads();
  unsigned int wpre = 0;
  for (int w = 0; w < warp_id(); ++w) wpre += s_wsum[w];
  if (t < nb) {
    s_off[t] = wpre + inc - c;
    s_base[t] = c ? atomicAdd(&cursor[t], (unsigned long long)c) : 0ull;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    if (slot[q] >= 0) {
      const int b = (int)(d[q] >> shift);
      const unsigned int p = s_off[b] + (unsigned int)slot[q];
      s_is[p] = (uint32_t)d[q];
      s_vs[p] = v[q];
      s_b[p] = (uint8_t)b;
    }
  }
  __syncthreads();
  const unsigned int total = s_wsum[0] + s_wsum[1] + s_wsum[2] + s_wsum[3] + s_wsum[4] + s_wsum[5] + s_wsum[6] + s_wsum[7];
  for (unsigned int p = t; p < total; p += 256) {  // each window's run is contiguous in s_* and in the output
    const int b = s_b[p];
    const unsigned long long g = s_base[b] + (p - s_off[b]);
    if (g < end[b]) {  // a run never outgrows its window (always true under the layout's contract)
      bis[g] = s_is[p];
      bvs[g] = s_vs[p];
    }
  }
}

}  // namespace ixg
