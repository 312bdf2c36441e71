// abi.cu -- the extern "C" entry points of libixgpu.so (include/ixgpu.h).
//
// Each function validates its arguments, lays out its workspace with a bump
// allocator (the same code path sizes it for ixg_ws_bytes), picks the fused
// ELIDED kernel or the materialising CHECKED sequence from the site bits,
// and enqueues everything on the caller's stream.  No host synchronisation.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <utility>
#include <vector>

#include "k_generic.cuh"
#include "k_stream.cuh"
#include "k_big.cuh"
#include "k_vm.cuh"
#include "k_contract.cuh"
#include "k_scatter.cuh"

using namespace ixg;

namespace {

std::atomic<unsigned long long> g_launches{0};

// ---- kernel timer (ixg_timer_start/stop): event pairs around one family
struct Timer {
  int target = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pool;
  size_t used = 0;
} g_timer;

struct TimedLaunch {
  cudaEvent_t stop = nullptr;
  cudaStream_t s;
  TimedLaunch(int kid, cudaStream_t s_) : s(s_) {
    if (g_timer.target != kid) return;
    if (g_timer.used == g_timer.pool.size()) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      g_timer.pool.emplace_back(a, b);
    }
    auto& pr = g_timer.pool[g_timer.used++];
    cudaEventRecord(pr.first, s);
    stop = pr.second;
  }
  ~TimedLaunch() {
    if (stop) cudaEventRecord(stop, s);
  }
};

constexpr size_t kHdrBlock = 8 * 256;  // fixed-offset look-back headers (8 channels)

struct WS {
  char* base;
  size_t off;
  bool dry;
  explicit WS(void* p) : base((char*)p), off(kHdrBlock), dry(p == nullptr) {}
  void* take(size_t bytes, size_t align = 256) {
    off = (off + align - 1) / align * align;
    void* p = dry ? nullptr : base + off;
    off += bytes ? bytes : 1;
    return p;
  }
  LBHeader* hdr(int i) const { return dry ? nullptr : (LBHeader*)(base + i * 256); }
  LBChan chan(int i, long long tiles) {
    LBChan c;
    const size_t t = (size_t)(tiles > 0 ? tiles : 1);
    c.hdr = hdr(i);
    c.slot = (ulonglong2*)take(t * sizeof(ulonglong2) * kSlotStride);
    return c;
  }
};

inline long long tiles_of(long long n, int tile) { return (n + tile - 1) / tile; }
// + slack: readers fetch whole windows past the last word (k_filter_b kSeg
// bulk-loads TILE/32 + 12 words from the tile's first flag word)
inline size_t bitmap_bytes(long long nbits) { return (size_t)((nbits + 31) / 32 + 2 + 512) * 4; }
inline int grid_for(long long work, int per_block = kGThreads) {
  long long g = (work + per_block - 1) / per_block;
  long long cap = (long long)num_sms() * 8;
  if (g > cap) g = cap;
  return (int)(g > 0 ? g : 1);
}
inline cudaStream_t S(void* s) { return (cudaStream_t)s; }
inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
// look-back slots for the big-tile kernels of either element width
inline long long lb_tiles(long long n) { return tiles_of(n, std::min(Big<int32_t>::TILE, Big<long long>::TILE)); }
inline bool aligned32(const void* p) { return ((uintptr_t)p & 31u) == 0; }

#define LAUNCHED() g_launches.fetch_add(1, std::memory_order_relaxed)
#define CHECK_LAUNCH()                          \
  do {                                          \
    cudaError_t e__ = cudaGetLastError();       \
    if (e__ != cudaSuccess) return cuda_rc(e__); \
  } while (0)

// The dynamic shared-memory opt-in is a per-DEVICE attribute of a kernel:
// set it once per (call site, device) -- `done` is that call site's bitmask
// of devices already configured.
template <typename K>
void allow_smem(K kernel, int bytes, std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ULL << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  done.fetch_or(bit, std::memory_order_acq_rel);
}

// ------------------------------------------------------------------ pieces
// per-launch nonce for look-back slots (lookback.cuh): 24 bits, never 0
std::atomic<uint32_t> g_nonce{0};
inline uint32_t next_nonce() {
  uint32_t v;
  do {
    v = (g_nonce.fetch_add(1, std::memory_order_relaxed) + 1) & kNonceMask;
  } while (v == 0);
  return v;
}

// IXG_PDL=0: launch the big-tile kernels without programmatic dependent launch (A/B)
inline bool pdl_enabled() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("IXG_PDL");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  return mode == 1;
}

// n = element count, or the capacity when d_n (device count) is given;
// pdl: launched as a programmatic dependent of the previous kernel (k_scan
// waits for it in-kernel before touching anything)
template <class M, class Src, class Epi>
int launch_scan(long long n, Src src, Epi epi, LBChan ch, cudaStream_t s, const long long* d_n = nullptr,
                bool pdl = false) {
  if (n <= 0) return IXG_OK;
  TimedLaunch tl(IXG_K_SCAN, s);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)tiles_of(n, kGTile));
  cfg.blockDim = dim3(kGThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = (pdl && pdl_enabled()) ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_scan<M, Src, Epi>, n, d_n, src, epi, ch, next_nonce());
  LAUNCHED();
  if (e != cudaSuccess) return cuda_rc(e);
  CHECK_LAUNCH();
  return IXG_OK;
}

template <typename E>
int launch_fill(E* out, long long n, const long long* d_n, E v, cudaStream_t s) {
  k_fill<E><<<grid_for(d_n ? (long long)num_sms() * 8 * kGThreads : n), kGThreads, 0, s>>>(out, n, d_n, v);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

// binned-scatter geometry for ndst destinations of E: window shift (32 MB
// windows) and window count; nb == 0 when binning does not apply
template <typename E>
inline void bin_geometry(long long ndst, int* shift, int* nb) {
  int sh = sizeof(E) == 4 ? 21 : 20;  // 8 MB destination windows (2^29 int32: 64.. 256 windows; measured
                                      // 6.45 ms against 6.74 / 6.93 for 16 / 32 MB windows)
  if (const char* e = getenv("IXG_BIN_SHIFT")) sh = atoi(e);  // tests: many windows at small sizes
  *shift = sh;
  *nb = 0;
  if (ndst <= 0 || ndst > (1LL << 32)) return;  // u32 binned indices
  while (((ndst - 1) >> sh) + 1 > kBinMax) ++sh;
  *shift = sh;
  *nb = (int)(((ndst - 1) >> sh) + 1);
}

// checked/elided scatter of m pairs into out[0..ndst) (ndst from d_ndst when
// given).  layout: IXG_SCATTER_DIRECT, or IXG_SCATTER_BINNED (pairs first
// partitioned by destination window; ndst <= 2^32 and a host-known ndst).
// IXG_SCATTER_SA=0: the CHECKED direct scatter with searched claim windows
// and per-thread window caches (k_scatter_pc) instead of the set-associative
// windows (k_scatter_sa), for A/B
inline bool scatter_sa_enabled() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("IXG_SCATTER_SA");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  return mode == 1;
}

template <typename E>
int launch_scatter(E* out, long long ndst, const long long* d_ndst, long long ndst_cap, const long long* is,
                   const E* vs, long long m, uint32_t bits, int stmt, int site, ixg_status* st, WS& ws,
                   int hdr_idx, cudaStream_t s, int layout = IXG_SCATTER_DIRECT) {
  const bool check = (bits & IXG_V_CONFLICT) != 0;
  int shift = 0, nb = 0;
  if (layout == IXG_SCATTER_BINNED && !d_ndst) bin_geometry<E>(ndst, &shift, &nb);
  const bool binned = nb > 1;
  uint32_t* claim = nullptr;
  if (check) claim = (uint32_t*)ws.take(bitmap_bytes(ndst_cap));
  unsigned long long *counts = nullptr, *cursor = nullptr, *end = nullptr;
  long long* d_m = nullptr;
  uint32_t* bis = nullptr;
  E* bvs = nullptr;
  if (layout == IXG_SCATTER_BINNED) {  // sized whether or not this call bins (ixg_ws_bytes)
    counts = (unsigned long long*)ws.take(3 * kBinMax * 8 + 64);
    cursor = counts + kBinMax;
    end = cursor + kBinMax;
    d_m = (long long*)(end + kBinMax);
    bis = (uint32_t*)ws.take((size_t)(m > 0 ? m : 1) * 4);
    bvs = (E*)ws.take((size_t)(m > 0 ? m : 1) * sizeof(E));
  }
  if (ws.dry || m <= 0) return IXG_OK;
  LBHeader* hdr = ws.hdr(hdr_idx);
  if (check) {
    cudaMemsetAsync(claim, 0, bitmap_bytes(ndst_cap), s);
    LAUNCHED();
  }
  const unsigned tiles = (unsigned)tiles_of(m, kScTile);
  if (binned) {
    // the window sizes of a bijection onto [0, ndst) when Sc1 holds (no init,
    // no checks: every destination written once), else pass 0 counts them
    const bool sc1 = (bits & (IXG_V_CONFLICT | IXG_V_INIT)) == 0;
    if (check) {  // the popcount accumulator of k_claim_count
      cudaMemsetAsync(counts + 3 * kBinMax + 4, 0, 8, s);
      LAUNCHED();
    }
    if (!sc1) {
      cudaMemsetAsync(counts, 0, kBinMax * 8, s);
      LAUNCHED();
      k_bin_count<<<grid_for(m), 256, 0, s>>>(is, m, ndst, shift, counts);
      LAUNCHED();
      CHECK_LAUNCH();
    }
    k_bin_layout<<<1, 32, 0, s>>>(sc1 ? nullptr : counts, nb, ndst, shift, cursor, end, d_m);
    LAUNCHED();
    CHECK_LAUNCH();
    {
      static std::atomic<unsigned long long> attr{0};
      allow_smem(k_bin_partition<E>, BinSmem<E>::BYTES, attr);
      TimedLaunch tl(IXG_K_BIN, s);
      k_bin_partition<E><<<tiles, 256, BinSmem<E>::BYTES, s>>>(is, vs, m, ndst, shift, nb, cursor, end, bis, bvs);
      LAUNCHED();
      CHECK_LAUNCH();
    }
    TimedLaunch tl(IXG_K_SCATTER, s);
    if (check) {
      static std::atomic<unsigned long long> attr{0};
      allow_smem(k_scatter_pc<uint32_t, E, false>, PcSmem<uint32_t, E>::BYTES, attr);
      k_scatter_pc<uint32_t, E, false><<<tiles, 256, PcSmem<uint32_t, E>::BYTES, s>>>(out, ndst, nullptr, bis, bvs, m,
                                                                                      d_m, claim, hdr);
    } else {
      static std::atomic<unsigned long long> attr{0};
      allow_smem(k_scatter_ti<uint32_t, E>, PcSmem<uint32_t, E>::BYTES, attr);
      k_scatter_ti<uint32_t, E><<<tiles, 256, PcSmem<uint32_t, E>::BYTES, s>>>(out, ndst, nullptr, bis, bvs, m, d_m);
    }
    LAUNCHED();
    CHECK_LAUNCH();
    if (check) {
      const long long nwords = (ndst + 31) / 32;
      k_claim_count<<<grid_for(nwords / 4 + 1), kGThreads, 0, s>>>(claim, nwords, d_m, counts + 3 * kBinMax + 4, hdr);
      LAUNCHED();
      CHECK_LAUNCH();
      k_scatter_verify_i<uint32_t, E><<<grid_for(m), kGThreads, 0, s>>>(out, ndst, nullptr, bis, bvs, m, d_m, hdr, st,
                                                                       stmt, site);
      LAUNCHED();
      CHECK_LAUNCH();
    }
    return IXG_OK;
  }
  {
    TimedLaunch tl(IXG_K_SCATTER, s);
    static int mode = -1;
    if (mode < 0) {
      const char* e = getenv("IXG_SCATTER");
      mode = e ? atoi(e) : 0;
    }
    // TMA-staged tiles walked striped (each warp store covers 32 consecutive
    // sources); CHECKED claims through the shared-memory windows
    // (k_scatter_pc); IXG_SCATTER=1: the register-blocked kernels for A/B
    if (mode == 0 && aligned16(is) && aligned16(vs)) {
      if (check && scatter_sa_enabled()) {
        static std::atomic<unsigned long long> attr{0};
        allow_smem(k_scatter_sa<E>, PcSmem<long long, E>::BYTES, attr);
        k_scatter_sa<E><<<tiles, 256, PcSmem<long long, E>::BYTES, s>>>(out, ndst, d_ndst, is, vs, m, claim, hdr);
      } else if (check) {
        static std::atomic<unsigned long long> attr{0};
        allow_smem(k_scatter_pc<long long, E>, PcSmem<long long, E>::BYTES, attr);
        k_scatter_pc<long long, E><<<tiles, 256, PcSmem<long long, E>::BYTES, s>>>(out, ndst, d_ndst, is, vs, m,
                                                                                  nullptr, claim, hdr);
      } else {
        static std::atomic<unsigned long long> attr{0};
        allow_smem(k_scatter_t<E>, ScSmem<E>::BYTES, attr);
        k_scatter_t<E><<<tiles, 256, ScSmem<E>::BYTES, s>>>(out, ndst, d_ndst, is, vs, m, 0, claim, hdr);
      }
    } else if (aligned32(is) && aligned32(vs))
      k_scatter_v<E><<<grid_for(m / 8 + 1, 256), 256, 0, s>>>(out, ndst, d_ndst, is, vs, m, check ? 1 : 0, claim,
                                                               hdr);
    else
      k_scatter<E><<<grid_for(m), kGThreads, 0, s>>>(out, ndst, d_ndst, is, vs, m, check ? 1 : 0, claim, hdr);
  }
  LAUNCHED();
  CHECK_LAUNCH();
  if (check) {
    k_scatter_verify<E><<<grid_for(m), kGThreads, 0, s>>>(out, ndst, d_ndst, is, vs, m, hdr, st, stmt, site);
    LAUNCHED();
    CHECK_LAUNCH();
  }
  return IXG_OK;
}

// --------------------------------------------------------------- filter
// the sharded partition2 reads xs once and places both classes (default
// tiles); IXG_PEER_DUAL=k (1..3) the same on k-chunk tiles, =0 the
// two-segment form over xs (A/B)
inline int peer_dual_chunks() {
  static int mode = -2;
  if (mode == -2) {
    const char* e = getenv("IXG_PEER_DUAL");
    mode = (e && e[0] >= '0' && e[0] <= '3') ? e[0] - '0' : -1;
  }
  return mode;
}

// IXG_BIG_SCAN=0: the CHECKED index scans on the generic k_scan instead of
// the big-tile kernel (A/B)
inline bool big_scan_enabled() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("IXG_BIG_SCAN");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  return mode == 1;
}

// IXG_SEG_SPLIT=1: C2 as two passes (filter, then sgmSum over ys) for A/B
inline bool seg_split_mode() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("IXG_SEG_SPLIT");
    mode = (e && e[0] == '1') ? 1 : 0;
  }
  return mode == 1;
}

template <typename T, bool kByCs, bool kSeg = false, typename Z = T, int NS = 1, bool kPeer = false, int CHO = 0>
int launch_filter_b(const T* xs, const uint8_t* cs, long long n, const ixg_pred& p, T* ys, LBChan ch,
                    long long* d_count, cudaStream_t s, Z* zs = nullptr, const uint32_t* segbits = nullptr,
                    long long out_base = 0, LBChan ch2 = LBChan{nullptr, nullptr}, ixg_status* st = nullptr,
                    const ixg_pred& q = ixg_pred{}, const PeerOut<T>& po = PeerOut<T>{}) {
  auto kern = k_filter_b<T, kByCs, kSeg, Z, NS, kPeer, CHO>;
  using B = Big<T, CHO>;
  constexpr int smem = B::SMEM;
  static std::atomic<unsigned long long> attr{0};
  allow_smem(kern, smem, attr);
  TimedLaunch tl(NS > 1 ? IXG_K_PLACE : IXG_K_FILTER_FUSED, s);
  const long long seg_tiles = tiles_of(n, B::TILE);
  // programmatic dependent launch: the CTAs become resident while the
  // previous kernel of the stream drains (k_filter_b waits for it itself)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(NS * seg_tiles));
  cfg.blockDim = dim3(kBT + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  la[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = la;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, xs, cs, n, p, ys, ch, next_nonce(), d_count, zs, segbits, out_base,
                                     ch2, st, q, seg_tiles, po);
  LAUNCHED();
  if (e != cudaSuccess) return cuda_rc(e);
  CHECK_LAUNCH();
  return IXG_OK;
}

// zs = sgmSum over the first *d_n elements of vs (capacity n)
template <typename T, typename Z, class M = SegOp, class F = ScanId>
int launch_segsum_b(const T* vs, long long n, const long long* d_n, const uint32_t* bits, long long flag_base, Z* zs,
                    LBChan ch, long long carry_v, int carry_f, longlong2* d_total, ixg_status* st, cudaStream_t s,
                    const long long* d_flag_base = nullptr, F fn = F{}) {
  auto kern = k_segsum_b<T, Z, M, F>;
  using B = Big<T, F::kCH ? F::kCH : kSegsumCH<T, Z>>;
  static std::atomic<unsigned long long> attr{0};
  allow_smem(kern, B::SMEM, attr);
  TimedLaunch tl(IXG_K_SEGSUM, s);
  if constexpr (F::kTrigger) {  // a programmatic dependent of the previous kernel (the bitmap clear)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tiles_of(n, B::TILE));
    cfg.blockDim = dim3(kBT + 32);
    cfg.dynamicSmemBytes = B::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute la[1];
    la[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    la[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = la;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, vs, n, d_n, bits, flag_base, d_flag_base, zs, ch, next_nonce(),
                                       carry_v, carry_f, d_total, st, fn);
    LAUNCHED();
    if (e != cudaSuccess) return cuda_rc(e);
  } else {
    kern<<<(unsigned)tiles_of(n, B::TILE), kBT + 32, B::SMEM, s>>>(vs, n, d_n, bits, flag_base, d_flag_base, zs, ch,
                                                                    next_nonce(), carry_v, carry_f, d_total, st, fn);
    LAUNCHED();
  }
  CHECK_LAUNCH();
  return IXG_OK;
}

// mkFlags into a cleared bitmap: the big-tile scan (TMA tiles, dedicated
// look-back warp, 8 K shape values per tile) setting the start bits; with
// IXG_MKF_BIG=0 the generic k_scan (A/B)
inline bool mkf_big_enabled() {
  static int mode = -1;
  if (mode < 0) {
    const char* e = getenv("IXG_MKF_BIG");
    mode = (e && e[0] == '0') ? 0 : 1;
  }
  return mode == 1;
}
int launch_mkflags(const long long* shape, long long m, uint32_t* bits, long long nbits, const long long* d_nbits,
                   LBChan c, cudaStream_t s, ixg_status* st = nullptr, const long long* d_lo = nullptr) {
  const bool big = mkf_big_enabled() && aligned16(shape) && aligned16(bits) && m > 0;
  if (big) {  // the clear heads a programmatic-launch chain (see k_bitmap_zero)
    k_bitmap_zero<<<grid_for((nbits + 127) / 128), kGThreads, 0, s>>>(
        bits, (long long)(bitmap_bytes(nbits) / 4), d_nbits);
    LAUNCHED();
    CHECK_LAUNCH();
  } else if (d_nbits) {
    k_bitmap_clear<<<grid_for((nbits + 31) / 32 + 514), kGThreads, 0, s>>>(bits, d_nbits);
    LAUNCHED();
    CHECK_LAUNCH();
  } else {
    cudaMemsetAsync(bits, 0, bitmap_bytes(nbits), s);
    LAUNCHED();
  }
  if (m <= 0) return IXG_OK;
  if (big) {
    ScanSegStartBits fn{};
    fn.bits = bits;
    fn.nb = nbits;
    fn.d_nb = d_nbits;
    fn.d_lo = d_lo;
    return launch_segsum_b<long long, long long, SumOp>(shape, m, nullptr, nullptr, 0, nullptr, c, 0, 0, nullptr,
                                                        st, s, nullptr, fn);
  }
  return launch_scan<SumOp>(m, SrcArrT<long long>{shape},
                            EpiSegStarts{m, shape, nullptr, bits, nbits, d_nbits, nullptr, st, d_lo}, c, s);
}

// filter / filter_by on element type T.  Sites: 0 = offs[n-1], 1 = scatter.
template <typename T>
int do_filter(const T* xs, const uint8_t* cs, long long n, const ixg_pred* p, T* ys, long long* d_count,
              uint32_t variant, ixg_status* st, WS& ws, cudaStream_t s) {
  const uint32_t sb = IXG_SITE_BITS(variant, 1);
  const bool fused = (sb & (IXG_V_CONFLICT | IXG_V_INIT)) == 0;  // Sc1 proved
  ixg_pred pp = p ? *p : ixg_pred{IXG_PRED_TRUE, 0, 0, 0};
  if (fused) {
    LBChan c0 = ws.chan(0, lb_tiles(n));
    if (ws.dry) return IXG_OK;
    if (n <= 0) return cuda_rc(cudaMemsetAsync(d_count, 0, sizeof(long long), s));
    if (!aligned16(xs) || !aligned16(ys)) return IXG_BADARG;
    if (cs) return launch_filter_b<T, true>(xs, cs, n, pp, ys, c0, d_count, s);
    return launch_filter_b<T, false>(xs, cs, n, pp, ys, c0, d_count, s);
  }
  // CHECKED: offs/inds materialised (filter.ixl:10-12), then the scatter
  // into `replicate count 0` with the dynamic checks (filter.ixl:13-14).
  LBChan c0 = ws.chan(0, tiles_of(n, kGTile));
  long long* inds = (long long*)ws.take((size_t)(n > 0 ? n : 1) * 8);
  if (ws.dry) return launch_scatter<T>(ys, 0, d_count, n, inds, xs, n, sb, 1, 1, st, ws, 1, s);
  if (n <= 0) return cuda_rc(cudaMemsetAsync(d_count, 0, sizeof(long long), s));
  int rc;
  if (!cs && big_scan_enabled() && aligned16(xs) && aligned32(inds)) {
    // the big-tile scan (TMA tiles, dedicated look-back warp) with the
    // predicate in front and the index formula behind
    ScanFilterInds<T> fn{};
    fn.pb.p = pp;
    fn.d_count = d_count;
    rc = launch_segsum_b<T, long long, SumOp>(xs, n, nullptr, nullptr, 0, inds, c0, 0, 0, nullptr, nullptr, s, nullptr,
                                              fn);
  } else {
    rc = launch_scan<SumOp>(n, SrcPredT<T>{xs, cs, pp}, EpiFilterInds{inds, d_count}, c0, s);
  }
  if (rc) return rc;
  if (sb & IXG_V_INIT) {
    if ((rc = launch_fill<T>(ys, 0, d_count, T(0), s))) return rc;
  }
  return launch_scatter<T>(ys, 0, d_count, n, inds, xs, n, sb, 1, 1, st, ws, 1, s);
}

// ------------------------------------------------------------ partition2/3
template <typename T, int kClasses>
int do_partition(const T* xs, long long n, const ixg_pred* p, const ixg_pred* q, T* ys, long long* d_tot,
                 uint32_t variant, ixg_status* st, WS& ws, cudaStream_t s) {
  const int scatter_site = kClasses == 2 ? 1 : 2;
  const uint32_t sb = IXG_SITE_BITS(variant, scatter_site);
  const bool fused = (sb & (IXG_V_CONFLICT | IXG_V_INIT)) == 0;
  const ixg_pred pp = *p;
  const ixg_pred qq = q ? *q : ixg_pred{IXG_PRED_FALSE, 0, 0, 0};
  const int cgrid = grid_for(n / (16 / (int)sizeof(T)) + 1);
  long long* partials = (long long*)ws.take((size_t)cgrid * 2 * 8);
  if (fused) {
    LBChan c0 = ws.chan(0, std::max(lb_tiles(n), kClasses * tiles_of(n, Big<long long>::TILE)));
    if (ws.dry) return IXG_OK;
    if (n <= 0) return cuda_rc(cudaMemsetAsync(d_tot, 0, sizeof(long long) * (kClasses - 1), s));
    if (!aligned16(xs) || !aligned16(ys)) return IXG_BADARG;
    // one pass: kClasses segments of big tiles on one look-back chain
    int rc = launch_filter_b<T, false, false, T, kClasses>(xs, nullptr, n, pp, ys, c0, d_tot, s, nullptr, nullptr, 0,
                                                           LBChan{nullptr, nullptr}, nullptr, qq);
    if (rc || kClasses == 2) return rc;
    k_sub_first<<<1, 1, 0, s>>>(d_tot);  // d_tot[1] held m1 + m2
    LAUNCHED();
    CHECK_LAUNCH();
    return IXG_OK;
  }
  // CHECKED: indices materialised exactly as partition2.ixl:9-16 /
  // partition3.ixl:12-24, then the checked scatter into `replicate n 0`.
  LBChan c0 = ws.chan(0, tiles_of(n, kGTile));
  long long* inds = (long long*)ws.take((size_t)(n > 0 ? n : 1) * 8);
  if (ws.dry) return launch_scatter<T>(ys, n, nullptr, n, inds, xs, n, sb, scatter_site, scatter_site, st, ws, 1, s);
  if (n <= 0) return cuda_rc(cudaMemsetAsync(d_tot, 0, sizeof(long long) * (kClasses - 1), s));
  {
    TimedLaunch tl(IXG_K_CLASS_COUNT, s);
    k_class_count<T, kClasses><<<cgrid, kSThreads, 0, s>>>(xs, n, pp, qq, partials, ws.hdr(5), d_tot);
  }
  LAUNCHED();
  CHECK_LAUNCH();
  int rc;
  if constexpr (kClasses == 2) {
    if (big_scan_enabled() && aligned16(xs) && aligned32(inds)) {
      ScanPart2Inds<T> fn{};
      fn.pb.p = pp;
      fn.d_nt = d_tot;
      rc = launch_segsum_b<T, long long, SumOp>(xs, n, nullptr, nullptr, 0, inds, c0, 0, 0, nullptr, nullptr, s,
                                                nullptr, fn);
    } else {
      rc = launch_scan<SumOp>(n, SrcPredT<T>{xs, nullptr, pp}, EpiPart2Inds{d_tot, inds}, c0, s);
    }
  } else {
    rc = launch_scan<Sum2Op>(n, SrcClass3T<T>{xs, pp, qq}, EpiPart3Inds{d_tot, inds}, c0, s);
  }
  if (rc) return rc;
  if (sb & IXG_V_INIT) {
    if ((rc = launch_fill<T>(ys, n, nullptr, T(0), s))) return rc;
  }
  return launch_scatter<T>(ys, n, nullptr, n, inds, xs, n, sb, scatter_site, scatter_site, st, ws, 1, s);
}

// --------------------------------------------------------------------- c2
// Sites: 0 = filter offs[n-1], 1 = filter scatter, 2 = mkFlags shape[i-1],
// 3 = mkFlags scatter.
template <typename T, typename Z>
int do_c2(const T* xs, long long n, const ixg_pred* p, const long long* shape, long long m, T* ys, Z* zs,
          long long* d_k, uint32_t variant, ixg_status* st, WS& ws, cudaStream_t s) {
  const uint32_t sb1 = IXG_SITE_BITS(variant, 1);
  const uint32_t sb3 = IXG_SITE_BITS(variant, 3);
  const bool fused = (sb1 & (IXG_V_CONFLICT | IXG_V_INIT)) == 0 && (sb3 & IXG_V_CONFLICT) == 0;
  const ixg_pred pp = *p;
  if (fused) {
    // mkFlags as a bitmap over the output positions: `replicate k 0` is the
    // memset (k <= n), the Ss2-proved scatter of ones is an atomicOr per
    // segment start (no conflict check), starts >= k are never read.
    uint32_t* bits = (uint32_t*)ws.take(bitmap_bytes(n));
    LBChan cs = ws.chan(2, tiles_of(m, kGTile));
    LBChan c0 = ws.chan(0, lb_tiles(n));
    LBChan c1 = ws.chan(1, lb_tiles(n));
    if (ws.dry) return IXG_OK;
    if (n <= 0) return cuda_rc(cudaMemsetAsync(d_k, 0, sizeof(long long), s));
    if (!aligned16(xs) || !aligned16(ys) || !aligned16(zs)) return IXG_BADARG;
    // the fused kernel is the mkFlags scan's programmatic dependent: its CTAs
    // load, count and compact while the scan runs and wait only before they
    // read the bitmap (a kernel clearing the bitmap instead of the memset, to
    // chain all three launches, measured no faster)
    int rc = launch_mkflags(shape, m, bits, n, nullptr, cs, s, st);  // clear + scan
    if (rc) return rc;
    if constexpr (sizeof(Z) == sizeof(T)) {
      if (!seg_split_mode()) {
        // one pass: filter + sgmSum in shared memory; the carry across
        // tiles takes a second look-back chain (channel 1)
        return launch_filter_b<T, false, true, Z>(xs, nullptr, n, pp, ys, c0, d_k, s, zs, bits, 0, c1, st);
      }
    }
    // two passes: ys = filter p xs, then zs = sgmSum flags ys over the k
    // outputs (the flag of output j is bit j of the bitmap)
    if ((rc = launch_filter_b<T, false>(xs, nullptr, n, pp, ys, c0, d_k, s))) return rc;
    return launch_segsum_b<T, Z>(ys, n, d_k, bits, 0, zs, c1, 0, 0, nullptr, st, s);
  }
  // CHECKED: filter (checked), mkFlags with materialised ind/flags arrays
  // and the checked scatter of `replicate m 1`, sgmSum as a 2-ary scan.
  int rc = do_filter<T>(xs, nullptr, n, p, ys, d_k, variant, st, ws, s);
  if (rc) return rc;
  LBChan cs = ws.chan(2, tiles_of(m, kGTile));
  LBChan cz = ws.chan(3, tiles_of(n, kGTile));
  long long* ind = (long long*)ws.take((size_t)(m > 0 ? m : 1) * 8);
  long long* ones = (long long*)ws.take((size_t)(m > 0 ? m : 1) * 8);
  long long* flags = (long long*)ws.take((size_t)(n > 0 ? n : 1) * 8);
  if (ws.dry) return launch_scatter<long long>(flags, 0, d_k, n, ind, ones, m, sb3, 3, 3, st, ws, 4, s);
  if (n <= 0) return IXG_OK;
  if ((rc = launch_scan<SumOp>(m, SrcArrT<long long>{shape}, EpiSegStarts{m, shape, ind, nullptr, 0, nullptr, nullptr, st}, cs, s)))
    return rc;
  if ((rc = launch_fill<long long>(ones, m, nullptr, 1LL, s))) return rc;
  if ((rc = launch_fill<long long>(flags, 0, d_k, 0LL, s))) return rc;
  if ((rc = launch_scatter<long long>(flags, 0, d_k, n, ind, ones, m, sb3, 3, 3, st, ws, 4, s))) return rc;
  // sgmSum over the k = *d_k outputs (a capacity-n grid; tiles past k retire)
  if (big_scan_enabled() && aligned16(ys) && aligned32(zs) && aligned32(flags)) {
    SegFlagArr fn{};
    fn.fa = flags;
    return launch_segsum_b<T, Z, SegOp>(ys, n, d_k, nullptr, 0, zs, cz, 0, 0, nullptr, st, s, nullptr, fn);
  }
  return launch_scan<SegOp>(n, SrcSegT<long long, T>{flags, ys},
                            EpiSegOut{sizeof(Z) == 4 ? IXG_I32 : IXG_I64, zs, nullptr, st}, cz, s, d_k);
}

}  // namespace

// =====================================================================
extern "C" {

int ixg_version(void) { return 1; }

int ixg_device_check(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return IXG_NODEVICE;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return (major == 10 && minor == 0) ? IXG_OK : IXG_NODEVICE;
}

unsigned long long ixg_launch_count(void) { return g_launches.load(); }

int ixg_trace_read(unsigned long long* host, size_t count) {
#ifdef IXG_TRACE
  const size_t cap = sizeof(g_trace) / sizeof(g_trace[0]);
  if (count > cap) count = cap;
  return cuda_rc(cudaMemcpyFromSymbol(host, g_trace, count * sizeof(unsigned long long)));
#else
  (void)host;
  (void)count;
  return IXG_BADARG;
#endif
}

int ixg_timer_start(int kernel_id) {
  g_timer.target = kernel_id;
  g_timer.used = 0;
  return IXG_OK;
}

int ixg_timer_stop(double* total_ms, int64_t* launches) {
  double tot = 0.0;
  for (size_t i = 0; i < g_timer.used; ++i) {
    auto& pr = g_timer.pool[i];
    cudaError_t e = cudaEventSynchronize(pr.second);
    if (e != cudaSuccess) return cuda_rc(e);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.first, pr.second);
    tot += ms;
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (int64_t)g_timer.used;
  g_timer.target = 0;
  g_timer.used = 0;
  return IXG_OK;
}

int ixg_ws_init(void* ws, size_t ws_bytes, void* stream) {
  if (!ws) return IXG_BADARG;
  LAUNCHED();
  return cuda_rc(cudaMemsetAsync(ws, 0, ws_bytes, S(stream)));
}

int ixg_status_init(ixg_status* st, void* stream) {
  if (!st) return IXG_BADARG;
  ixg_status h;
  h.first = ~0ULL;
  h.codes = 0;
  h.flags = 0;
  LAUNCHED();
  return cuda_rc(cudaMemcpyAsync(st, &h, sizeof(h), cudaMemcpyHostToDevice, S(stream)));
}

size_t ixg_ws_bytes(int op, int64_t n, int64_t m) {
  WS ws(nullptr);
  ixg_pred p{IXG_PRED_TRUE, 0, 0, 0};
  switch (op) {
    case IXG_OP_SCAN: ws.chan(0, tiles_of(n, kGTile)); break;
    case IXG_OP_SEGSCAN: ws.chan(0, tiles_of(n, kGTile)); break;
    case IXG_OP_SCATTER: ws.take(bitmap_bytes(m)); break;  // n = pairs, m = ndst
    case IXG_OP_SCATTER_BINNED:  // the claim bitmap + the binned (u32, i64) pairs
      launch_scatter<long long>(nullptr, m, nullptr, m, nullptr, nullptr, n, IXG_V_CONFLICT, 0, 0, nullptr, ws, 1,
                                0, IXG_SCATTER_BINNED);
      break;
    case IXG_OP_FILTER:
      do_filter<int64_t>(nullptr, nullptr, n, &p, nullptr, nullptr, IXG_VARIANT_CHECKED, nullptr, ws, 0);
      {
        WS w2(nullptr);
        do_filter<int64_t>(nullptr, nullptr, n, &p, nullptr, nullptr, 0, nullptr, w2, 0);
        if (w2.off > ws.off) ws.off = w2.off;
      }
      break;
    case IXG_OP_PARTITION2:
    case IXG_OP_PARTITION3: {
      do_partition<int64_t, 3>(nullptr, n, &p, &p, nullptr, nullptr, IXG_VARIANT_CHECKED, nullptr, ws, 0);
      WS w2(nullptr);
      do_partition<int64_t, 3>(nullptr, n, &p, &p, nullptr, nullptr, 0, nullptr, w2, 0);
      if (w2.off > ws.off) ws.off = w2.off;
      break;
    }
    case IXG_OP_C2: {
      do_c2<int64_t, int64_t>(nullptr, n, &p, nullptr, m, nullptr, nullptr, nullptr, IXG_VARIANT_CHECKED, nullptr,
                              ws, 0);
      WS w2(nullptr);
      do_c2<int64_t, int64_t>(nullptr, n, &p, nullptr, m, nullptr, nullptr, nullptr, 0, nullptr, w2, 0);
      if (w2.off > ws.off) ws.off = w2.off;
      break;
    }
    case IXG_OP_MKFLAGS:
      ws.chan(0, tiles_of(m, kGTile));
      ws.take((size_t)(m > 0 ? m : 1) * 8);
      ws.take((size_t)(m > 0 ? m : 1) * 8);
      ws.take(bitmap_bytes(n));  // n = k
      break;
    case IXG_OP_HIST: ws.take((size_t)(m > 0 ? m : 1) * 8); break;  // m = dlen: the bins' high words
    case IXG_OP_MKSGMDESCR:
      ws.chan(0, tiles_of(m, kGTile));
      ws.take((size_t)(m > 0 ? m : 1) * 8);
      ws.take(bitmap_bytes(n));  // n = destination capacity
      break;
    default: return 0;
  }
  return ws.off + 256;
}

int ixg_scan_add(int dt, const void* xs, int64_t n, int64_t ne, int exclusive, int64_t* out, void* ws,
                 size_t ws_bytes, ixg_status* st, void* stream) {
  if (n < 0 || (n > 0 && (!xs || !out))) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_SCAN, n, 0)) return IXG_BADARG;
  WS w(ws);
  LBChan c = w.chan(0, tiles_of(n, kGTile));
  // inclusive scans of int32 / int64: the big-tile sgmSum kernel without
  // flags (TMA-loaded 48 KB int32 tiles, one look-back per tile), `ne` as the
  // carry into the first tile; exclusive / u8 keep the generic k_scan
  // (k_segsum_b stores 32-byte vectors: `out` must be 32-byte aligned)
  if (!exclusive && n > 0 && (dt == IXG_I32 || dt == IXG_I64) && aligned16(xs) && aligned32(out)) {
    if (dt == IXG_I32)
      return launch_segsum_b<int32_t, long long, SumOp>((const int32_t*)xs, n, nullptr, nullptr, 0, (long long*)out, c,
                                                        ne, 0, nullptr, st, S(stream));
    return launch_segsum_b<long long, long long, SumOp>((const long long*)xs, n, nullptr, nullptr, 0, (long long*)out, c,
                                                         ne, 0, nullptr, st, S(stream));
  }
  const EpiScanOut epi{ne, exclusive, (long long*)out, st};
  if (dt == IXG_I32) return launch_scan<SumOp>(n, SrcArrT<int32_t>{(const int32_t*)xs}, epi, c, S(stream));
  if (dt == IXG_U8) return launch_scan<SumOp>(n, SrcArrT<uint8_t>{(const uint8_t*)xs}, epi, c, S(stream));
  return launch_scan<SumOp>(n, SrcArrT<long long>{(const long long*)xs}, epi, c, S(stream));
}

int ixg_reduce_add(int dt, const void* xs, int64_t n, int64_t* out, void* stream) {
  if (n < 0 || !out || (n > 0 && !xs)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  int rc = cuda_rc(cudaMemsetAsync(out, 0, 8, s));
  if (rc || n == 0) return rc;
  unsigned long long* o = reinterpret_cast<unsigned long long*>(out);
  if (dt == IXG_I32)
    k_reduce_add<int32_t><<<grid_for(n / 4 + 1), kGThreads, 0, s>>>((const int32_t*)xs, n, o);
  else if (dt == IXG_U8)
    k_reduce_add<uint8_t><<<grid_for(n / 16 + 1), kGThreads, 0, s>>>((const uint8_t*)xs, n, o);
  else
    k_reduce_add<long long><<<grid_for(n / 2 + 1), kGThreads, 0, s>>>((const long long*)xs, n, o);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_jagged_dest(const uint32_t* bits, int64_t n, const uint8_t* cs, const int64_t* tb, int64_t* dest,
                    void* stream) {
  if (n < 0 || (n > 0 && (!bits || !cs || !tb || !dest))) return IXG_BADARG;
  if (n == 0) return IXG_OK;
  k_jagged_dest<<<grid_for(n), kGThreads, 0, S(stream)>>>(bits, n, cs, (const long long*)tb, (long long*)dest);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_segscan_add(int dt_f, const void* flags, int dt_x, const void* xs, int64_t n, int f0, int64_t v0,
                    int64_t* out_v, uint8_t* out_f, void* ws, size_t ws_bytes, ixg_status* st, void* stream) {
  if (n < 0 || (n > 0 && (!flags || !xs || !out_v))) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_SEGSCAN, n, 0)) return IXG_BADARG;
  WS w(ws);
  LBChan c = w.chan(0, tiles_of(n, kGTile));
  (void)f0;
  (void)v0;
  if (f0 != 0 || v0 != 0) return IXG_BADARG;  // only the (false, 0) neutral of sgmSum is supported
  const EpiSegOut epi{IXG_I64, out_v, out_f, st};
  cudaStream_t s = S(stream);
  auto run = [&](auto fl) -> int {
    using EF = typename std::remove_const<typename std::remove_pointer<decltype(fl)>::type>::type;
    if (dt_x == IXG_I32) return launch_scan<SegOp>(n, SrcSegT<EF, int32_t>{fl, (const int32_t*)xs}, epi, c, s);
    if (dt_x == IXG_U8) return launch_scan<SegOp>(n, SrcSegT<EF, uint8_t>{fl, (const uint8_t*)xs}, epi, c, s);
    return launch_scan<SegOp>(n, SrcSegT<EF, long long>{fl, (const long long*)xs}, epi, c, s);
  };
  if (dt_f == IXG_U8) return run((const uint8_t*)flags);
  if (dt_f == IXG_I32) return run((const int32_t*)flags);
  return run((const long long*)flags);
}

int ixg_scatter(int dt, void* out, int64_t ndst, const int64_t* is, int64_t nis, const void* vs, int64_t nvs,
                uint32_t site_bits, int stmt, int site, int layout, ixg_status* st, void* ws, size_t ws_bytes,
                void* stream) {
  const long long m = nis < nvs ? nis : nvs;  // zip truncation, oracle.py:299
  if (ndst < 0 || m < 0 || (m > 0 && (!is || !vs)) || (ndst > 0 && !out)) return IXG_BADARG;
  if (layout != IXG_SCATTER_DIRECT && layout != IXG_SCATTER_BINNED) return IXG_BADARG;
  const long long need = layout == IXG_SCATTER_BINNED ? ixg_ws_bytes(IXG_OP_SCATTER_BINNED, m, ndst)
                                                      : ixg_ws_bytes(IXG_OP_SCATTER, m, ndst);
  if (((site_bits & IXG_V_CONFLICT) || layout == IXG_SCATTER_BINNED) && (long long)ws_bytes < need) return IXG_BADARG;
  WS w(ws);
  if (dt == IXG_I32)
    return launch_scatter<int32_t>((int32_t*)out, ndst, nullptr, ndst, (const long long*)is, (const int32_t*)vs, m,
                                   site_bits, stmt, site, st, w, 1, S(stream), layout);
  return launch_scatter<long long>((long long*)out, ndst, nullptr, ndst, (const long long*)is,
                                   (const long long*)vs, m, site_bits, stmt, site, st, w, 1, S(stream), layout);
}

int ixg_scatter_probe(const int64_t* is, int64_t m, int* d_flag, void* stream) {
  if (m < 0 || !d_flag || (m > 0 && !is)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  if (m < 512) return cuda_rc(cudaMemsetAsync(d_flag, 0, sizeof(int), s));
  k_scatter_probe<<<1, 256, 0, s>>>((const long long*)is, m, d_flag);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_gather(int dt, const void* arr, int64_t len, const int64_t* idx, int64_t n, void* out,
               uint32_t site_bits, int stmt, int site, ixg_status* st, void* stream) {
  if (n < 0 || (n > 0 && (!idx || !out))) return IXG_BADARG;
  if (n == 0) return IXG_OK;
  const int check = (site_bits & IXG_V_BOUNDS) ? 1 : 0;
  cudaStream_t s = S(stream);
  if (dt == IXG_I32)
    k_gather<int32_t><<<grid_for(n), kGThreads, 0, s>>>((const int32_t*)arr, len, (const long long*)idx, n,
                                                         (int32_t*)out, check, st, stmt, site);
  else if (dt == IXG_F64)
    k_gather<double><<<grid_for(n), kGThreads, 0, s>>>((const double*)arr, len, (const long long*)idx, n,
                                                        (double*)out, check, st, stmt, site);
  else
    k_gather<long long><<<grid_for(n), kGThreads, 0, s>>>((const long long*)arr, len, (const long long*)idx, n,
                                                           (long long*)out, check, st, stmt, site);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_hist(int op, int64_t ne, int64_t dlen, const int64_t* is, int64_t nis, const int64_t* vs, int64_t nvs,
             int64_t* out, void* ws, size_t ws_bytes, ixg_status* st, void* stream) {
  const long long m = nis < nvs ? nis : nvs;
  if (dlen < 0) dlen = 0;  // [ne] * negative == []
  if (op < 0 || op > 2 || m < 0 || (dlen > 0 && !out)) return IXG_BADARG;
  const bool add = op == IXG_HIST_ADD;
  if (add && dlen > 0 && (!ws || ws_bytes < ixg_ws_bytes(IXG_OP_HIST, 0, dlen))) return IXG_BADARG;
  cudaStream_t s = S(stream);
  WS w(ws);
  long long* hi = add ? (long long*)w.take((size_t)(dlen > 0 ? dlen : 1) * 8) : nullptr;
  int rc;
  if (dlen > 0 && (rc = launch_fill<long long>((long long*)out, dlen, nullptr, (long long)ne, s))) return rc;
  if (add && dlen > 0 && (rc = launch_fill<long long>(hi, dlen, nullptr, ne < 0 ? -1LL : 0LL, s))) return rc;
  if (m == 0 || dlen == 0) return IXG_OK;
  k_hist<<<grid_for(m), kGThreads, 0, s>>>(op, dlen, (const long long*)is, (const long long*)vs, m,
                                            (long long*)out, hi);
  LAUNCHED();
  CHECK_LAUNCH();
  if (add) {
    k_hist_check<<<grid_for(dlen), kGThreads, 0, s>>>((const long long*)out, hi, dlen, st);
    LAUNCHED();
    CHECK_LAUNCH();
  }
  return IXG_OK;
}

int ixg_fill(int dt, void* out, int64_t n, int64_t v, void* stream) {
  if (n <= 0) return IXG_OK;
  if (!out) return IXG_BADARG;
  if (dt == IXG_I32) return launch_fill<int32_t>((int32_t*)out, n, nullptr, (int32_t)v, S(stream));
  if (dt == IXG_U8) {
    LAUNCHED();
    return cuda_rc(cudaMemsetAsync(out, (int)(uint8_t)v, (size_t)n, S(stream)));
  }
  return launch_fill<long long>((long long*)out, n, nullptr, (long long)v, S(stream));
}

int ixg_iota(int64_t* out, int64_t n, void* stream) {
  if (n <= 0) return IXG_OK;
  k_iota<<<grid_for(n), kGThreads, 0, S(stream)>>>((long long*)out, n);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_filter(int dt, const void* xs, int64_t n, const ixg_pred* p, void* ys, int64_t* d_count, uint32_t variant,
               ixg_status* st, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !p || !d_count || (n > 0 && (!xs || !ys))) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_FILTER, n, 0)) return IXG_BADARG;
  WS w(ws);
  if (dt == IXG_I32)
    return do_filter<int32_t>((const int32_t*)xs, nullptr, n, p, (int32_t*)ys, (long long*)d_count, variant, st, w,
                              S(stream));
  return do_filter<int64_t>((const int64_t*)xs, nullptr, n, p, (int64_t*)ys, (long long*)d_count, variant, st, w,
                            S(stream));
}

int ixg_filter_by(int dt, const uint8_t* cs, const void* xs, int64_t n, void* ys, int64_t* d_count,
                  uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !d_count || (n > 0 && (!cs || !xs || !ys))) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_FILTER, n, 0)) return IXG_BADARG;
  WS w(ws);
  if (dt == IXG_I32)
    return do_filter<int32_t>((const int32_t*)xs, cs, n, nullptr, (int32_t*)ys, (long long*)d_count, variant, st,
                              w, S(stream));
  return do_filter<int64_t>((const int64_t*)xs, cs, n, nullptr, (int64_t*)ys, (long long*)d_count, variant, st, w,
                            S(stream));
}

// ---- sharded partition2 with the exchange fused into the kernel (C5) ----
int ixg_partition_counts(int dt, const void* xs, int64_t n, const ixg_pred* p, const ixg_pred* q, int classes,
                         int64_t* d_tot, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !p || !d_tot || (classes != 2 && classes != 3) || (n > 0 && !xs)) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_PARTITION2, n, 0)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  if (n == 0) return cuda_rc(cudaMemsetAsync(d_tot, 0, sizeof(int64_t) * (classes - 1), s));
  WS w(ws);
  const int cgrid = grid_for(n / 4 + 1);
  long long* partials = (long long*)w.take((size_t)cgrid * 2 * 8);
  const ixg_pred qq = q ? *q : ixg_pred{IXG_PRED_FALSE, 0, 0, 0};
  TimedLaunch tl(IXG_K_CLASS_COUNT, s);
  if (dt == IXG_I32) {
    if (classes == 2)
      k_class_count<int32_t, 2><<<cgrid, kSThreads, 0, s>>>((const int32_t*)xs, n, *p, qq, partials, w.hdr(5),
                                                           (long long*)d_tot);
    else
      k_class_count<int32_t, 3><<<cgrid, kSThreads, 0, s>>>((const int32_t*)xs, n, *p, qq, partials, w.hdr(5),
                                                           (long long*)d_tot);
  } else {
    if (classes == 2)
      k_class_count<long long, 2><<<cgrid, kSThreads, 0, s>>>((const long long*)xs, n, *p, qq, partials, w.hdr(5),
                                                             (long long*)d_tot);
    else
      k_class_count<long long, 3><<<cgrid, kSThreads, 0, s>>>((const long long*)xs, n, *p, qq, partials, w.hdr(5),
                                                             (long long*)d_tot);
  }
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_partition2_peer(int dt, const void* xs, int64_t n, const ixg_pred* p, void* const* dst, int ranks,
                        int64_t shard, const int64_t* d_counts, int rank, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !p || !dst || !d_counts || ranks < 1 || ranks > 8 || rank < 0 || rank >= ranks || shard <= 0 ||
      n != shard || (n > 0 && !xs))
    return IXG_BADARG;
  const int ep = dt == IXG_I32 ? 4 : 2;
  if (shard % ep) return IXG_BADARG;  // a 16-byte chunk never straddles two shards
  if (ws_bytes < ixg_ws_bytes(IXG_OP_PARTITION2, n, 0)) return IXG_BADARG;
  if (n == 0) return IXG_OK;
  for (int r = 0; r < ranks; ++r)
    if (!dst[r] || !aligned16(dst[r])) return IXG_BADARG;
  if (!aligned16(xs)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  WS w(ws);
  LBChan c0 = w.chan(0, std::max(lb_tiles(n), 2 * tiles_of(n, Big<long long>::TILE)));
  long long* scratch = (long long*)w.take(64);
  const ixg_pred pp = *p;
  if (dt == IXG_I32) {
    PeerOut<int32_t> po{};
    for (int r = 0; r < ranks; ++r) po.dst[r] = (int32_t*)dst[r];
    po.shard = shard;
    po.ranks = ranks;
    po.d_counts = (const long long*)d_counts;
    po.rank = rank;
    po.in_shard = n;
    switch (peer_dual_chunks()) {  // one read of xs, both classes placed (12 -> 8 B per element)
#define IXG_DUAL32(K)                                                                                           \
  case K:                                                                                                       \
    return launch_filter_b<int32_t, false, false, int32_t, 1, true, K>((const int32_t*)xs, nullptr, n, pp, nullptr, \
                                                                       c0, scratch, s, nullptr, nullptr, 0,      \
                                                                       LBChan{nullptr, nullptr}, nullptr,        \
                                                                       ixg_pred{}, po);
      case -1:
        return launch_filter_b<int32_t, false, false, int32_t, 1, true>((const int32_t*)xs, nullptr, n, pp, nullptr,
                                                                        c0, scratch, s, nullptr, nullptr, 0,
                                                                        LBChan{nullptr, nullptr}, nullptr, ixg_pred{},
                                                                        po);
      IXG_DUAL32(1)
      IXG_DUAL32(2)
      IXG_DUAL32(3)
#undef IXG_DUAL32
      default:
        break;
    }
    return launch_filter_b<int32_t, false, false, int32_t, 2, true>((const int32_t*)xs, nullptr, n, pp, nullptr, c0,
                                                                    scratch, s, nullptr, nullptr, 0,
                                                                    LBChan{nullptr, nullptr}, nullptr, ixg_pred{},
                                                                    po);
  }
  PeerOut<long long> po{};
  for (int r = 0; r < ranks; ++r) po.dst[r] = (long long*)dst[r];
  po.shard = shard;
  po.ranks = ranks;
  po.d_counts = (const long long*)d_counts;
  po.rank = rank;
  po.in_shard = n;
  switch (peer_dual_chunks()) {
#define IXG_DUAL64(K)                                                                                          \
  case K:                                                                                                      \
    return launch_filter_b<long long, false, false, long long, 1, true, K>((const long long*)xs, nullptr, n, pp, \
                                                                           nullptr, c0, scratch, s, nullptr,      \
                                                                           nullptr, 0, LBChan{nullptr, nullptr},  \
                                                                           nullptr, ixg_pred{}, po);
    case -1:
      return launch_filter_b<long long, false, false, long long, 1, true>((const long long*)xs, nullptr, n, pp,
                                                                          nullptr, c0, scratch, s, nullptr, nullptr, 0,
                                                                          LBChan{nullptr, nullptr}, nullptr,
                                                                          ixg_pred{}, po);
    IXG_DUAL64(1)
#undef IXG_DUAL64
    default:
      break;
  }
  return launch_filter_b<long long, false, false, long long, 2, true>((const long long*)xs, nullptr, n, pp, nullptr,
                                                                      c0, scratch, s, nullptr, nullptr, 0,
                                                                      LBChan{nullptr, nullptr}, nullptr, ixg_pred{},
                                                                      po);
}

// ---- device memory shared across processes (CUDA IPC over NVLink) ----
int ixg_dev_alloc(size_t bytes, void** out) {
  if (!out) return IXG_BADARG;
  return cuda_rc(cudaMalloc(out, bytes ? bytes : 16));
}
int ixg_dev_free(void* p) { return cuda_rc(cudaFree(p)); }
int ixg_ipc_handle(const void* p, void* handle) {
  if (!p || !handle) return IXG_BADARG;
  cudaIpcMemHandle_t h;
  int rc = cuda_rc(cudaIpcGetMemHandle(&h, const_cast<void*>(p)));
  if (rc) return rc;
  memcpy(handle, &h, sizeof(h));
  return IXG_OK;
}
int ixg_ipc_open(const void* handle, void** out) {
  if (!handle || !out) return IXG_BADARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return cuda_rc(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
}
int ixg_ipc_close(void* p) { return cuda_rc(cudaIpcCloseMemHandle(p)); }

int ixg_partition2(int dt, const void* xs, int64_t n, const ixg_pred* p, void* ys, int64_t* d_num_true,
                   uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !p || !d_num_true || (n > 0 && (!xs || !ys))) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_PARTITION2, n, 0)) return IXG_BADARG;
  WS w(ws);
  if (dt == IXG_I32)
    return do_partition<int32_t, 2>((const int32_t*)xs, n, p, nullptr, (int32_t*)ys, (long long*)d_num_true,
                                    variant, st, w, S(stream));
  return do_partition<int64_t, 2>((const int64_t*)xs, n, p, nullptr, (int64_t*)ys, (long long*)d_num_true, variant,
                                  st, w, S(stream));
}

int ixg_partition3(int dt, const void* xs, int64_t n, const ixg_pred* p, const ixg_pred* q, void* ys, int64_t* d_m,
                   uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || !p || !q || !d_m || (n > 0 && (!xs || !ys))) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_PARTITION3, n, 0)) return IXG_BADARG;
  WS w(ws);
  if (dt == IXG_I32)
    return do_partition<int32_t, 3>((const int32_t*)xs, n, p, q, (int32_t*)ys, (long long*)d_m, variant, st, w,
                                    S(stream));
  return do_partition<int64_t, 3>((const int64_t*)xs, n, p, q, (int64_t*)ys, (long long*)d_m, variant, st, w,
                                  S(stream));
}

int ixg_c2(int dt, const void* xs, int64_t n, const ixg_pred* p, const int64_t* shape, int64_t m, void* ys, int dt_z,
           void* zs, int64_t* d_k, uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || m < 0 || !p || !d_k || (n > 0 && (!xs || !ys || !zs)) || (m > 0 && !shape)) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_C2, n, m)) return IXG_BADARG;
  WS w(ws);
  cudaStream_t s = S(stream);
  const long long* sh = (const long long*)shape;
  long long* dk = (long long*)d_k;
  if (dt == IXG_I32 && dt_z == IXG_I32)
    return do_c2<int32_t, int32_t>((const int32_t*)xs, n, p, sh, m, (int32_t*)ys, (int32_t*)zs, dk, variant, st, w, s);
  if (dt == IXG_I32)
    return do_c2<int32_t, int64_t>((const int32_t*)xs, n, p, sh, m, (int32_t*)ys, (int64_t*)zs, dk, variant, st, w, s);
  if (dt_z == IXG_I32) return IXG_BADARG;
  return do_c2<int64_t, int64_t>((const int64_t*)xs, n, p, sh, m, (int64_t*)ys, (int64_t*)zs, dk, variant, st, w, s);
}

int ixg_mksgmdescr(const int64_t* shape, const int64_t* xs, int64_t m, int64_t nxs, int64_t* res, int64_t cap,
                   int64_t* d_len, uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes, void* stream) {
  if (m < 0 || nxs < 0 || cap < 0 || !d_len || (m > 0 && !shape) || (nxs > 0 && !xs) || (cap > 0 && !res))
    return IXG_BADARG;
  const long long pairs = m < nxs ? m : nxs;  // scatter's zip(ind, xs) truncates (oracle.py:299)
  if (ws_bytes < ixg_ws_bytes(IXG_OP_MKSGMDESCR, cap, m)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  WS w(ws);
  LBChan c = w.chan(0, tiles_of(m, kGTile));
  long long* ind = (long long*)w.take((size_t)(m > 0 ? m : 1) * 8);
  if (m == 0) return cuda_rc(cudaMemsetAsync(d_len, 0, 8, s));
  // scn / ind / len (mksgmdescr.ixl:6-9); len = scn[m-1] + shape[m-1] = sum shape
  int rc = launch_scan<SumOp>(m, SrcArrT<long long>{(const long long*)shape},
                              EpiSegStarts{m, (const long long*)shape, ind, nullptr, 0, nullptr, (long long*)d_len, st}, c,
                              s);
  if (rc || cap == 0) return rc;
  // the scatter is never proved for mkSgmDescr: the host
  // passes cap >= len (read back from d_len), res[0..len) = 0, checked scatter.
  const uint32_t sb = IXG_SITE_BITS(variant, 3) | IXG_V_INIT;
  if ((rc = launch_fill<long long>((long long*)res, 0, (const long long*)d_len, 0LL, s))) return rc;
  return launch_scatter<long long>((long long*)res, 0, (const long long*)d_len, cap, ind, (const long long*)xs, pairs,
                                   sb, 3, 3, st, w, 1, s);
}

int ixg_csr_gather(int dt, const void* x, int64_t num_cols, const void* values, const int64_t* indices, int64_t nnz,
                   void* out, uint32_t variant, ixg_status* st, void* stream) {
  if (nnz < 0 || (nnz > 0 && (!values || !indices || !out))) return IXG_BADARG;
  if (nnz == 0) return IXG_OK;
  if (!aligned16(values) || !aligned16(indices) || !aligned16(out)) return IXG_BADARG;
  const int check = (IXG_SITE_BITS(variant, 0) & IXG_V_BOUNDS) ? 1 : 0;
  cudaStream_t s = S(stream);
  TimedLaunch tl(IXG_K_CSR_GATHER, s);
  const long long work = nnz / 4 + 1;
  if (dt == IXG_I32)
    k_csr_gather<int32_t><<<grid_for(work), kGThreads, 0, s>>>((const int32_t*)x, num_cols, (const int32_t*)values,
                                                                (const long long*)indices, nnz, (int32_t*)out, check,
                                                                st);
  else
    k_csr_gather<long long><<<grid_for(work), kGThreads, 0, s>>>((const long long*)x, num_cols,
                                                                  (const long long*)values, (const long long*)indices,
                                                                  nnz, (long long*)out, check, st);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_kmeans_ker(const int64_t* rows, int64_t nrows, const int64_t* pointers, int64_t np1, const double* cluster,
                   int64_t num_cols, const double* values, const int64_t* indices, int64_t nnz, double* out,
                   uint32_t variant, ixg_status* st, void* stream) {
  if (nrows < 0 || (nrows > 0 && (!rows || !out))) return IXG_BADARG;
  if (nrows == 0) return IXG_OK;
  k_kmeans<<<(unsigned)((nrows + 127) / 128), 128, 0, S(stream)>>>(
      (const long long*)rows, nrows, (const long long*)pointers, np1, cluster, num_cols, values,
      (const long long*)indices, nnz, out, variant, st);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_eq_gather(const int64_t* H, int64_t hlen, const int64_t* es, const int64_t* is, int64_t n, uint8_t* cs,
                  uint32_t variant, int stmt, ixg_status* st, void* stream) {
  if (n < 0 || (n > 0 && (!es || !is || !cs))) return IXG_BADARG;
  if (n == 0) return IXG_OK;
  const int check = (IXG_SITE_BITS(variant, 0) & IXG_V_BOUNDS) ? 1 : 0;
  k_eq_gather<<<grid_for(n), kGThreads, 0, S(stream)>>>((const long long*)H, hlen, (const long long*)es,
                                                         (const long long*)is, n, cs, check, st, stmt);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

// ---- preconditions (contract.py): Range / Mono / Inj / Bij on the device ----
int ixg_minmax(int dt, const void* xs, int64_t n, int64_t* out2, void* stream) {
  if (n < 0 || !out2 || (n > 0 && !xs)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  const long long init[2] = {LLONG_MAX, LLONG_MIN};
  int rc = cuda_rc(cudaMemcpyAsync(out2, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (rc || n == 0) return rc;
  if (dt == IXG_I32)
    k_minmax<int32_t><<<grid_for(n / 4 + 1), kGThreads, 0, s>>>((const int32_t*)xs, n, (long long*)out2);
  else if (dt == IXG_U8)
    k_minmax<uint8_t><<<grid_for(n / 16 + 1), kGThreads, 0, s>>>((const uint8_t*)xs, n, (long long*)out2);
  else
    k_minmax<long long><<<grid_for(n / 2 + 1), kGThreads, 0, s>>>((const long long*)xs, n, (long long*)out2);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_mono_check(int dt, const void* xs, int64_t n, int op, int64_t* out_bad, void* stream) {
  if (n < 0 || !out_bad || op < 0 || op > 3 || (n > 0 && !xs)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  int rc = cuda_rc(cudaMemsetAsync(out_bad, 0, 8, s));
  if (rc || n < 2) return rc;
  unsigned long long* b = (unsigned long long*)out_bad;
  if (dt == IXG_I32)
    k_mono<int32_t><<<grid_for(n), kGThreads, 0, s>>>((const int32_t*)xs, n, op, b);
  else
    k_mono<long long><<<grid_for(n), kGThreads, 0, s>>>((const long long*)xs, n, op, b);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int64_t ixg_inj_bitmap_bytes(int64_t lo, int64_t hi) {
  if (hi < lo) return 0;
  const unsigned long long span = (unsigned long long)hi - (unsigned long long)lo + 1ULL;
  if (span == 0 || span > (1ULL << 31)) return -1;  // wider than 2^31 values (256 MB of bitmap): not checked here
  return (int64_t)bitmap_bytes((long long)span);
}

int ixg_inj_check(const int64_t* xs, int64_t n, int64_t lo, int64_t hi, int64_t img_lo, int64_t img_hi,
                  uint32_t* bitmap, int64_t bitmap_bytes_, int64_t* out3, void* stream) {
  if (n < 0 || !out3 || (n > 0 && !xs)) return IXG_BADARG;
  const int64_t need = ixg_inj_bitmap_bytes(lo, hi);
  if (need < 0 || (need > 0 && (!bitmap || bitmap_bytes_ < need))) return IXG_BADARG;
  cudaStream_t s = S(stream);
  int rc = cuda_rc(cudaMemsetAsync(out3, 0, 3 * 8, s));
  if (rc || n == 0 || need == 0) return rc;
  if ((rc = cuda_rc(cudaMemsetAsync(bitmap, 0, (size_t)need, s)))) return rc;
  LAUNCHED();
  const unsigned long long span = (unsigned long long)hi - (unsigned long long)lo + 1ULL;
  k_inj_claim<<<grid_for(n), kGThreads, 0, s>>>((const long long*)xs, n, lo, span, img_lo, img_hi, bitmap,
                                                (unsigned long long*)out3);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_gen_uniform(int dt, void* out, int64_t n, int64_t lo, int64_t hi, uint64_t seed, int64_t offset,
                    void* stream) {
  if (n <= 0) return IXG_OK;
  if (!out || hi < lo) return IXG_BADARG;
  const unsigned long long span = (unsigned long long)hi - (unsigned long long)lo + 1ULL;  // 0 = full 2^64
  const uint64_t smix = seed_mix_host(seed);
  cudaStream_t s = S(stream);
  if (dt == IXG_I32)
    k_gen_uniform<int32_t><<<grid_for(n), kGThreads, 0, s>>>((int32_t*)out, n, lo, span, smix, offset);
  else
    k_gen_uniform<long long><<<grid_for(n), kGThreads, 0, s>>>((long long*)out, n, lo, span, smix, offset);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_mkflags(int64_t k, const int64_t* shape, int64_t m, int64_t* flags, uint32_t variant, ixg_status* st,
                void* ws, size_t ws_bytes, void* stream) {
  if (m < 0 || (m > 0 && !shape) || (k > 0 && !flags)) return IXG_BADARG;
  if (k < 0) k = 0;  // replicate k 0 with k < 0 is []
  if (ws_bytes < ixg_ws_bytes(IXG_OP_MKFLAGS, k, m)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  WS w(ws);
  LBChan c = w.chan(0, tiles_of(m, kGTile));
  long long* ind = (long long*)w.take((size_t)(m > 0 ? m : 1) * 8);
  long long* ones = (long long*)w.take((size_t)(m > 0 ? m : 1) * 8);
  int rc;
  if (k > 0 && (rc = launch_fill<long long>((long long*)flags, k, nullptr, 0LL, s))) return rc;
  if (m == 0) return IXG_OK;
  if ((rc = launch_scan<SumOp>(m, SrcArrT<long long>{(const long long*)shape},
                               EpiSegStarts{m, (const long long*)shape, ind, nullptr, 0, nullptr, nullptr, st}, c, s)))
    return rc;
  if ((rc = launch_fill<long long>(ones, m, nullptr, 1LL, s))) return rc;
  return launch_scatter<long long>((long long*)flags, k, nullptr, k, ind, ones, m,
                                   IXG_SITE_BITS(variant, 1) | IXG_V_INIT, 1, 1, st, w, 1, s);
}

int ixg_rank_offsets(const int64_t* d_counts, int ranks, int rank, int stride, int64_t* out2, void* stream) {
  if (!d_counts || !out2 || ranks < 1 || rank < 0 || rank >= ranks || stride < 1) return IXG_BADARG;
  k_rank_offsets<<<1, 32, 0, S(stream)>>>((const long long*)d_counts, ranks, rank, stride, (long long*)out2);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int64_t ixg_bitmap_words(int64_t nbits) { return (int64_t)(bitmap_bytes(nbits) / 4); }

int ixg_flag_bitmap(const int64_t* shape, int64_t m, uint32_t* bits, int64_t nbits, const int64_t* d_nbits, void* ws,
                    size_t ws_bytes, void* stream) {
  if (m < 0 || nbits < 0 || (m > 0 && !shape) || !bits) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_SCAN, m, 0)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  WS w(ws);
  LBChan c = w.chan(0, tiles_of(m, kGTile));
  // (d_nbits: nbits on the device, <= the capacity nbits -- only those words are cleared)
  return launch_mkflags((const long long*)shape, m, bits, nbits, (const long long*)d_nbits, c, s);
}

int ixg_flag_bitmap_window(const int64_t* shape, int64_t m, uint32_t* bits, int64_t nbits, const int64_t* d_nbits,
                           const int64_t* d_lo, void* ws, size_t ws_bytes, void* stream) {
  if (m < 0 || nbits < 0 || (m > 0 && !shape) || !bits || !d_lo) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_SCAN, m, 0)) return IXG_BADARG;
  cudaStream_t s = S(stream);
  WS w(ws);
  LBChan c = w.chan(0, tiles_of(m, kGTile));
  return launch_mkflags((const long long*)shape, m, bits, nbits, (const long long*)d_nbits, c, s, nullptr,
                        (const long long*)d_lo);
}

int ixg_segsum(int dt, const void* vs, int64_t n, const int64_t* d_n, const uint32_t* bits, int64_t flag_base,
               const int64_t* d_flag_base, int dt_z, void* zs, int64_t carry_v, int carry_f, int64_t* d_total,
               ixg_status* st, void* ws, size_t ws_bytes, void* stream) {
  if (n < 0 || (n > 0 && (!vs || !zs || !bits))) return IXG_BADARG;
  if (ws_bytes < ixg_ws_bytes(IXG_OP_SEGSCAN, n, 0)) return IXG_BADARG;
  if (n == 0) return IXG_OK;
  if (!aligned16(vs) || !aligned32(zs)) return IXG_BADARG;  // TMA loads / 32-byte vector stores
  WS w(ws);
  LBChan c = w.chan(0, tiles_of(n, kGTile));
  cudaStream_t s = S(stream);
  const long long* dn = (const long long*)d_n;
  const long long* dfb = (const long long*)d_flag_base;
  longlong2* tot = (longlong2*)d_total;
  if (dt == IXG_I32 && dt_z == IXG_I32)
    return launch_segsum_b<int32_t, int32_t>((const int32_t*)vs, n, dn, bits, flag_base, (int32_t*)zs, c, carry_v,
                                             carry_f, tot, st, s, dfb);
  if (dt == IXG_I32)
    return launch_segsum_b<int32_t, long long>((const int32_t*)vs, n, dn, bits, flag_base, (long long*)zs, c,
                                               carry_v, carry_f, tot, st, s, dfb);
  if (dt_z == IXG_I32) return IXG_BADARG;
  return launch_segsum_b<long long, long long>((const long long*)vs, n, dn, bits, flag_base, (long long*)zs, c,
                                               carry_v, carry_f, tot, st, s, dfb);
}

int ixg_seg_carry(const uint32_t* bits, int64_t flag_base, const int64_t* d_flag_base, int dt_z, void* zs, int64_t n,
                  const int64_t* d_n, int64_t carry_v, const int64_t* d_aggs, int rank, void* scratch8, ixg_status* st,
                  void* stream) {
  if (n < 0 || !bits || !scratch8 || (n > 0 && !zs) || (d_aggs && rank < 0)) return IXG_BADARG;
  if (n == 0 || (!d_aggs && carry_v == 0)) return IXG_OK;
  cudaStream_t s = S(stream);
  unsigned long long* first = (unsigned long long*)scratch8;
  cudaMemsetAsync(first, 0xff, sizeof(unsigned long long), s);
  LAUNCHED();
  k_first_flag<<<grid_for(n / 32 + 1), 256, 0, s>>>(bits, flag_base, (const long long*)d_flag_base, n,
                                                     (const long long*)d_n, first);
  LAUNCHED();
  CHECK_LAUNCH();
  const long long* ag = (const long long*)d_aggs;
  if (dt_z == IXG_I32)
    k_add_prefix<int32_t><<<grid_for(n), 256, 0, s>>>((int32_t*)zs, first, n, (const long long*)d_n, carry_v, ag,
                                                       rank, st);
  else
    k_add_prefix<long long><<<grid_for(n), 256, 0, s>>>((long long*)zs, first, n, (const long long*)d_n, carry_v, ag,
                                                         rank, st);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

int ixg_map(const ixg_vm_insn* prog, int ninsn, const ixg_array* ins, int nins, const ixg_array* outs, int nouts,
            const ixg_pred* preds, int npreds, int64_t n, int stmt, ixg_status* st, void* stream) {
  if (ninsn < 0 || ninsn > IXG_VM_MAX_INSN || nins < 0 || nins > IXG_VM_MAX_IN || nouts < 0 ||
      nouts > IXG_VM_MAX_OUT || npreds < 0 || npreds > IXG_VM_MAX_PRED || n < 0)
    return IXG_BADARG;
  if (n == 0) return IXG_OK;
  VmProgram P;
  memset(&P, 0, sizeof(P));
  for (int i = 0; i < ninsn; ++i) {
    const ixg_vm_insn& I = prog[i];
    if (I.dst < 0 || I.dst >= IXG_VM_REGS || I.a < 0 || I.a >= IXG_VM_REGS) return IXG_BADARG;
    if ((I.op == IXG_VM_JZ || I.op == IXG_VM_JMP) && (I.c < 0 || I.c > ninsn)) return IXG_BADARG;
    if ((I.op == IXG_VM_ADD || I.op == IXG_VM_SUB || I.op == IXG_VM_MUL || (I.op >= IXG_VM_EQ && I.op <= IXG_VM_GE)) &&
        (I.b < 0 || I.b >= IXG_VM_REGS))
      return IXG_BADARG;
    if ((I.op == IXG_VM_IN && I.a >= nins) || ((I.op == IXG_VM_IDX || I.op == IXG_VM_LEN) && (I.b < 0 || I.b >= nins)) ||
        (I.op == IXG_VM_OUT && (I.b < 0 || I.b >= nouts)) || (I.op == IXG_VM_PRED && (I.b < 0 || I.b >= npreds)))
      return IXG_BADARG;
    P.insn[i] = I;
  }
  for (int i = 0; i < nins; ++i) P.in[i] = ins[i];
  for (int i = 0; i < nouts; ++i) P.out[i] = outs[i];
  for (int i = 0; i < npreds; ++i) P.pred[i] = preds[i];
  P.ninsn = ninsn;
  P.nin = nins;
  P.nout = nouts;
  P.npred = npreds;
  k_map_vm<<<grid_for(n), 256, 0, S(stream)>>>(P, n, stmt, st);
  LAUNCHED();
  CHECK_LAUNCH();
  return IXG_OK;
}

}  // extern "C"
