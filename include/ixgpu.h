/*
 * ixgpu.h -- C ABI of libixgpu.so, the B200 (sm_100a) execution path for the
 * index-array combinators of arXiv 2506.23058 (reference: `ixverify`).
 *
 * What this replaces.  The reference executes programs with its interpreter,
 * `ixverify.oracle.eval_program(program, fun, args, step_budget)`
 * (/root/reference/pkg/src/ixverify/oracle.py:332-333 -> Interp.call :127-135),
 * whose builtins are dispatched by name in `Interp._app` (oracle.py:269-329):
 *   map :274-280, scan :281-293, scatter :294-305, hist :306-316,
 *   iota :317-318, replicate :319-322, length :323-324,
 * plus array indexing with a bounds check in `Interp.eval` (oracle.py:177-184).
 * Each entry point below is one of those builtins, or one corpus program
 * (`/root/reference/pkg/corpus`) executed as a fused pipeline.  The Python
 * host side (`paper_2506_23058_b200.eval_program`) keeps the reference's
 * signature and binds these symbols with ctypes.
 *
 * Conventions (every function):
 *   - all array pointers are DEVICE pointers owned by the caller; the library
 *     allocates nothing persistent;
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *     and asynchronous (the return code only reports argument / launch errors);
 *   - `ws`/`ws_bytes` is caller-provided device scratch: size it with
 *     ixg_ws_bytes(), zero it ONCE with ixg_ws_init() after allocation (the
 *     kernels leave it ready for the next call);
 *   - `dt` selects the element width of value arrays: IXG_I32 or IXG_I64
 *     (the language type is i64; i32 storage is used where values fit);
 *   - data-dependent scalars (counts, lengths) are written to DEVICE int64
 *     slots so that pipelines never synchronise the host;
 *   - failures of the reference's dynamic checks are recorded in a device
 *     `ixg_status` (first failure in the reference's sequential order); the
 *     host maps it back to OutOfBounds / NonIdempotentScatter (oracle.py:51-77).
 *
 * Variant bits.  The verifier (`ixverify.infer.Analyzer`, infer.py:172-226)
 * proves obligations per source site; the selector turns them into 4 bits per
 * site, packed as `variant = sum(bits_s << (4*s))` over the pipeline's sites:
 *   IXG_V_BOUNDS    perform the bounds check of an indexing site
 *                   (cleared when both `bounds` obligations are proved,
 *                   infer.py:612-632);
 *   IXG_V_CONFLICT  perform the scatter idempotence check (cleared when
 *                   `scatter-safety` is proved via Ss1/Ss2/Ss3, infer.py:1129-1143);
 *   IXG_V_INIT      initialise the scatter destination and test indices
 *                   against its length (cleared only when Sc1 holds with full
 *                   image, infer.py:1101-1122).
 * IXG_VARIANT_CHECKED (all bits set) is the reference interpreter's behaviour.
 */
#ifndef IXGPU_H
#define IXGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return / status codes (oracle.py:51-77) ---------------------------- */
#define IXG_OK 0
#define IXG_OOB 1        /* OutOfBounds(site, pos)        oracle.py:55-59   */
#define IXG_CONFLICT 2   /* NonIdempotentScatter(pos)     oracle.py:62-65   */
#define IXG_LENGTH 3     /* OracleError(map lengths)      oracle.py:278-279 */
#define IXG_BADARG 4
#define IXG_NOMEM 5
#define IXG_OVERFLOW 6   /* a value does not fit the storage width          */
#define IXG_NODEVICE 7
#define IXG_CUDA_ERR 100 /* + cudaError_t                                    */

#define IXG_I32 0
#define IXG_I64 1
#define IXG_U8 2
#define IXG_F64 3

#define IXG_V_BOUNDS 1u
#define IXG_V_CONFLICT 2u
#define IXG_V_INIT 4u
#define IXG_VARIANT_CHECKED 0x77777777u
#define IXG_VARIANT_ELIDED 0u
#define IXG_SITE_BITS(variant, site) (((variant) >> (4 * (site))) & 0xfu)

/* predicate descriptor for `p : i64 -> bool` parameters (the reference passes
 * Python callables, oracle.py:686-696; paper_2506_23058_b200.Pred is both). */
#define IXG_PRED_LT 0
#define IXG_PRED_GT 1
#define IXG_PRED_LE 2
#define IXG_PRED_GE 3
#define IXG_PRED_EQ 4
#define IXG_PRED_NE 5
#define IXG_PRED_HASH 6
#define IXG_PRED_TRUE 7
#define IXG_PRED_FALSE 8
typedef struct ixg_pred {
  int32_t kind;
  int32_t pad;
  int64_t thr;
  uint64_t seed;
} ixg_pred;

/* device-resident status: `first` = min over failures of
 * [stmt:8][elem:48][site:8] (UINT64_MAX = none), `codes` = OR of 1<<code,
 * `flags` = internal (IXG_F_*). */
typedef struct ixg_status {
  unsigned long long first;
  unsigned int codes;
  unsigned int flags;
} ixg_status;
/* An integer result left int64.  The reference's ints are unbounded
 * (oracle.py:214-240; a scan of [2^62, 2^62, 2^62] gives 3*2^62), the device
 * computes in int64: every i64 path checks its results exactly (scans: each
 * output against its predecessor, hist (+): 128-bit bins, lambdas: every
 * + - *) and records IXG_OVERFLOW with site IXG_OVF_SITE; the host raises
 * instead of returning a wrapped value. */
#define IXG_OVF_SITE 254
#define IXG_F_DUP 1u      /* a scatter destination was claimed twice       */
#define IXG_F_NARROW 2u   /* a result did not fit its i32 storage          */

/* hist operators (oracle.py:110-114 _NAMED_OPS, plus (+)) */
#define IXG_HIST_MIN 0
#define IXG_HIST_MAX 1
#define IXG_HIST_ADD 2

/* ops for ixg_ws_bytes */
#define IXG_OP_SCAN 1
#define IXG_OP_SEGSCAN 2
#define IXG_OP_SCATTER 3
#define IXG_OP_FILTER 4
#define IXG_OP_PARTITION2 5
#define IXG_OP_PARTITION3 6
#define IXG_OP_C2 7
#define IXG_OP_MKSGMDESCR 8
#define IXG_OP_MKFLAGS 9
#define IXG_OP_HIST 10     /* m = dlen */
#define IXG_OP_SCATTER_BINNED 11  /* n = pairs, m = ndst */

/* scatter layouts (ixg_scatter) */
#define IXG_SCATTER_DIRECT 0  /* pairs stored in their own order            */
#define IXG_SCATTER_BINNED 1  /* pairs first partitioned by destination
                                 window (16 MB windows, ndst <= 2^32)      */

/* ---- library / device --------------------------------------------------- */
int ixg_version(void);
/* IXG_OK if the current device is sm_100 (B200); IXG_NODEVICE otherwise */
int ixg_device_check(void);
size_t ixg_ws_bytes(int op, int64_t n, int64_t m);
int ixg_ws_init(void* ws, size_t ws_bytes, void* stream);
int ixg_status_init(ixg_status* st, void* stream);
/* number of kernels this library launched since load (bench evidence) */
unsigned long long ixg_launch_count(void);

/* ---- builtins ------------------------------------------------------------ */

/* scan (+) ne xs  (oracle.py:281-293, k = 1, f = (+)): out[i] = ne + sum_{j<=i} xs[j]
 * (ne folded once).  `exclusive` != 0 gives out[i] = ne + sum_{j<i} xs[j].
 * xs: dt in {I32, I64, U8}; out: int64.  st (nullable): IXG_OVERFLOW at the
 * first element whose sum leaves int64. */
int ixg_scan_add(int dt, const void* xs, int64_t n, int64_t ne, int exclusive, int64_t* out,
                 void* ws, size_t ws_bytes, ixg_status* st, void* stream);

/* partition2L's scatter destinations (corpus/partition2l.ixl:41, PAPER.md:
 * 3250-3261) for a jagged array with sum shp == n: bits = row starts (the
 * mkFlags bitmap of shp over n positions, ixg_flag_bitmap), cs = the
 * per-element predicate (u8), tb = the per-row inclusive count of cs
 * (ixg_segsum of cs).  dest[i] = row start + trues before i in its row for
 * a true element, i + trues after i in its row for a false one. */
int ixg_jagged_dest(const uint32_t* bits, int64_t n, const uint8_t* cs, const int64_t* tb, int64_t* dest,
                    void* stream);

/* total of `scan (+) 0 xs` -- the last element of oracle.py:281-293's inclusive
 * scan -- written to *out (device int64).  The sharded scan (dist.py) needs it
 * before the seeded local scan; dt in {I32, I64, U8}. */
int ixg_reduce_add(int dt, const void* xs, int64_t n, int64_t* out, void* stream);

/* 2-ary scan with the segmented-sum operator (the k-ary scan
 * of oracle.py:281-293 with \f1 v1 f2 v2 -> (f1 || f2, if f2 then v2 else v1+v2),
 * ne = (f0, v0)): out_v[i] = value component; out_f (nullable, u8) = flag
 * component.  flags: dt_f in {U8, I32, I64} (non-zero = true); xs: dt_x. */
int ixg_segscan_add(int dt_f, const void* flags, int dt_x, const void* xs, int64_t n, int f0,
                    int64_t v0, int64_t* out_v, uint8_t* out_f, void* ws, size_t ws_bytes,
                    ixg_status* st, void* stream);

/* scatter dst is vs (oracle.py:294-305).  `out` must already hold the copy of
 * dst (length ndst) unless the site's IXG_V_INIT bit is clear (Sc1: every
 * destination is written).  m = min(nis, nvs) pairs (zip truncation).
 * Out-of-range indices are skipped in every variant (oracle.py:300).  With
 * IXG_V_CONFLICT the idempotence check runs: conflicting values at one
 * in-range index -> IXG_CONFLICT in `st` (stmt, site).  is: int64; vs/out: dt.
 * layout: IXG_SCATTER_DIRECT or IXG_SCATTER_BINNED (ws sized with
 * IXG_OP_SCATTER_BINNED); CHECKED claims are privatised per tile in shared
 * memory windows, merged with one atomic per bitmap word. */
int ixg_scatter(int dt, void* out, int64_t ndst, const int64_t* is, int64_t nis, const void* vs,
                int64_t nvs, uint32_t site_bits, int stmt, int site, int layout, ixg_status* st, void* ws,
                size_t ws_bytes, void* stream);
/* Which layout suits an index array: *d_flag = 1 when sampled runs of `is`
 * jump between 4096-destination windows at most elements (no locality:
 * IXG_SCATTER_BINNED pays off), 0 otherwise.  The host reads the flag. */
int ixg_scatter_probe(const int64_t* is, int64_t m, int* d_flag, void* stream);

/* gather: out[i] = arr[idx[i]] (IndexE, oracle.py:177-184).  With
 * IXG_V_BOUNDS, out-of-range -> IXG_OOB at (stmt, elem i, site).  arr/out: dt. */
int ixg_gather(int dt, const void* arr, int64_t len, const int64_t* idx, int64_t n, void* out,
               uint32_t site_bits, int stmt, int site, ixg_status* st, void* stream);

/* hist op ne dlen is vs (oracle.py:306-316): out[0..dlen) = ne, then
 * out[i] = op(out[i], v) for in-range i.  is: int64; vs/out: int64.
 * IXG_HIST_ADD accumulates each bin in 128 bits (the high words live in
 * ws, ixg_ws_bytes(IXG_OP_HIST, 0, dlen)) and records IXG_OVERFLOW in st
 * for a bin whose sum leaves int64. */
int ixg_hist(int op, int64_t ne, int64_t dlen, const int64_t* is, int64_t nis, const int64_t* vs,
             int64_t nvs, int64_t* out, void* ws, size_t ws_bytes, ixg_status* st, void* stream);

/* replicate n v (oracle.py:319-322) / iota n (oracle.py:317-318) */
int ixg_fill(int dt, void* out, int64_t n, int64_t v, void* stream);
int ixg_iota(int64_t* out, int64_t n, void* stream);

/* ---- corpus programs as fused pipelines -------------------------------- */

/* filter (corpus/filter.ixl:4-15; sites: 0 = offs[n-1], 1 = scatter).
 * ys: capacity n, *d_count = result length.  filter_by (maxmatching.ixl:1-9)
 * takes the boolean array cs (u8) instead of p. */
int ixg_filter(int dt, const void* xs, int64_t n, const ixg_pred* p, void* ys, int64_t* d_count,
               uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes, void* stream);
int ixg_filter_by(int dt, const uint8_t* cs, const void* xs, int64_t n, void* ys,
                  int64_t* d_count, uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes,
                  void* stream);

/* Sharded partition2 (BASELINE configs[4]) with the exchange
 * fused into the kernel.  ixg_partition_counts: class totals of the shard
 * (d_tot[0] = trues; classes 3 adds d_tot[1] = class 1), the all-gather input.
 * ixg_partition2_peer: the single-pass partition of this rank's shard whose
 * runs are stored straight to their global positions of the output sharded
 * over `ranks` GPUs (`shard` elements each = this rank's n, shard % (16 / elem
 * size) == 0): dst[r] = rank r's shard, mapped with ixg_ipc_open for r != this
 * rank (peer stores over NVLink); d_counts = DEVICE int64[ranks], every rank's
 * true count (all-gathered on the device, e.g. ncclAllGather of d_tot): the
 * kernel derives this rank's class bases itself (trues at T_<rank, falses at
 * NT + F_<rank), so a sharded step needs no host round trip.
 * Replaces partition2.ixl's scatter (:17) for the sharded case. */
int ixg_partition_counts(int dt, const void* xs, int64_t n, const ixg_pred* p, const ixg_pred* q, int classes,
                         int64_t* d_tot, void* ws, size_t ws_bytes, void* stream);
int ixg_partition2_peer(int dt, const void* xs, int64_t n, const ixg_pred* p, void* const* dst, int ranks,
                        int64_t shard, const int64_t* d_counts, int rank, void* ws, size_t ws_bytes, void* stream);
/* out2 = [sum of d_counts[r * stride] over r < rank, over all r]: a rank's
 * exclusive offset and the global total from an all-gathered device array. */
int ixg_rank_offsets(const int64_t* d_counts, int ranks, int rank, int stride, int64_t* out2, void* stream);
/* device buffers shared between the ranks' processes (CUDA IPC):
 * handle = 64 opaque bytes, exchanged by the host (torch.distributed). */
int ixg_dev_alloc(size_t bytes, void** out);
int ixg_dev_free(void* p);
int ixg_ipc_handle(const void* p, void* handle);
int ixg_ipc_open(const void* handle, void** out);
int ixg_ipc_close(void* p);

/* partition2 (corpus/partition2.ixl:4-19; sites: 0 = indicesT[n-1],
 * 1 = scatter).  ys: length n; *d_num_true. */
int ixg_partition2(int dt, const void* xs, int64_t n, const ixg_pred* p, void* ys,
                   int64_t* d_num_true, uint32_t variant, ixg_status* st, void* ws,
                   size_t ws_bytes, void* stream);

/* partition3 (corpus/partition3.ixl:4-27; sites: 0 = offs1[n-1],
 * 1 = offs2[n-1], 2 = scatter).  d_m: two int64 (m1, m2). */
int ixg_partition3(int dt, const void* xs, int64_t n, const ixg_pred* p, const ixg_pred* q,
                   void* ys, int64_t* d_m, uint32_t variant, ixg_status* st, void* ws,
                   size_t ws_bytes, void* stream);

/* c2 = filter + mkFlags + sgmSum (corpus/c2_filter_sgmsum.ixl; BASELINE
 * configs[1]).  Sites: 0 = filter offs[n-1], 1 = filter scatter,
 * 2 = mkFlags shape[i-1], 3 = mkFlags scatter.  ys, zs: capacity n;
 * zs has width dt_z (IXG_I32 sets IXG_F_NARROW in st if a sum does not fit).
 * *d_k = length of ys and zs.  shape: int64[m]. */
int ixg_c2(int dt, const void* xs, int64_t n, const ixg_pred* p, const int64_t* shape, int64_t m,
           void* ys, int dt_z, void* zs, int64_t* d_k, uint32_t variant, ixg_status* st,
           void* ws, size_t ws_bytes, void* stream);

/* mkSgmDescr (corpus/mksgmdescr.ixl:4-11; sites 0 = shape[i-1], 1 = scn[m-1],
 * 2 = shape[m-1], 3 = scatter).  shape: m elements, xs: nxs elements (the
 * scatter pairs min(m, nxs) of them, zip truncation, oracle.py:299).
 * res: capacity `cap`, *d_len = max(len, 0); call once with cap = 0 to get
 * len, then with cap >= len. */
int ixg_mksgmdescr(const int64_t* shape, const int64_t* xs, int64_t m, int64_t nxs, int64_t* res, int64_t cap,
                   int64_t* d_len, uint32_t variant, ixg_status* st, void* ws, size_t ws_bytes,
                   void* stream);

/* CSR flat gather (corpus/c4_csr_gather.ixl; BASELINE configs[3]):
 * out[i] = values[i] * x[indices[i]], site 0 = x[c]. dt for x/values/out. */
int ixg_csr_gather(int dt, const void* x, int64_t num_cols, const void* values,
                   const int64_t* indices, int64_t nnz, void* out, uint32_t variant,
                   ixg_status* st, void* stream);

/* kmeans_ker (corpus/kmeans_ker.ixl), one result per requested row (the
 * reference computes one row per call): sites 0 = pointers[row],
 * 1 = pointers[row+1], 2 = values[index_start+j], 3 = indices[index_start+j],
 * 4 = cluster[column]; f64 arithmetic without contraction. */
int ixg_kmeans_ker(const int64_t* rows, int64_t nrows, const int64_t* pointers, int64_t np1,
                   const double* cluster, int64_t num_cols, const double* values,
                   const int64_t* indices, int64_t nnz, double* out, uint32_t variant,
                   ixg_status* st, void* stream);

/* get_smallest_pairs' map (maxmatching.ixl:18): cs[i] = (H[es[i]] == is[i]),
 * site 0 = H[i]. */
int ixg_eq_gather(const int64_t* H, int64_t hlen, const int64_t* es, const int64_t* is, int64_t n,
                  uint8_t* cs, uint32_t variant, int stmt, ixg_status* st, void* stream);

/* mkFlags (corpus/c2_filter_sgmsum.ixl; sites 0 = shape[i-1], 1 = scatter):
 * flags[0..k) = 0, then 1 at the exclusive scan of shape for non-empty
 * segments (scatter of `replicate m 1`). */
int ixg_mkflags(int64_t k, const int64_t* shape, int64_t m, int64_t* flags, uint32_t variant, ixg_status* st,
                void* ws, size_t ws_bytes, void* stream);

/* ---- C2 building blocks for sharded (multi-GPU) execution ---------------
 * A rank filters its contiguous shard (ixg_filter), learns its global output
 * offset K from an all-gather of counts, then:
 *   ixg_flag_bitmap  the mkFlags array of ALL shards' outputs as a bitmap
 *                    (bit scn[i] for non-empty segments below nbits, or below
 *                    *d_nbits <= nbits when the total is on the device);
 *   ixg_segsum       zs = sgmSum over its n (or *d_n) outputs, flags = bits
 *                    [flag_base + j] (or *d_flag_base + j), seeded with the
 *                    carry (carry_v, carry_f); *d_total (2 x int64) = its
 *                    segmented aggregate (v, f);
 *   ixg_seg_carry    after the all-gather of aggregates: adds the carry of
 *                    the earlier ranks to its outputs before its first flag
 *                    (carry_v, or -- device-resident -- folded from d_aggs
 *                    = every rank's (v, f) and this rank's index).
 * Every count / offset / carry can stay on the device (d_* arguments). 
 * ixg_bitmap_words(nbits) = uint32 words to allocate for `bits`. */
int64_t ixg_bitmap_words(int64_t nbits);
int ixg_flag_bitmap(const int64_t* shape, int64_t m, uint32_t* bits, int64_t nbits, const int64_t* d_nbits, void* ws,
                    size_t ws_bytes, void* stream);
/* The same bitmap restricted to one shard's outputs: bit j = flag of global
 * output position *d_lo + j, j < nbits (or *d_nbits) -- a rank's window
 * [K, K + k) of the mkFlags array, so a rank clears and sets k bits instead
 * of all shards' K_total.  Replaces, for the sharded sgmSum, the reference's
 * mkFlags (scatter of `replicate m 1` at the exclusive scan of shape,
 * corpus/c2_filter_sgmsum.ixl; oracle.py:294-305) restricted to the
 * positions this shard's outputs occupy. */
int ixg_flag_bitmap_window(const int64_t* shape, int64_t m, uint32_t* bits, int64_t nbits, const int64_t* d_nbits,
                           const int64_t* d_lo, void* ws, size_t ws_bytes, void* stream);
int ixg_segsum(int dt, const void* vs, int64_t n, const int64_t* d_n, const uint32_t* bits, int64_t flag_base,
               const int64_t* d_flag_base, int dt_z, void* zs, int64_t carry_v, int carry_f, int64_t* d_total,
               ixg_status* st, void* ws, size_t ws_bytes, void* stream);
int ixg_seg_carry(const uint32_t* bits, int64_t flag_base, const int64_t* d_flag_base, int dt_z, void* zs, int64_t n,
                  const int64_t* d_n, int64_t carry_v, const int64_t* d_aggs, int rank, void* scratch8, ixg_status* st,
                  void* stream);

/* ---- map with a compiled lambda (oracle.py:274-280) ----------------------
 * The host compiles the lambda body (paper_2506_23058_b200/vm.py) into a
 * short register program; the kernel interprets it per element, all
 * elements in parallel.  Registers are int64 (bools are 0/1).  Indexing
 * (IXG_VM_IDX) is bounds-checked when its site bit is set, failing at
 * (stmt, element, site) in `st` exactly like the reference's IndexE. */
#define IXG_VM_MAX_INSN 96
#define IXG_VM_MAX_IN 8
#define IXG_VM_MAX_OUT 4
#define IXG_VM_MAX_PRED 4
#define IXG_VM_REGS 24
enum {
  IXG_VM_HALT = 0,
  IXG_VM_IN,     /* r[dst] = in[a][i]                                  */
  IXG_VM_CONST,  /* r[dst] = imm                                       */
  IXG_VM_ADD, IXG_VM_SUB, IXG_VM_MUL,
  IXG_VM_EQ, IXG_VM_NE, IXG_VM_LT, IXG_VM_LE, IXG_VM_GT, IXG_VM_GE,
  IXG_VM_NOT,    /* r[dst] = !r[a]                                     */
  IXG_VM_MOV,    /* r[dst] = r[a]                                      */
  IXG_VM_JZ,     /* if r[a] == 0: pc = c                               */
  IXG_VM_JMP,    /* pc = c                                             */
  IXG_VM_IDX,    /* r[dst] = in[b][r[a]]; site c; imm != 0: check       */
  IXG_VM_PRED,   /* r[dst] = pred[b](r[a])                             */
  IXG_VM_OUT,    /* out[b][i] = r[a]                                   */
  IXG_VM_LEN,    /* r[dst] = len(in[b])                                */
  IXG_VM_IDX_F64 /* reserved                                           */
};
typedef struct ixg_vm_insn {
  int32_t op, dst, a, b, c, pad;
  int64_t imm;
} ixg_vm_insn;
typedef struct ixg_array {
  const void* ptr;
  int64_t len;
  int32_t dt;
  int32_t pad;
} ixg_array;
int ixg_map(const ixg_vm_insn* prog, int ninsn, const ixg_array* ins, int nins, const ixg_array* outs, int nouts,
            const ixg_pred* preds, int npreds, int64_t n, int stmt, ixg_status* st, void* stream);

/* ---- measurement: CUDA events recorded on the launching stream around
 * every launch of one kernel family (bench.py's roofline numerator). ------ */
#define IXG_K_FILTER_FUSED 1 /* k_filter (filter / filter+sgmSum, ELIDED)  */
#define IXG_K_PLACE 2        /* k_place (partition2/3 placement, ELIDED)   */
#define IXG_K_CLASS_COUNT 3  /* k_class_count (partition count pass)       */
#define IXG_K_SCAN 4         /* k_scan (every generic single-pass scan)    */
#define IXG_K_SCATTER 5      /* k_scatter                                  */
#define IXG_K_CSR_GATHER 6   /* k_csr_gather                               */
#define IXG_K_SEGSUM 7       /* k_segsum_b (C2 sgmSum pass)                */
#define IXG_K_BIN 8          /* k_bin_partition (binned scatter, pass 1)   */
int ixg_timer_start(int kernel_id);
/* development builds (-DIXG_TRACE) only: per-CTA %globaltimer trace of the
 * compaction kernels; IXG_BADARG otherwise */
int ixg_trace_read(unsigned long long* host, size_t count);
/* synchronises the recorded events; total device time (ms) and launch count */
int ixg_timer_stop(double* total_ms, int64_t* launches);

/* ---- preconditions of an entry function (contract.py) --------------------
 * The verifier's proofs ASSUME the parameter annotations (infer.py:231-338);
 * the reference interpreter never checks them (oracle.py:117-135).  Before
 * the executor uses ELIDED variants it checks them with these, restating
 * oracle.py chk_range / chk_mono / chk_inj / chk_bij (:478-520):
 *   ixg_minmax      out2 = [min, max] of xs ([INT64_MAX, INT64_MIN] if n == 0);
 *   ixg_mono_check  *out_bad = adjacent pairs violating op (0 <=, 1 <, 2 >=, 3 >);
 *   ixg_inj_check   over the values v of xs with lo <= v <= hi: out3[0] = how
 *                   many, out3[1] = repeated values, out3[2] = how many lie
 *                   outside [img_lo, img_hi]; `bitmap` = device scratch of
 *                   ixg_inj_bitmap_bytes(lo, hi) bytes (-1: more than 2^31
 *                   values -- the caller then treats the annotation as
 *                   unchecked and runs CHECKED). */
int ixg_minmax(int dt, const void* xs, int64_t n, int64_t* out2, void* stream);
int ixg_mono_check(int dt, const void* xs, int64_t n, int op, int64_t* out_bad, void* stream);
int64_t ixg_inj_bitmap_bytes(int64_t lo, int64_t hi);
int ixg_inj_check(const int64_t* xs, int64_t n, int64_t lo, int64_t hi, int64_t img_lo, int64_t img_hi,
                  uint32_t* bitmap, int64_t bitmap_bytes, int64_t* out3, void* stream);

/* ---- synthetic inputs (bench / tests): counter-based, identical to
 * paper_2506_23058_b200.gen and oracle/ixoracle.c ixo_rand ----------------- */
int ixg_gen_uniform(int dt, void* out, int64_t n, int64_t lo, int64_t hi, uint64_t seed,
                    int64_t offset, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* IXGPU_H */
