/*
 * ixoracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference interpreter's semantics for the
 * index-array hot path (`/root/reference/pkg/src/ixverify/oracle.py:90-333`)
 * and of the corpus programs built from it (the `.ixl` files of `/root/reference/pkg/corpus`,
 * plus the composed programs under `corpus/` of this repo).
 *
 * It is the CHECKER for the CUDA path: only `tests/`, `__graft_entry__.smoke()`
 * and the `cpu_baseline` / `--impl reference` legs of `bench.py` may load it.
 * The product (`paper_2506_23058_b200`) never links or calls it.
 *
 * Parity pinning: every function here is checked against golden vectors
 * produced by running the Python reference itself (`tests/golden/make_golden.py`
 * imports `ixverify.oracle.eval_program`), see `tests/test_oracle_golden.py`.
 *
 * Values: the reference computes with unbounded Python ints; this restatement
 * uses int64 and reports IXO_OVERFLOW where a sum leaves the int64 range
 * (the reference would keep going; inputs for parity are generated so that it
 * never happens).  Every function follows the *sequential* order of the
 * reference interpreter, so "first failure" is the reference's first failure.
 */
#ifndef IXORACLE_H
#define IXORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: the reference's exception classes (oracle.py:51-77) */
enum {
  IXO_OK = 0,
  IXO_OOB = 1,        /* OutOfBounds(site, pos)              oracle.py:55-59, :182-183 */
  IXO_CONFLICT = 2,   /* NonIdempotentScatter(pos)           oracle.py:62-65, :301-302 */
  IXO_LENGTH = 3,     /* OracleError("map arrays disagree")  oracle.py:278-279 */
  IXO_BADARG = 4,
  IXO_NOMEM = 5,
  IXO_OVERFLOW = 6    /* value outside int64 (reference: unbounded int) */
};

/* predicate descriptor: a reproducible stand-in for the Python callables the
 * reference passes for `p : i64 -> bool` parameters (oracle.py:686-696). */
enum { IXP_LT = 0, IXP_GT, IXP_LE, IXP_GE, IXP_EQ, IXP_NE, IXP_HASH, IXP_TRUE, IXP_FALSE };
typedef struct { int32_t kind; int32_t pad; int64_t thr; uint64_t seed; } ixo_pred;

/* hist operators (oracle.py:110-114) */
enum { IXH_MIN = 0, IXH_MAX = 1, IXH_ADD = 2 };

typedef struct { int32_t code; int32_t site; int64_t elem; } ixo_status;

uint64_t ixo_mix64(uint64_t z);
uint64_t ixo_rand(uint64_t seed, uint64_t i);
int ixo_pred_eval(const ixo_pred* p, int64_t x);

/* ---- builtins (oracle.py:269-329) ---- */
int ixo_scan_add(int64_t ne, const int64_t* xs, int64_t n, int64_t* out);
int ixo_sgmsum(const int64_t* flags, const int64_t* xs, int64_t n, int64_t* out);
int ixo_scatter(const int64_t* dst, int64_t ndst, const int64_t* is, int64_t nis,
                const int64_t* vs, int64_t nvs, int64_t* out);
int ixo_hist(int op, int64_t ne, int64_t dlen, const int64_t* is, int64_t nis,
             const int64_t* vs, int64_t nvs, int64_t* out);
int ixo_gather(const int64_t* arr, int64_t len, const int64_t* idx, int64_t n,
               int64_t* out, int64_t* first_bad);

/* ---- corpus programs ---- */
int ixo_sum(const int64_t* xs, int64_t n, int64_t* out);
int ixo_partition2(const ixo_pred* p, const int64_t* xs, int64_t n,
                   int64_t* num_true, int64_t* ys);
int ixo_partition3(const ixo_pred* p, const ixo_pred* q, const int64_t* xs, int64_t n,
                   int64_t* m1, int64_t* m2, int64_t* ys);
int ixo_filter(const ixo_pred* p, const int64_t* xs, int64_t n, int64_t* ys, int64_t* count);
int ixo_filter_by(const int64_t* cs, const int64_t* xs, int64_t n, int64_t* ys, int64_t* count);
int ixo_mksgmdescr(const int64_t* shape, const int64_t* xs, int64_t m, int64_t nxs,
                   int64_t* res, int64_t cap, int64_t* len_out);
int ixo_mkii(const int64_t* shape, int64_t m, int64_t* out, int64_t cap, int64_t* len);
int ixo_mkflags(int64_t k, const int64_t* shape, int64_t m, int64_t* flags);
int ixo_c2(const ixo_pred* p, const int64_t* xs, int64_t n, const int64_t* shape, int64_t m,
           int64_t* ys, int64_t* zs, int64_t* k);
int ixo_get_smallest_pairs(int64_t n_verts, int64_t n_es, const int64_t* es, const int64_t* is,
                           int64_t n, int64_t* xs, int64_t* ys, int64_t* count,
                           ixo_status* st);
int ixo_kmeans_ker(int64_t row, const int64_t* pointers, int64_t np1,
                   const double* cluster, int64_t num_cols, const double* values,
                   const int64_t* indices, int64_t nnz, double* out, ixo_status* st);
int ixo_csrg(const int64_t* x, int64_t num_cols, const int64_t* values, const int64_t* indices,
             int64_t nnz, int64_t* out, int64_t* first_bad);
/* the jagged programs corpus/partition2l.ixl and corpus/filter_seg.ixl.
 * Inputs with sum shp > n make the reference's own k-ary scan index past the
 * shorter array (an uncaught IndexError): IXO_BADARG here. */
int ixo_partition2l(const int64_t* shp, int64_t m, const int64_t* cs, const int64_t* xs, int64_t n,
                    int64_t* ys);
int ixo_filter_seg(const int64_t* shp, int64_t m, const int64_t* cs, const int64_t* xs, int64_t n,
                   int64_t* newshp, int64_t* ys, int64_t* count);

/* ---- multi-threaded restatements used only as the timed CPU baseline
 *      (bench.py cpu_baseline / --impl reference).  Same results as the
 *      sequential functions above (checked in tests/test_oracle_golden.py). */
int ixo_par_threads(void);
int ixo_par_c2_i32(const ixo_pred* p, const int32_t* xs, int64_t n, const int64_t* shape,
                   int64_t m, int32_t* ys, int32_t* zs, int64_t* k, int threads);
int ixo_par_partition2_i32(const ixo_pred* p, const int32_t* xs, int64_t n,
                           int64_t* num_true, int32_t* ys, int threads);
/* scatter (oracle.py:294-305, with its idempotence check) and the CSR
 * gather (with its bounds check) at the BASELINE widths, OpenMP */
int ixo_par_scatter_i32(const int32_t* dst, int64_t ndst, const int64_t* is, const int32_t* vs, int64_t m,
                        int32_t* out, int threads);
int ixo_par_csrg_i32(const int32_t* x, int64_t ncols, const int32_t* vals, const int64_t* idx, int64_t nnz,
                     int32_t* out, int64_t* first_bad, int threads);

#ifdef __cplusplus
}
#endif
#endif
