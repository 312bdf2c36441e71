/*
 * ixoracle_par.c -- TEST INFRASTRUCTURE ONLY (see ixoracle.h).
 *
 * Multi-threaded (OpenMP) CPU restatements of two corpus pipelines at the
 * BASELINE storage widths (int32 values).  They are the timed CPU baseline of
 * bench.py (`cpu_baseline`, `--impl reference`): the reference itself is a
 * single-threaded Python interpreter that cannot travel to the GPU box, so the
 * baseline is this port, using every host thread.  Results are identical to
 * the sequential restatement (tests/test_oracle_golden.py checks it).
 *
 * Algorithm: blocked two-pass scans -- each thread reduces its contiguous
 * chunk, the per-chunk totals are scanned serially, each thread re-walks its
 * chunk with its carry-in.  This is the classic CPU form of the reference's
 * `scan (+) 0` (oracle.py:281-293) and of the segmented scan.
 */
#include <omp.h>
#include <stdlib.h>
#include <string.h>

#include "ixoracle.h"

int ixo_par_threads(void) { return omp_get_max_threads(); }

static void chunk(int64_t n, int t, int T, int64_t* lo, int64_t* hi) {
  *lo = n * t / T;
  *hi = n * (t + 1) / T;
}

/* partition2 (corpus/partition2.ixl) on int32 values. */
int ixo_par_partition2_i32(const ixo_pred* p, const int32_t* xs, int64_t n,
                           int64_t* num_true, int32_t* ys, int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  omp_set_dynamic(0);
  int64_t* cnt = (int64_t*)calloc((size_t)threads + 1, sizeof(int64_t));
  if (!cnt) return IXO_NOMEM;
  int Tn = threads;
  const ixo_pred P = *p;
#pragma omp parallel num_threads(threads)
  {
    int t = omp_get_thread_num(), T = omp_get_num_threads();
    int64_t lo, hi, c = 0;
    chunk(n, t, T, &lo, &hi);
    for (int64_t i = lo; i < hi; ++i) c += ixo_pred_eval(&P, xs[i]);
    cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
    {
      Tn = T;
      for (int k = 0; k < T; ++k) cnt[k + 1] += cnt[k];
    }
    int64_t nt = cnt[T];
    int64_t tb = cnt[t], fb = nt + (lo - cnt[t]);
    for (int64_t i = lo; i < hi; ++i) {
      int32_t x = xs[i];
      if (ixo_pred_eval(&P, x)) ys[tb++] = x; else ys[fb++] = x;
    }
  }
  *num_true = cnt[Tn];
  free(cnt);
  return IXO_OK;
}

/* c2 (corpus/c2_filter_sgmsum.ixl) on int32 values: filter, flag array from
 * shape (bitmap of segment starts below k), segmented inclusive sum.  zs is
 * accumulated in int64 and stored as int32 (IXO_OVERFLOW if it does not fit). */
int ixo_par_c2_i32(const ixo_pred* p, const int32_t* xs, int64_t n, const int64_t* shape,
                   int64_t m, int32_t* ys, int32_t* zs, int64_t* k_out, int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  omp_set_dynamic(0);
  int Tn = threads;
  int64_t* cnt = (int64_t*)calloc((size_t)threads + 1, sizeof(int64_t));
  int64_t* tail = (int64_t*)calloc((size_t)threads, sizeof(int64_t));
  unsigned char* hasf = (unsigned char*)calloc((size_t)threads, 1);
  int64_t* carry = (int64_t*)calloc((size_t)threads, sizeof(int64_t));
  int64_t* scn = (int64_t*)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
  uint64_t* bits = (uint64_t*)calloc((size_t)(n / 64 + 1), sizeof(uint64_t));
  int ovf = 0;
  if (!cnt || !tail || !hasf || !carry || !scn || !bits) {
    free(cnt); free(tail); free(hasf); free(carry); free(scn); free(bits);
    return IXO_NOMEM;
  }
  const ixo_pred P = *p;
  /* exclusive scan of shape (scan (+) 0 rot), serial: m << n */
  int64_t acc = 0;
  for (int64_t i = 0; i < m; ++i) { scn[i] = acc; acc += shape[i]; }
#pragma omp parallel num_threads(threads) reduction(| : ovf)
  {
    int t = omp_get_thread_num(), T = omp_get_num_threads();
    int64_t lo, hi, c = 0;
    chunk(n, t, T, &lo, &hi);
    for (int64_t i = lo; i < hi; ++i) c += ixo_pred_eval(&P, xs[i]);
    cnt[t + 1] = c;
#pragma omp barrier
#pragma omp single
    {
      Tn = T;
      for (int k = 0; k < T; ++k) cnt[k + 1] += cnt[k];
    }
    int64_t k_tot = cnt[T];
    /* flags: 1 at scn[i] for non-empty segments inside [0, k) (mkFlags) */
    int64_t slo, shi;
    chunk(m, t, T, &slo, &shi);
    for (int64_t i = slo; i < shi; ++i)
      if (shape[i] > 0 && scn[i] >= 0 && scn[i] < k_tot)
        __atomic_fetch_or(&bits[scn[i] >> 6], 1ULL << (scn[i] & 63), __ATOMIC_RELAXED);
    /* compaction */
    int64_t o = cnt[t];
    for (int64_t i = lo; i < hi; ++i)
      if (ixo_pred_eval(&P, xs[i])) ys[o++] = xs[i];
#pragma omp barrier
    /* segmented sum over ys[cnt[t], cnt[t+1]) : local aggregate */
    int64_t a = cnt[t], b = cnt[t + 1], v = 0;
    int hf = 0;
    for (int64_t j = a; j < b; ++j) {
      if ((bits[j >> 6] >> (j & 63)) & 1) { v = ys[j]; hf = 1; } else v += ys[j];
    }
    tail[t] = v;
    hasf[t] = (unsigned char)hf;
#pragma omp barrier
#pragma omp single
    {
      int64_t cv = 0;
      for (int k = 0; k < T; ++k) {
        carry[k] = cv;
        cv = hasf[k] ? tail[k] : cv + tail[k];
      }
    }
    v = carry[t];
    for (int64_t j = a; j < b; ++j) {
      if ((bits[j >> 6] >> (j & 63)) & 1) v = ys[j]; else v += ys[j];
      if (v != (int32_t)v) ovf = 1;
      zs[j] = (int32_t)v;
    }
  }
  *k_out = cnt[Tn];
  free(cnt); free(tail); free(hasf); free(carry); free(scn); free(bits);
  return ovf ? IXO_OVERFLOW : IXO_OK;
}

/* scatter dst is vs (oracle.py:294-305) on int32 values with int64 indices,
 * with the reference's dynamic checks: out = copy of dst, out-of-range
 * indices skipped, and NonIdempotentScatter (IXO_CONFLICT) iff one in-range
 * index receives two DIFFERENT values (equal-valued duplicates are legal,
 * oracle.py:301).  Parallel form: every in-range destination is claimed in a
 * bitmap with an atomic OR; only if some destination was claimed twice does a
 * second pass compare each pair's value with the value that landed. */
int ixo_par_scatter_i32(const int32_t* dst, int64_t ndst, const int64_t* is, const int32_t* vs, int64_t m,
                        int32_t* out, int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  omp_set_dynamic(0);
  uint64_t* claim = (uint64_t*)calloc((size_t)(ndst / 64 + 1), sizeof(uint64_t));
  if (!claim) return IXO_NOMEM;
  int dup = 0, conflict = 0;
#pragma omp parallel num_threads(threads) reduction(| : dup, conflict)
  {
    int t = omp_get_thread_num(), T = omp_get_num_threads();
    int64_t lo, hi;
    chunk(ndst, t, T, &lo, &hi);
    if (out != dst) memcpy(out + lo, dst + lo, (size_t)(hi - lo) * sizeof(int32_t));
#pragma omp barrier
    chunk(m, t, T, &lo, &hi);
    for (int64_t k = lo; k < hi; ++k) {
      const int64_t i = is[k];
      if (0 <= i && i < ndst) {
        const uint64_t bit = 1ULL << (i & 63);
        if (__atomic_fetch_or(&claim[i >> 6], bit, __ATOMIC_RELAXED) & bit) dup = 1;
        out[i] = vs[k];
      }
    }
  }
  if (dup) {
#pragma omp parallel for num_threads(threads) reduction(| : conflict)
    for (int64_t k = 0; k < m; ++k) {
      const int64_t i = is[k];
      if (0 <= i && i < ndst && out[i] != vs[k]) conflict = 1;
    }
  }
  free(claim);
  return conflict ? IXO_CONFLICT : IXO_OK;
}

/* CSR flat gather map2 (\v c -> v * x[c]) values indices (corpus
 * c4_csr_gather.ixl) on int32 values, with the reference's bounds check on
 * x[c] (oracle.py:177-184): IXO_OOB and *first_bad = the first failing index
 * in sequential order. */
int ixo_par_csrg_i32(const int32_t* x, int64_t ncols, const int32_t* vals, const int64_t* idx, int64_t nnz,
                     int32_t* out, int64_t* first_bad, int threads) {
  if (threads <= 0) threads = omp_get_max_threads();
  omp_set_dynamic(0);
  int64_t bad = nnz;
#pragma omp parallel for num_threads(threads) schedule(static) reduction(min : bad)
  for (int64_t i = 0; i < nnz; ++i) {
    const int64_t c = idx[i];
    if ((uint64_t)c >= (uint64_t)ncols) {
      if (i < bad) bad = i;
      continue;
    }
    out[i] = (int32_t)((int64_t)vals[i] * (int64_t)x[c]);
  }
  if (first_bad) *first_bad = bad;
  return bad < nnz ? IXO_OOB : IXO_OK;
}
