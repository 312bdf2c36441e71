/*
 * ixoracle.c -- TEST INFRASTRUCTURE ONLY (see ixoracle.h).
 *
 * Sequential, literal restatement of the reference interpreter
 * (/root/reference/pkg/src/ixverify/oracle.py) for the builtins on the hot path
 * and of the corpus programs statement by statement.  Intermediates are
 * materialised exactly as the interpreter materialises them, so the order of
 * evaluation -- and therefore which failure is reported first -- is the
 * reference's.  Compile with -ffp-contract=off (kmeans_ker is f64 and must not
 * be FMA-contracted, Python floats round after every operation).
 */
#include "ixoracle.h"

#include <stdlib.h>
#include <string.h>

#define ALLOC(T, n) ((T*)malloc(((n) > 0 ? (size_t)(n) : 1) * sizeof(T)))

/* ------------------------------------------------------------------------ */
/* counter-based generator + predicate semantics (shared with the device)   */

uint64_t ixo_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t ixo_rand(uint64_t seed, uint64_t i) {
  return ixo_mix64(i * 0x9E3779B97F4A7C15ULL + ixo_mix64(seed ^ 0x5851F42D4C957F2DULL));
}

/* `p x` of a predicate parameter (oracle.py:327-329 calls the bound value). */
int ixo_pred_eval(const ixo_pred* p, int64_t x) {
  switch (p->kind) {
    case IXP_LT: return x < p->thr;
    case IXP_GT: return x > p->thr;
    case IXP_LE: return x <= p->thr;
    case IXP_GE: return x >= p->thr;
    case IXP_EQ: return x == p->thr;
    case IXP_NE: return x != p->thr;
    case IXP_HASH: return (int)(ixo_mix64((uint64_t)x ^ p->seed) >> 63);
    case IXP_TRUE: return 1;
    default: return 0;
  }
}

static int add_ovf(int64_t a, int64_t b, int64_t* r) { return __builtin_add_overflow(a, b, r); }

/* ------------------------------------------------------------------------ */
/* builtins                                                                  */

/* scan (+) ne xs  -- oracle.py:281-293 with f = (+), k = 1:
 *   acc = ne; for i: acc = acc + xs[i]; out.append(acc)      (ne folded once) */
int ixo_scan_add(int64_t ne, const int64_t* xs, int64_t n, int64_t* out) {
  int64_t acc = ne;
  for (int64_t i = 0; i < n; ++i) {
    if (add_ovf(acc, xs[i], &acc)) return IXO_OVERFLOW;
    out[i] = acc;
  }
  return IXO_OK;
}

/* sgmSum (corpus/c2_filter_sgmsum.ixl sgmSum): the 2-ary
 * scan of oracle.py:281-293 with the lifted operator
 *   \f1 v1 f2 v2 -> (f1 || f2, if f2 then v2 else v1 + v2),  ne = (false, 0).
 * Only the value component is returned (the program binds `(_, zs)`). */
int ixo_sgmsum(const int64_t* flags, const int64_t* xs, int64_t n, int64_t* out) {
  int64_t v = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (flags[i]) {
      v = xs[i];
    } else if (add_ovf(v, xs[i], &v)) {
      return IXO_OVERFLOW;
    }
    out[i] = v;
  }
  return IXO_OK;
}

/* scatter dst is vs -- oracle.py:294-305:
 *   dst = list(dst); written = {}
 *   for i, v in zip(is, vs):                 # zip truncates
 *     if 0 <= i < len(dst):                  # OOB silently ignored
 *       if i in written and written[i] != v: raise NonIdempotentScatter
 *       written[i] = v; dst[i] = v
 * out must hold ndst values (it receives the copy). */
int ixo_scatter(const int64_t* dst, int64_t ndst, const int64_t* is, int64_t nis,
                const int64_t* vs, int64_t nvs, int64_t* out) {
  int64_t m = nis < nvs ? nis : nvs;
  if (ndst < 0) ndst = 0;
  if (out != dst && ndst) memcpy(out, dst, (size_t)ndst * sizeof(int64_t));
  unsigned char* written = (unsigned char*)calloc(ndst > 0 ? (size_t)ndst : 1, 1);
  if (!written) return IXO_NOMEM;
  int rc = IXO_OK;
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = is[k];
    if (0 <= i && i < ndst) {
      if (written[i] && out[i] != vs[k]) { rc = IXO_CONFLICT; break; }
      written[i] = 1;
      out[i] = vs[k];
    }
  }
  free(written);
  return rc;
}

/* hist op ne dlen is vs -- oracle.py:306-316:
 *   dst = [ne] * dlen; for i, v in zip(is, vs): if 0 <= i < dlen: dst[i] = op(dst[i], v) */
int ixo_hist(int op, int64_t ne, int64_t dlen, const int64_t* is, int64_t nis,
             const int64_t* vs, int64_t nvs, int64_t* out) {
  int64_t m = nis < nvs ? nis : nvs;
  for (int64_t i = 0; i < dlen; ++i) out[i] = ne;
  for (int64_t k = 0; k < m; ++k) {
    int64_t i = is[k];
    if (0 <= i && i < dlen) {
      int64_t a = out[i], v = vs[k];
      if (op == IXH_MIN) out[i] = v < a ? v : a;
      else if (op == IXH_MAX) out[i] = v > a ? v : a;
      else if (add_ovf(a, v, &out[i])) return IXO_OVERFLOW;
    }
  }
  return IXO_OK;
}

/* map (\i -> arr[i]) idx -- IndexE, oracle.py:177-184:
 *   if not 0 <= idx < len(arr): raise OutOfBounds(expr_str(e), e.pos)
 * The map stops at the first failing element (oracle.py:280 list comp). */
int ixo_gather(const int64_t* arr, int64_t len, const int64_t* idx, int64_t n,
               int64_t* out, int64_t* first_bad) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = idx[i];
    if (!(0 <= c && c < len)) { if (first_bad) *first_bad = i; return IXO_OOB; }
    out[i] = arr[c];
  }
  return IXO_OK;
}

/* ------------------------------------------------------------------------ */
/* corpus programs                                                           */

/* sum -- filter.ixl:1-2 (and every corpus file):
 *   if n > 0 then (scan (+) 0 xs)[n-1] else 0 */
int ixo_sum(const int64_t* xs, int64_t n, int64_t* out) {
  if (n <= 0) { *out = 0; return IXO_OK; }
  int64_t* s = ALLOC(int64_t, n);
  if (!s) return IXO_NOMEM;
  int rc = ixo_scan_add(0, xs, n, s);
  if (rc == IXO_OK) *out = s[n - 1];
  free(s);
  return rc;
}

/* partition2 -- /root/reference/pkg/corpus/partition2.ixl:8-19 */
int ixo_partition2(const ixo_pred* p, const int64_t* xs, int64_t n,
                   int64_t* num_true_out, int64_t* ys) {
  int rc = IXO_NOMEM;
  int64_t *cs = ALLOC(int64_t, n), *flagsT = ALLOC(int64_t, n), *flagsF = ALLOC(int64_t, n);
  int64_t *indicesT = ALLOC(int64_t, n), *tmp = ALLOC(int64_t, n), *indicesF = ALLOC(int64_t, n);
  int64_t *indices = ALLOC(int64_t, n), *zeros = ALLOC(int64_t, n);
  if (!cs || !flagsT || !flagsF || !indicesT || !tmp || !indicesF || !indices || !zeros) goto out;
  for (int64_t i = 0; i < n; ++i) cs[i] = ixo_pred_eval(p, xs[i]);          /* :8  */
  for (int64_t i = 0; i < n; ++i) flagsT[i] = cs[i] ? 1 : 0;                /* :9  */
  for (int64_t i = 0; i < n; ++i) flagsF[i] = 1 - flagsT[i];                 /* :10 */
  if ((rc = ixo_scan_add(0, flagsT, n, indicesT))) goto out;                 /* :11 */
  int64_t num_true = n > 0 ? indicesT[n - 1] : 0;                            /* :12 */
  if ((rc = ixo_scan_add(0, flagsF, n, tmp))) goto out;                      /* :13 */
  for (int64_t i = 0; i < n; ++i) indicesF[i] = tmp[i] + num_true;           /* :14 */
  for (int64_t i = 0; i < n; ++i)                                            /* :15-16 */
    indices[i] = cs[i] ? indicesT[i] - 1 : indicesF[i] - 1;
  for (int64_t i = 0; i < n; ++i) zeros[i] = 0;                              /* :17 */
  rc = ixo_scatter(zeros, n, indices, n, xs, n, ys);                         /* :18 */
  *num_true_out = num_true;                                                  /* :19 */
out:
  free(cs); free(flagsT); free(flagsF); free(indicesT); free(tmp); free(indicesF);
  free(indices); free(zeros);
  return rc;
}

/* partition3 -- /root/reference/pkg/corpus/partition3.ixl:10-27 */
int ixo_partition3(const ixo_pred* p, const ixo_pred* q, const int64_t* xs, int64_t n,
                   int64_t* m1_out, int64_t* m2_out, int64_t* ys) {
  int rc = IXO_NOMEM;
  int64_t *cs1 = ALLOC(int64_t, n), *cs2 = ALLOC(int64_t, n), *f1 = ALLOC(int64_t, n);
  int64_t *f2 = ALLOC(int64_t, n), *o1 = ALLOC(int64_t, n), *o2 = ALLOC(int64_t, n);
  int64_t *inds = ALLOC(int64_t, n), *zeros = ALLOC(int64_t, n);
  if (!cs1 || !cs2 || !f1 || !f2 || !o1 || !o2 || !inds || !zeros) goto out;
  for (int64_t i = 0; i < n; ++i) cs1[i] = ixo_pred_eval(p, xs[i]);                 /* :10 */
  for (int64_t i = 0; i < n; ++i) cs2[i] = !cs1[i] && ixo_pred_eval(q, xs[i]);      /* :11 */
  for (int64_t i = 0; i < n; ++i) f1[i] = cs1[i] ? 1 : 0;                           /* :12 */
  for (int64_t i = 0; i < n; ++i) f2[i] = cs2[i] ? 1 : 0;                           /* :13 */
  if ((rc = ixo_scan_add(0, f1, n, o1))) goto out;                                  /* :14 */
  if ((rc = ixo_scan_add(0, f2, n, o2))) goto out;                                  /* :15 */
  int64_t m1 = n > 0 ? o1[n - 1] : 0;                                               /* :16 */
  int64_t m2 = n > 0 ? o2[n - 1] : 0;                                               /* :17 */
  for (int64_t i = 0; i < n; ++i) {                                                 /* :18-24 */
    int64_t is = i;                                  /* iota n */
    int64_t inds1 = o1[i] - 1;
    int64_t inds2 = m1 + o2[i] - 1;
    int64_t tmp = o1[i] + o2[i];
    int64_t inds3 = m1 + m2 + is - tmp;
    int64_t rest = cs2[i] ? inds2 : inds3;
    inds[i] = cs1[i] ? inds1 : rest;
  }
  for (int64_t i = 0; i < n; ++i) zeros[i] = 0;                                     /* :25 */
  rc = ixo_scatter(zeros, n, inds, n, xs, n, ys);                                   /* :26 */
  *m1_out = m1;
  *m2_out = m2;
out:
  free(cs1); free(cs2); free(f1); free(f2); free(o1); free(o2); free(inds); free(zeros);
  return rc;
}

/* filter_by -- /root/reference/pkg/corpus/maxmatching.ixl:1-9 (cs given);
 * ys must hold n values, *count receives the result length. */
int ixo_filter_by(const int64_t* cs, const int64_t* xs, int64_t n, int64_t* ys, int64_t* count_out) {
  int rc = IXO_NOMEM;
  int64_t *flags = ALLOC(int64_t, n), *offs = ALLOC(int64_t, n), *inds = ALLOC(int64_t, n);
  int64_t* zeros = NULL;
  if (!flags || !offs || !inds) goto out;
  for (int64_t i = 0; i < n; ++i) flags[i] = cs[i] ? 1 : 0;                 /* :3 */
  if ((rc = ixo_scan_add(0, flags, n, offs))) goto out;                      /* :4 */
  int64_t count = n > 0 ? offs[n - 1] : 0;                                   /* :5 */
  for (int64_t i = 0; i < n; ++i) inds[i] = cs[i] ? offs[i] - 1 : -1;       /* :6 */
  zeros = ALLOC(int64_t, count);                                              /* :7 */
  if (!zeros) { rc = IXO_NOMEM; goto out; }
  for (int64_t i = 0; i < count; ++i) zeros[i] = 0;
  rc = ixo_scatter(zeros, count, inds, n, xs, n, ys);                        /* :8 */
  *count_out = count;
out:
  free(flags); free(offs); free(inds); free(zeros);
  return rc;
}

/* filter -- /root/reference/pkg/corpus/filter.ixl:8-15 */
int ixo_filter(const ixo_pred* p, const int64_t* xs, int64_t n, int64_t* ys, int64_t* count) {
  int64_t* cs = ALLOC(int64_t, n);
  if (!cs) return IXO_NOMEM;
  for (int64_t i = 0; i < n; ++i) cs[i] = ixo_pred_eval(p, xs[i]);          /* :8 */
  int rc = ixo_filter_by(cs, xs, n, ys, count);                              /* :9-14, same body */
  free(cs);
  return rc;
}

/* shared prefix of mkSgmDescr / mkFlags (mksgmdescr.ixl:6-8):
 *   rot = map (\i -> if i == 0 then 0 else shape[i-1]) (iota m)
 *   scn = scan (+) 0 rot
 *   ind = map2 (\s o -> if s <= 0 then -1 else o) shape scn              */
static int seg_starts(const int64_t* shape, int64_t m, int64_t* scn, int64_t* ind) {
  int64_t* rot = ALLOC(int64_t, m);
  if (!rot) return IXO_NOMEM;
  for (int64_t i = 0; i < m; ++i) rot[i] = i == 0 ? 0 : shape[i - 1];
  int rc = ixo_scan_add(0, rot, m, scn);
  free(rot);
  if (rc) return rc;
  for (int64_t i = 0; i < m; ++i) ind[i] = shape[i] <= 0 ? -1 : scn[i];
  return IXO_OK;
}

/* mkSgmDescr -- /root/reference/pkg/corpus/mksgmdescr.ixl:4-11.
 * *len receives max(len, 0); IXO_BADARG if it exceeds cap. */
int ixo_mksgmdescr(const int64_t* shape, const int64_t* xs, int64_t m, int64_t nxs,
                   int64_t* res, int64_t cap, int64_t* len_out) {
  int64_t *scn = ALLOC(int64_t, m), *ind = ALLOC(int64_t, m);
  int64_t* zeros = NULL;
  int rc = IXO_NOMEM;
  if (!scn || !ind) goto out;
  if ((rc = seg_starts(shape, m, scn, ind))) goto out;
  int64_t len = 0;                                                          /* :9 */
  if (m > 0 && add_ovf(scn[m - 1], shape[m - 1], &len)) { rc = IXO_OVERFLOW; goto out; }
  if (len < 0) len = 0;                       /* [0] * negative == [] in Python */
  *len_out = len;
  if (len > cap) { rc = IXO_BADARG; goto out; }
  zeros = ALLOC(int64_t, len);
  if (!zeros) { rc = IXO_NOMEM; goto out; }
  for (int64_t i = 0; i < len; ++i) zeros[i] = 0;
  rc = ixo_scatter(zeros, len, ind, m, xs, nxs, res);     /* :10, zip(ind, xs) truncates */
out:
  free(scn); free(ind); free(zeros);
  return rc;
}

/* mkII -- PAPER.md:412-417 (corpus/mkii.ixl of this repo) */
int ixo_mkii(const int64_t* shape, int64_t m, int64_t* out, int64_t cap, int64_t* len) {
  int64_t* beg = ALLOC(int64_t, m);
  if (!beg) return IXO_NOMEM;
  for (int64_t i = 0; i < m; ++i) beg[i] = i + 1;
  int64_t* s1 = ALLOC(int64_t, cap);
  int64_t* fl = ALLOC(int64_t, cap);
  int rc = IXO_NOMEM;
  if (!s1 || !fl) goto out;
  if ((rc = ixo_mksgmdescr(shape, beg, m, m, s1, cap, len))) goto out;
  for (int64_t i = 0; i < *len; ++i) s1[i] = s1[i] == 0 ? 0 : s1[i] - 1;
  for (int64_t i = 0; i < *len; ++i) fl[i] = s1[i] > 0;
  rc = ixo_sgmsum(fl, s1, *len, out);
out:
  free(beg); free(s1); free(fl);
  return rc;
}

/* mkFlags -- corpus/c2_filter_sgmsum.ixl of this repo: the Ss2 flag-array
 * builder: scatter (replicate k 0) ind (replicate m 1). */
int ixo_mkflags(int64_t k, const int64_t* shape, int64_t m, int64_t* flags) {
  int64_t *scn = ALLOC(int64_t, m), *ind = ALLOC(int64_t, m), *ones = ALLOC(int64_t, m);
  int64_t* zeros = NULL;
  int rc = IXO_NOMEM;
  if (!scn || !ind || !ones) goto out;
  if ((rc = seg_starts(shape, m, scn, ind))) goto out;
  for (int64_t i = 0; i < m; ++i) ones[i] = 1;
  if (k < 0) k = 0;
  zeros = ALLOC(int64_t, k);
  if (!zeros) { rc = IXO_NOMEM; goto out; }
  for (int64_t i = 0; i < k; ++i) zeros[i] = 0;
  rc = ixo_scatter(zeros, k, ind, m, ones, m, flags);
out:
  free(scn); free(ind); free(ones); free(zeros);
  return rc;
}

/* c2 -- corpus/c2_filter_sgmsum.ixl: ys = filter p xs; k = length ys;
 * flags = mkFlags k shape; zs = sgmSum flags ys.  ys, zs hold n values. */
int ixo_c2(const ixo_pred* p, const int64_t* xs, int64_t n, const int64_t* shape, int64_t m,
           int64_t* ys, int64_t* zs, int64_t* k_out) {
  int64_t k = 0;
  int rc = ixo_filter(p, xs, n, ys, &k);
  if (rc) return rc;
  int64_t* flags = ALLOC(int64_t, k);
  if (!flags) return IXO_NOMEM;
  rc = ixo_mkflags(k, shape, m, flags);
  if (!rc) rc = ixo_sgmsum(flags, ys, k, zs);
  free(flags);
  *k_out = k;
  return rc;
}

/* get_smallest_pairs -- /root/reference/pkg/corpus/maxmatching.ixl:11-21 */
int ixo_get_smallest_pairs(int64_t n_verts, int64_t n_es, const int64_t* es, const int64_t* is,
                           int64_t n, int64_t* xs, int64_t* ys, int64_t* count, ixo_status* st) {
  int64_t dlen = n_verts > 0 ? n_verts : 0;
  int64_t *H = ALLOC(int64_t, dlen), *cs = ALLOC(int64_t, n);
  int rc = IXO_NOMEM;
  if (st) { st->code = 0; st->site = 0; st->elem = 0; }
  if (!H || !cs) goto out;
  if ((rc = ixo_hist(IXH_MIN, n_es, n_verts, es, n, is, n, H))) goto out;   /* :17 */
  for (int64_t i = 0; i < n; ++i) {                                         /* :18 */
    int64_t e = es[i];
    if (!(0 <= e && e < dlen)) {
      rc = IXO_OOB;
      if (st) { st->code = IXO_OOB; st->site = 0; st->elem = i; }
      goto out;
    }
    cs[i] = H[e] == is[i];
  }
  int64_t c2 = 0;
  if ((rc = ixo_filter_by(cs, es, n, xs, count))) goto out;                  /* :19 */
  rc = ixo_filter_by(cs, is, n, ys, &c2);                                    /* :20 */
out:
  free(H); free(cs);
  return rc;
}

/* kmeans_ker -- /root/reference/pkg/corpus/kmeans_ker.ixl:8-16, the five
 * indexing sites in evaluation order:
 *   0 pointers[row]  1 pointers[row+1]  2 values[index_start+j]
 *   3 indices[index_start+j]  4 cluster[column]
 * f64 arithmetic with one rounding per operation (Python float). */
int ixo_kmeans_ker(int64_t row, const int64_t* pointers, int64_t np1,
                   const double* cluster, int64_t num_cols, const double* values,
                   const int64_t* indices, int64_t nnz, double* out, ixo_status* st) {
#define KFAIL(s, e) do { if (st) { st->code = IXO_OOB; st->site = (s); st->elem = (e); } return IXO_OOB; } while (0)
  if (st) { st->code = 0; st->site = 0; st->elem = 0; }
  if (!(0 <= row && row < np1)) KFAIL(0, 0);
  int64_t index_start = pointers[row];
  if (!(0 <= row + 1 && row + 1 < np1)) KFAIL(1, 0);
  int64_t nnz_sgm = pointers[row + 1] - index_start;
  volatile double correction = 0.0;
  for (int64_t j = 0; j < nnz_sgm; ++j) {
    int64_t a = index_start + j;
    if (!(0 <= a && a < nnz)) KFAIL(2, j);
    double element_value = values[a];
    if (!(0 <= a && a < nnz)) KFAIL(3, j);
    int64_t column = indices[a];
    if (!(0 <= column && column < num_cols)) KFAIL(4, j);
    double cluster_value = cluster[column];
    volatile double two_c = 2.0 * cluster_value;
    volatile double diff = element_value - two_c;
    volatile double prod = diff * element_value;
    correction = correction + prod;
  }
  *out = correction;
  return IXO_OK;
#undef KFAIL
}

/* csrg -- corpus/c4_csr_gather.ixl: map2 (\v c -> v * x[c]) values indices */
int ixo_csrg(const int64_t* x, int64_t num_cols, const int64_t* values, const int64_t* indices,
             int64_t nnz, int64_t* out, int64_t* first_bad) {
  for (int64_t i = 0; i < nnz; ++i) {
    int64_t c = indices[i];
    if (!(0 <= c && c < num_cols)) { if (first_bad) *first_bad = i; return IXO_OOB; }
    if (__builtin_mul_overflow(values[i], x[c], &out[i])) return IXO_OVERFLOW;
  }
  return IXO_OK;
}

/* partition2L -- corpus/partition2l.ixl, statement by
 * statement.  II = mkII shp has length L = sum shp; the reference's sgmSum
 * scans L elements of fs (so L <= n, else its scan raises IndexError). */
int ixo_partition2l(const int64_t* shp, int64_t m, const int64_t* cs, const int64_t* xs, int64_t n,
                    int64_t* ys) {
  int64_t L = 0;
  for (int64_t k = 0; k < m; ++k) L += shp[k] > 0 ? shp[k] : 0;
  if (L > n) return IXO_BADARG;
  int64_t cap = L > 0 ? L : 1;
  int64_t *II = ALLOC(int64_t, cap), *offs = ALLOC(int64_t, m > 0 ? m : 1), *ones = ALLOC(int64_t, m > 0 ? m : 1);
  int64_t *descr = ALLOC(int64_t, cap), *fl = ALLOC(int64_t, cap), *tb = ALLOC(int64_t, cap);
  int64_t *rtot = ALLOC(int64_t, m > 0 ? m : 1), *inds = ALLOC(int64_t, n > 0 ? n : 1), *zeros = ALLOC(int64_t, n > 0 ? n : 1);
  int64_t len = 0;
  int rc = IXO_NOMEM;
  if (!II || !offs || !ones || !descr || !fl || !tb || !rtot || !inds || !zeros) goto out;
  if ((rc = ixo_mkii(shp, m, II, cap, &len))) goto out;                          /* :32 */
  int64_t acc = 0;                                                                /* :33-34 */
  for (int64_t k = 0; k < m; ++k) {
    acc += k == 0 ? 0 : shp[k - 1];
    offs[k] = acc;
    ones[k] = 1;                                                                  /* :35 */
  }
  if ((rc = ixo_mksgmdescr(shp, ones, m, m, descr, cap, &len))) goto out;       /* :36 */
  for (int64_t i = 0; i < len; ++i) fl[i] = descr[i] > 0;                         /* :37 */
  if ((rc = ixo_sgmsum(fl, cs, len, tb))) goto out;                               /* :38-39: fs = cs as 0/1 */
  for (int64_t k = 0; k < m; ++k) {                                               /* :40 */
    if (shp[k] > 0) {
      const int64_t j = offs[k] + shp[k] - 1;
      if (j < 0 || j >= len) { rc = IXO_OOB; goto out; }
      rtot[k] = tb[j];
    } else {
      rtot[k] = 0;
    }
  }
  for (int64_t i = 0; i < n; ++i) {                                               /* :41 */
    if (i >= len) { rc = IXO_OOB; goto out; }                                     /* II[i] */
    inds[i] = cs[i] ? offs[II[i]] + tb[i] - 1 : i + rtot[II[i]] - tb[i];
  }
  for (int64_t i = 0; i < n; ++i) zeros[i] = 0;
  rc = ixo_scatter(zeros, n, inds, n, xs, n, ys);                                 /* :42 */
out:
  free(II); free(offs); free(ones); free(descr); free(fl); free(tb); free(rtot); free(inds); free(zeros);
  return rc;
}

/* filter_seg -- corpus/filter_seg.ixl: filter.ixl's compaction, then the new
 * row sizes from the running count at each row's ends (statement order: all
 * `before` gathers, then all `upto` gathers). */
int ixo_filter_seg(const int64_t* shp, int64_t m, const int64_t* cs, const int64_t* xs, int64_t n,
                   int64_t* newshp, int64_t* ys, int64_t* count) {
  int64_t *offs = ALLOC(int64_t, n > 0 ? n : 1), *starts = ALLOC(int64_t, m > 0 ? m : 1);
  int64_t *before = ALLOC(int64_t, m > 0 ? m : 1), *upto = ALLOC(int64_t, m > 0 ? m : 1);
  int rc = IXO_NOMEM;
  if (!offs || !starts || !before || !upto) goto out;
  int64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) offs[i] = (acc += cs[i] ? 1 : 0);                /* :9-10 */
  if ((rc = ixo_filter_by(cs, xs, n, ys, count))) goto out;                          /* :11-13 */
  acc = 0;
  for (int64_t k = 0; k < m; ++k) starts[k] = (acc += k == 0 ? 0 : shp[k - 1]);     /* :14-15 */
  for (int64_t k = 0; k < m; ++k) {                                                  /* :16 */
    const int64_t st = starts[k];
    if (st > 0) {
      if (st - 1 >= n) { rc = IXO_OOB; goto out; }
      before[k] = offs[st - 1];
    } else {
      before[k] = 0;
    }
  }
  for (int64_t k = 0; k < m; ++k) {                                                  /* :17 */
    if (shp[k] > 0) {
      const int64_t j = starts[k] + shp[k] - 1;
      if (j < 0 || j >= n) { rc = IXO_OOB; goto out; }
      upto[k] = offs[j];
    } else {
      upto[k] = 0;
    }
  }
  for (int64_t k = 0; k < m; ++k) newshp[k] = shp[k] > 0 ? upto[k] - before[k] : 0;  /* :18 */
  rc = IXO_OK;
out:
  free(offs); free(starts); free(before); free(upto);
  return rc;
}
