"""TEST INFRASTRUCTURE ONLY -- numpy/ctypes front-end of oracle/libixoracle.so.

The C library restates the reference interpreter (``oracle.py:90-333`` of
``/root/reference/pkg/src/ixverify``) and the corpus programs.  Only tests,
``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may import this
module; the product package never does.  Every function takes numpy arrays
(int64 unless stated) and returns numpy arrays, raising :class:`OracleFail`
with the reference's status code where the reference interpreter would raise.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libixoracle.so")

OK, OOB, CONFLICT, LENGTH, BADARG, NOMEM, OVERFLOW = range(7)
BUDGET = 100  # StepBudgetExceeded (oracle.py:118-125); Python-side cases only
HIST_MIN, HIST_MAX, HIST_ADD = 0, 1, 2


class OracleFail(Exception):
    def __init__(self, code, site=None, elem=None):
        super().__init__(f"oracle status {code} (site={site}, elem={elem})")
        self.code, self.site, self.elem = code, site, elem


class _Pred(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("pad", ctypes.c_int32), ("thr", ctypes.c_int64), ("seed", ctypes.c_uint64)]


class _Status(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int32), ("site", ctypes.c_int32), ("elem", ctypes.c_int64)]


_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else ctypes.c_void_p(0)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def cpred(p) -> _Pred:
    """Any object with kind/thr/seed (paper_2506_23058_b200.Pred)."""
    return _Pred(int(p.kind), 0, int(p.thr), int(p.seed) & ((1 << 64) - 1))


def _ok(rc, st=None):
    if rc != OK:
        if st is not None and st.code:
            raise OracleFail(rc, st.site, st.elem)
        raise OracleFail(rc)


# ---------------------------------------------------------------- builtins
def scan_add(xs, ne=0):
    xs = _i64(xs)
    out = np.empty_like(xs)
    _ok(lib().ixo_scan_add(ctypes.c_int64(ne), _p(xs), ctypes.c_int64(len(xs)), _p(out)))
    return out


def sgmsum(flags, xs):
    flags, xs = _i64(flags), _i64(xs)
    out = np.empty_like(xs)
    _ok(lib().ixo_sgmsum(_p(flags), _p(xs), ctypes.c_int64(len(xs)), _p(out)))
    return out


def scatter(dst, is_, vs):
    dst, is_, vs = _i64(dst), _i64(is_), _i64(vs)
    out = np.empty_like(dst)
    _ok(lib().ixo_scatter(_p(dst), ctypes.c_int64(len(dst)), _p(is_), ctypes.c_int64(len(is_)), _p(vs),
                          ctypes.c_int64(len(vs)), _p(out)))
    return out


def hist(op, ne, dlen, is_, vs):
    is_, vs = _i64(is_), _i64(vs)
    out = np.empty(max(dlen, 0), dtype=np.int64)
    _ok(lib().ixo_hist(op, ctypes.c_int64(ne), ctypes.c_int64(dlen), _p(is_), ctypes.c_int64(len(is_)), _p(vs),
                       ctypes.c_int64(len(vs)), _p(out)))
    return out


def gather(arr, idx):
    arr, idx = _i64(arr), _i64(idx)
    out = np.empty_like(idx)
    bad = ctypes.c_int64(-1)
    rc = lib().ixo_gather(_p(arr), ctypes.c_int64(len(arr)), _p(idx), ctypes.c_int64(len(idx)), _p(out),
                          ctypes.byref(bad))
    if rc:
        raise OracleFail(rc, 0, bad.value)
    return out


# ---------------------------------------------------------------- corpus
def sum_(xs):
    xs = _i64(xs)
    out = ctypes.c_int64(0)
    _ok(lib().ixo_sum(_p(xs), ctypes.c_int64(len(xs)), ctypes.byref(out)))
    return out.value


def partition2(p, xs):
    xs = _i64(xs)
    ys = np.empty_like(xs)
    nt = ctypes.c_int64(0)
    cp = cpred(p)
    _ok(lib().ixo_partition2(ctypes.byref(cp), _p(xs), ctypes.c_int64(len(xs)), ctypes.byref(nt), _p(ys)))
    return nt.value, ys


def partition3(p, q, xs):
    xs = _i64(xs)
    ys = np.empty_like(xs)
    m1, m2 = ctypes.c_int64(0), ctypes.c_int64(0)
    cp, cq = cpred(p), cpred(q)
    _ok(lib().ixo_partition3(ctypes.byref(cp), ctypes.byref(cq), _p(xs), ctypes.c_int64(len(xs)), ctypes.byref(m1),
                             ctypes.byref(m2), _p(ys)))
    return m1.value, m2.value, ys


def filter_(p, xs):
    xs = _i64(xs)
    ys = np.empty_like(xs)
    cnt = ctypes.c_int64(0)
    cp = cpred(p)
    _ok(lib().ixo_filter(ctypes.byref(cp), _p(xs), ctypes.c_int64(len(xs)), _p(ys), ctypes.byref(cnt)))
    return ys[: cnt.value].copy()


def filter_by(cs, xs):
    cs, xs = _i64(cs), _i64(xs)
    ys = np.empty_like(xs)
    cnt = ctypes.c_int64(0)
    _ok(lib().ixo_filter_by(_p(cs), _p(xs), ctypes.c_int64(len(xs)), _p(ys), ctypes.byref(cnt)))
    return ys[: cnt.value].copy()


def mksgmdescr(shape, xs):
    shape, xs = _i64(shape), _i64(xs)
    cap = int(max(0, shape.sum())) if len(shape) else 0
    cap = max(cap, 1)
    for _ in range(2):
        res = np.empty(cap, dtype=np.int64)
        ln = ctypes.c_int64(0)
        rc = lib().ixo_mksgmdescr(_p(shape), _p(xs), ctypes.c_int64(len(shape)), ctypes.c_int64(len(xs)), _p(res),
                                  ctypes.c_int64(cap), ctypes.byref(ln))
        if rc == BADARG and ln.value > cap:
            cap = ln.value
            continue
        _ok(rc)
        return res[: ln.value].copy()
    raise OracleFail(BADARG)


def mkii(shape):
    shape = _i64(shape)
    cap = max(1, int(max(0, shape.sum())) if len(shape) else 0)
    out = np.empty(cap, dtype=np.int64)
    ln = ctypes.c_int64(0)
    _ok(lib().ixo_mkii(_p(shape), ctypes.c_int64(len(shape)), _p(out), ctypes.c_int64(cap), ctypes.byref(ln)))
    return out[: ln.value].copy()


def mkflags(k, shape):
    shape = _i64(shape)
    out = np.empty(max(k, 1), dtype=np.int64)
    _ok(lib().ixo_mkflags(ctypes.c_int64(k), _p(shape), ctypes.c_int64(len(shape)), _p(out)))
    return out[: max(k, 0)].copy()


def c2(p, xs, shape):
    xs, shape = _i64(xs), _i64(shape)
    ys = np.empty(max(len(xs), 1), dtype=np.int64)
    zs = np.empty(max(len(xs), 1), dtype=np.int64)
    k = ctypes.c_int64(0)
    cp = cpred(p)
    _ok(lib().ixo_c2(ctypes.byref(cp), _p(xs), ctypes.c_int64(len(xs)), _p(shape), ctypes.c_int64(len(shape)), _p(ys),
                     _p(zs), ctypes.byref(k)))
    return ys[: k.value].copy(), zs[: k.value].copy()


def get_smallest_pairs(n_verts, n_es, es, is_):
    es, is_ = _i64(es), _i64(is_)
    n = len(es)
    xs = np.empty(max(n, 1), dtype=np.int64)
    ys = np.empty(max(n, 1), dtype=np.int64)
    cnt = ctypes.c_int64(0)
    st = _Status()
    rc = lib().ixo_get_smallest_pairs(ctypes.c_int64(n_verts), ctypes.c_int64(n_es), _p(es), _p(is_),
                                      ctypes.c_int64(n), _p(xs), _p(ys), ctypes.byref(cnt), ctypes.byref(st))
    _ok(rc, st)
    return xs[: cnt.value].copy(), ys[: cnt.value].copy()


def kmeans_ker(row, pointers, cluster, values, indices):
    pointers, indices = _i64(pointers), _i64(indices)
    cluster = np.ascontiguousarray(np.asarray(cluster, dtype=np.float64))
    values = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    out = ctypes.c_double(0.0)
    st = _Status()
    rc = lib().ixo_kmeans_ker(ctypes.c_int64(row), _p(pointers), ctypes.c_int64(len(pointers)), _p(cluster),
                              ctypes.c_int64(len(cluster)), _p(values), _p(indices), ctypes.c_int64(len(indices)),
                              ctypes.byref(out), ctypes.byref(st))
    _ok(rc, st)
    return out.value


def csrg(x, values, indices):
    x, values, indices = _i64(x), _i64(values), _i64(indices)
    out = np.empty_like(values)
    bad = ctypes.c_int64(-1)
    rc = lib().ixo_csrg(_p(x), ctypes.c_int64(len(x)), _p(values), _p(indices), ctypes.c_int64(len(values)), _p(out),
                        ctypes.byref(bad))
    if rc:
        raise OracleFail(rc, 0, bad.value)
    return out


# ---------------------------------------------------------------- CPU baseline (OpenMP)
def threads() -> int:
    return int(lib().ixo_par_threads())


def par_c2_i32(p, xs, shape, nthreads=0):
    xs = np.ascontiguousarray(xs, dtype=np.int32)
    shape = _i64(shape)
    ys = np.empty(max(len(xs), 1), dtype=np.int32)
    zs = np.empty(max(len(xs), 1), dtype=np.int32)
    k = ctypes.c_int64(0)
    cp = cpred(p)
    _ok(lib().ixo_par_c2_i32(ctypes.byref(cp), _p(xs), ctypes.c_int64(len(xs)), _p(shape), ctypes.c_int64(len(shape)),
                             _p(ys), _p(zs), ctypes.byref(k), int(nthreads)))
    return ys[: k.value], zs[: k.value]


def par_partition2_i32(p, xs, nthreads=0):
    xs = np.ascontiguousarray(xs, dtype=np.int32)
    ys = np.empty(max(len(xs), 1), dtype=np.int32)
    nt = ctypes.c_int64(0)
    cp = cpred(p)
    _ok(lib().ixo_par_partition2_i32(ctypes.byref(cp), _p(xs), ctypes.c_int64(len(xs)), ctypes.byref(nt), _p(ys),
                                     int(nthreads)))
    return nt.value, ys[: len(xs)]


def par_scatter_i32(dst, is_, vs, nthreads=0, out=None):
    """scatter with the reference's checks (ixo_par_scatter_i32, OpenMP)."""
    dst = np.ascontiguousarray(dst, dtype=np.int32)
    is_ = _i64(is_)
    vs = np.ascontiguousarray(vs, dtype=np.int32)
    out = np.empty(max(len(dst), 1), dtype=np.int32) if out is None else out
    m = min(len(is_), len(vs))
    _ok(lib().ixo_par_scatter_i32(_p(dst), ctypes.c_int64(len(dst)), _p(is_), _p(vs), ctypes.c_int64(m), _p(out),
                                  int(nthreads)))
    return out[: len(dst)]


def par_csrg_i32(x, vals, idx, nthreads=0, out=None):
    """map2 (\\v c -> v * x[c]) with its bounds check (ixo_par_csrg_i32, OpenMP)."""
    x = np.ascontiguousarray(x, dtype=np.int32)
    vals = np.ascontiguousarray(vals, dtype=np.int32)
    idx = _i64(idx)
    out = np.empty(max(len(vals), 1), dtype=np.int32) if out is None else out
    bad = ctypes.c_int64(0)
    rc = lib().ixo_par_csrg_i32(_p(x), ctypes.c_int64(len(x)), _p(vals), _p(idx), ctypes.c_int64(len(vals)), _p(out),
                                ctypes.byref(bad), int(nthreads))
    if rc:
        raise OracleFail(rc, 0, bad.value)
    return out[: len(vals)]


def partition2l(shp, cs, xs):
    """corpus/partition2l.ixl (ixo_partition2l)."""
    shp, cs, xs = _i64(shp), _i64(cs), _i64(xs)
    ys = np.empty_like(xs)
    _ok(lib().ixo_partition2l(_p(shp), ctypes.c_int64(len(shp)), _p(cs), _p(xs), ctypes.c_int64(len(xs)), _p(ys)))
    return ys


def filter_seg(shp, cs, xs):
    """corpus/filter_seg.ixl (ixo_filter_seg) -> (new row sizes, filtered values)."""
    shp, cs, xs = _i64(shp), _i64(cs), _i64(xs)
    newshp = np.empty_like(shp)
    ys = np.empty_like(xs)
    cnt = ctypes.c_int64(0)
    _ok(lib().ixo_filter_seg(_p(shp), ctypes.c_int64(len(shp)), _p(cs), _p(xs), ctypes.c_int64(len(xs)), _p(newshp),
                             _p(ys), ctypes.byref(cnt)))
    return newshp, ys[: cnt.value].copy()


# ---------------------------------------------------------------------------
# corpus/scanops.ixl: scan / hist with other operators.  Pure-Python loops
# (small cases only) restating the reference's folds: scan seeds the
# accumulators with the neutrals once and folds left to right
# (oracle.py:281-293); hist fills [ne] * dlen and applies the operator to each
# in-bounds bin in index order (oracle.py:306-316).
def fold_scan(op, nes, arrs):
    k = len(nes)
    acc = list(nes)
    n = len(arrs[0])
    outs = [[] for _ in range(k)]
    for i in range(n):
        r = op(*acc, *[a[i] for a in arrs])
        acc = list(r) if k > 1 else [r]
        for j in range(k):
            outs[j].append(acc[j])
    return tuple(outs) if k > 1 else outs[0]


def fold_hist(op, ne, dlen, is_, vs):
    dst = [ne] * dlen
    for i, v in zip(is_, vs):
        if 0 <= i < dlen:
            dst[i] = op(dst[i], v)
    return dst


def _lookup(tbl):
    def op(a, b):
        if not 0 <= b < len(tbl):
            raise OracleFail(OOB, site=0)
        return a + tbl[b]
    return op


def scanops(fun, a):
    """One corpus/scanops.ixl function on Python lists."""
    if fun == "scan_min":
        return fold_scan(lambda x, y: x if x < y else y, [7], [a[0]])
    if fun == "scan_max":
        return fold_scan(lambda x, y: x if y <= x else y, [-1], [a[0]])
    if fun == "scan_mul":
        return fold_scan(lambda x, y: x * y, [1], [a[0]])
    if fun == "scan_and":
        return fold_scan(lambda x, y: bool(x) and bool(y), [True], [a[0]])
    if fun == "scan_pair":
        return fold_scan(lambda a1, a2, b1, b2: (a1 + b1, a2 if a2 > b2 else b2), [3, -100], [a[0], a[1]])
    if fun == "scan_segmax":
        return fold_scan(lambda f1, v1, f2, v2: (bool(f1) or bool(f2), v2 if f2 else (v2 if v1 < v2 else v1)),
                         [False, -50], [a[0], a[1]])[1]
    if fun == "scan_clip":
        return fold_scan(lambda x, y: y if x > 20 else x + y, [0], [a[0]])
    if fun == "scan_lookup":
        return fold_scan(_lookup(a[0]), [0], [a[1]])
    if fun == "scan_fsum":
        return fold_scan(lambda x, y: x + y, [0.5], [a[0]])
    if fun == "scan_fmax":
        return fold_scan(lambda x, y: y if x < y else x, [0.0 - 100.0], [a[0]])
    if fun == "scan_decay":
        return fold_scan(lambda x, y: x * 0.5 + y, [0], [a[0]])
    if fun == "hist_fadd":
        return fold_hist(lambda x, y: x + y, 0.25, a[0], a[1], a[2])
    if fun == "hist_fmin":
        return fold_hist(lambda x, y: min(x, y), 100.0, a[0], a[1], a[2])
    if fun == "pairs":
        return [(x * 2, x > 3) for x in a[0]]
    if fun == "unpair":
        return [p[0] - p[1] for p in a[0]]
    if fun == "pair_pick":
        if not 0 <= a[1] < len(a[0]):
            raise OracleFail(OOB, site=0)
        x = a[0][a[1]]
        return (x + 1, x < 0)
    if fun == "hist_mul":
        return fold_hist(lambda x, y: x * y, 1, a[0], a[1], a[2])
    if fun == "hist_lmin":
        return fold_hist(lambda x, y: y if y < x else x, 9, a[0], a[1], a[2])
    if fun == "hist_last":
        return fold_hist(lambda x, y: y, 0, a[0], a[1], a[2])
    if fun == "hist_horner":
        return fold_hist(lambda x, y: x * 3 + y, 0, a[0], a[1], a[2])
    raise KeyError(fun)
