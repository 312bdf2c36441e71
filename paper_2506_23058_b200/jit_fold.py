"""scan and hist with any operator (oracle.py:281-293, 306-316), compiled
from the operator lambda with NVRTC like the generic map (jit.py).

The reference folds a scan left to right, seeded with the neutrals once
(`acc = f(*acc, *x_i)`, oracle.py:288-292), and a hist updates each
in-bounds bin in index order (`dst[i] = op(dst[i], v)`, oracle.py:313-315).
A parallel evaluation reproduces that only where the operator is
associative (scan) or associative and commutative (hist), so the operator
is classified first, structurally, after resolving normalization's
let-bound temporaries:

* associative (scan -> three-kernel tiled scan, reduce / carry / down):
  `a + b`, `a * b`, `a && b`, `a || b`, the projections `a` and `b`, and
  `if a <cmp> b then a|b else b|a` (min, max or a projection); k-ary
  operators that apply one of those per component; the segmented lift
  `(f1 || f2, if f2 then v2 else v1 (+) v2)` of any of them
  (PAPER.md:399-402).  Modular int64 arithmetic keeps `+` and `*`
  associative, so the parallel result is bit-identical to the left fold.
* associative and commutative (hist -> one CAS loop per element): `+`, `*`,
  `&&`, `||`, min and max (`+`, min and max go to the existing k_hist).
* anything else -- including an operator that indexes a captured array,
  whose CHECKED sites must fail at the first failure in sequential order --
  runs as the exact left fold on the device: one thread walks the elements
  in order over shared-memory-staged tiles, evaluating the operator inline
  with the same site checks as the map kernels.

Every value is an int64 on the device (bool as 0/1, like Python's bools in
arithmetic); the caller converts bool-typed components back.
"""

from __future__ import annotations

import ctypes
import hashlib

import torch

from . import ir
from .jit import _CACHE, _PRELUDE, LAUNCHES, _ctype, _Gen, _Kernel, _ok, _scalar_param, budget_arg, scalar_args
from .vm import Unsupported

_CMPS = ("<", "<=", ">", ">=", "==", "!=")


# --------------------------------------------------------------- classifier
class _Shape:
    """A lambda body with its let-bound temporaries resolvable (names from
    normalization are fresh; anything shadowed or impure is rejected)."""

    def __init__(self, lam):
        self.ok = True
        self.binds: dict = {}
        self._walk(lam.body, set(lam.params))

    def _walk(self, e, params):
        k = ir.kind(e)
        if k in ("IndexE", "App", "Loop", "Lambda"):
            self.ok = False
            return
        if k == "Let":
            if len(e.names) != 1 or e.names[0] in self.binds or e.names[0] in params:
                self.ok = False
                return
            self.binds[e.names[0]] = e.rhs
        for f in ("lhs", "rhs", "arg", "cond", "then", "els", "body"):
            x = getattr(e, f, None)
            if x is not None and not isinstance(x, (str, int, float, bool)):
                self._walk(x, params)
        for x in getattr(e, "items", ()) or ():
            self._walk(x, params)

    def r(self, e):
        while True:
            k = ir.kind(e)
            if k == "Let":
                e = e.body
            elif k == "VarE" and e.name in self.binds:
                e = self.binds[e.name]
            else:
                return e

    def var(self, e):
        e = self.r(e)
        return e.name if ir.kind(e) == "VarE" else None

    def binary(self, e, a, b):
        """-> 'add' | 'mul' | 'and' | 'or' | 'min' | 'max' | 'left' |
        'right' | None: e as an operator of (a, b) in that order."""
        e = self.r(e)
        k = ir.kind(e)
        if k == "VarE":
            return {a: "left", b: "right"}.get(e.name)
        if k == "BinOp" and e.op in ("+", "*", "&&", "||"):
            if {self.var(e.lhs), self.var(e.rhs)} == {a, b}:
                return {"+": "add", "*": "mul", "&&": "and", "||": "or"}[e.op]
            return None
        if k == "If":
            c = self.r(e.cond)
            if ir.kind(c) != "BinOp" or c.op not in _CMPS:
                return None
            x, y, t, f = self.var(c.lhs), self.var(c.rhs), self.var(e.then), self.var(e.els)
            if {x, y} != {a, b} or {t, f} != {a, b}:
                return None
            if c.op in ("==", "!="):  # x == y ? t : f  is always f (resp. t)
                keep = f if c.op == "==" else t
                return "left" if keep == a else "right"
            smaller_first = c.op in ("<", "<=")  # cond true <=> x is the smaller
            picks_x = t == x
            return "min" if smaller_first == picks_x else "max"
        return None


def classify_scan(lam, k: int) -> bool:
    """True iff the k-ary scan operator is recognisably associative."""
    if ir.kind(lam) != "Lambda" or len(lam.params) != 2 * k:
        return False
    sh = _Shape(lam)
    if not sh.ok:
        return False
    accs, els = lam.params[:k], lam.params[k:]
    if len(set(lam.params)) != 2 * k or "_" in lam.params:
        return False
    if k == 1:
        return sh.binary(lam.body, accs[0], els[0]) is not None
    body = sh.r(lam.body)
    if ir.kind(body) != "TupleE" or len(body.items) != k:
        return False
    if all(sh.binary(it, accs[j], els[j]) is not None for j, it in enumerate(body.items)):
        return True
    if k == 2:  # segmented lift (f1 || f2, if f2 then v2 else v1 (+) v2)
        f1, v1 = accs
        f2, v2 = els
        fl, v = body.items[0], sh.r(body.items[1])
        if sh.binary(fl, f1, f2) != "or" or ir.kind(v) != "If":
            return False
        c = sh.r(v.cond)
        if sh.var(c) == f2:
            keep, comb = v.then, v.els
        elif ir.kind(c) == "NotE" and sh.var(c.arg) == f2:
            keep, comb = v.els, v.then
        else:
            return False
        return sh.var(keep) == v2 and sh.binary(comb, v1, v2) is not None
    return False


def classify_hist(lam) -> str | None:
    """'add' | 'mul' | 'and' | 'or' | 'min' | 'max' when the operator is
    associative and commutative, else None (the in-order fold)."""
    if ir.kind(lam) != "Lambda" or len(lam.params) != 2 or len(set(lam.params)) != 2 or "_" in lam.params:
        return None
    sh = _Shape(lam)
    if not sh.ok:
        return None
    op = sh.binary(lam.body, *lam.params)
    return op if op in ("add", "mul", "and", "or", "min", "max") else None


# ---------------------------------------------------------------- codegen
def _params_scope(lam, k):
    scope = {}
    for j, p in enumerate(lam.params):
        if p != "_":
            scope[p] = f"A[{j}]" if j < k else f"B[{j - k}]"
    return scope


def _op_function(lam, k):
    """The operator as `V op(const V&, const V&)` (no captures: the
    associative forms only name their parameters and constants), modular,
    for the tree combines; and `V op_ck(const V&, const V&, int& ovf_)`, the
    same with checked int64 arithmetic, for the down pass's per-element
    left-fold steps: there the accumulator is the exact wrapped prefix, so a
    step that leaves int64 is exactly a result the reference would hold as a
    big int (oracle.py:288-292) -- a combine of two partial aggregates may
    overflow harmlessly and is never checked."""
    out = []
    for name, mode in (("op", "wrap"), ("op_ck", "flag")):
        g = _Gen({}, lambda node: 0)
        g.ovf = mode
        g.depth = 1
        res = g.tuple_expr(lam.body, _params_scope(lam, k), k)
        _ints_only(g, res)
        extra = ", int& ovf_" if mode == "flag" else ""
        lines = [f"__device__ __forceinline__ V {name}(const V& A_, const V& B_{extra}) {{",
                 "  const long long* A = A_.c; const long long* B = B_.c; (void)A; (void)B;"]
        lines += g.body
        lines += ["  V R;"] + [f"  R.c[{j}] = {r};" for j, r in enumerate(res)] + ["  return R;", "}"]
        out.append("\n".join(lines))
    return "\n".join(out)


_VHELP = r"""
struct V { long long c[K]; };
__device__ __forceinline__ V vzero() { V v; for (int j = 0; j < K; ++j) v.c[j] = 0; return v; }
__device__ __forceinline__ V vshfl_up(const V& v, int d) {
  V r; for (int j = 0; j < K; ++j) r.c[j] = __shfl_up_sync(0xffffffffu, v.c[j], d); return r;
}
#define TILE (256 * IPT)
#define PADI(j) ((j) + ((j) >> 5))
"""


def _par_scan_source(lam, k, in_types):
    ipt = max(1, 8 // k)
    ins = ", ".join(f"const {t}* __restrict__ in{j}" for j, t in enumerate(in_types))
    outs = ", ".join(f"long long* __restrict__ out{j}" for j in range(k))
    nes = ", ".join(f"long long ne{j}" for j in range(k))
    load = "\n".join(f"    sm[{j}][PADI(q)] = (long long)in{j}[base + q];" for j in range(k))
    item = lambda idx: "V b_; " + " ".join(f"b_.c[{j}] = sm[{j}][PADI({idx})];" for j in range(k))  # noqa: E731
    tile_fold = f"""
  __shared__ long long sm[K][TILE + TILE / 32];
  __shared__ V wv[8];
  const long long base = (long long)blockIdx.x * TILE;
  const int cnt = (int)min((long long)TILE, n - base);
  for (int q = threadIdx.x; q < cnt; q += 256) {{
{load}
  }}
  __syncthreads();
  const int f0 = threadIdx.x * IPT;
  const int mine = max(0, min(IPT, cnt - f0));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V acc = vzero();
  if (mine > 0) {{
    {item("f0")} acc = b_;
    for (int q = 1; q < mine; ++q) {{ {item("f0 + q")} acc = op(acc, b_); }}
  }}
  for (int d = 1; d < 32; d <<= 1) {{
    const V o = vshfl_up(acc, d);
    if (lane >= d && mine > 0) acc = op(o, acc);
  }}
  const V ex = vshfl_up(acc, 1);
  if (mine > 0 && (lane == 31 || f0 + IPT >= cnt)) wv[w] = acc;
  const int nw = (cnt + 32 * IPT - 1) / (32 * IPT);
  __syncthreads();
"""
    stores = "\n".join(f"    out{j}[base + q] = sm[{j}][PADI(q)];" for j in range(k))
    return (_PRELUDE + f"#define K {k}\n#define IPT {ipt}\n" + _VHELP + _op_function(lam, k) + f"""
extern "C" __global__ void __launch_bounds__(256) ixg_scan_red({ins}, long long n, long long* __restrict__ agg) {{
{tile_fold}
  if (threadIdx.x == 0) {{
    V t = wv[0];
    for (int q = 1; q < nw; ++q) t = op(t, wv[q]);
    for (int j = 0; j < K; ++j) agg[blockIdx.x * (long long)K + j] = t.c[j];
  }}
}}

extern "C" __global__ void __launch_bounds__(1024) ixg_scan_top(const long long* __restrict__ agg, long long T,
    {nes}, long long* __restrict__ carry) {{
  __shared__ V wv[32];
  const long long per = (T + 1023) / 1024;
  const long long lo = threadIdx.x * per, hi = min(T, lo + per);
  const bool has = lo < hi;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  V acc = vzero();
  if (has) {{
    for (int j = 0; j < K; ++j) acc.c[j] = agg[lo * K + j];
    for (long long t = lo + 1; t < hi; ++t) {{
      V b_; for (int j = 0; j < K; ++j) b_.c[j] = agg[t * K + j];
      acc = op(acc, b_);
    }}
  }}
  for (int d = 1; d < 32; d <<= 1) {{
    const V o = vshfl_up(acc, d);
    if (lane >= d && has) acc = op(o, acc);
  }}
  const V ex = vshfl_up(acc, 1);
  const bool next_has = (long long)(threadIdx.x + 1) * per < T;
  if (has && (lane == 31 || !next_has)) wv[w] = acc;
  const int nw = (int)min(32LL, (((T + per - 1) / per) + 31) / 32);
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 1; q < nw; ++q) wv[q] = op(wv[q - 1], wv[q]);
  __syncthreads();
  if (has) {{
    V run; {" ".join(f"run.c[{j}] = ne{j};" for j in range(k))}
    if (w > 0) run = op(run, wv[w - 1]);
    if (lane > 0) run = op(run, ex);
    for (long long t = lo; t < hi; ++t) {{
      for (int j = 0; j < K; ++j) carry[t * K + j] = run.c[j];
      V b_; for (int j = 0; j < K; ++j) b_.c[j] = agg[t * K + j];
      run = op(run, b_);
    }}
  }}
}}

extern "C" __global__ void __launch_bounds__(256) ixg_scan_down({ins}, {outs}, long long n,
    const long long* __restrict__ carry, ixg_status* st) {{
{tile_fold}
  if (threadIdx.x == 0)
    for (int q = 1; q < nw; ++q) wv[q] = op(wv[q - 1], wv[q]);
  __syncthreads();
  if (mine > 0) {{
    V run; for (int j = 0; j < K; ++j) run.c[j] = carry[blockIdx.x * (long long)K + j];
    if (w > 0) run = op(run, wv[w - 1]);
    if (lane > 0) run = op(run, ex);
    int ovf_ = 0, seen = 0;
    for (int q = 0; q < mine; ++q) {{
      {item("f0 + q")}
      run = op_ck(run, b_, ovf_);  // the left fold's step on the exact prefix
      if (ovf_ && !seen) {{ fail_ovf(st, 0, base + f0 + q); seen = 1; }}
      for (int j = 0; j < K; ++j) sm[j][PADI(f0 + q)] = run.c[j];
    }}
  }}
  __syncthreads();
  for (int q = threadIdx.x; q < cnt; q += 256) {{
{stores}
  }}
}}
"""), ipt


_SEQ_TILE = 512
_CT2 = {"f": "double", "i": "long long"}


def fold_types(lam, k: int, in_f: list, ne_f: list, env=None) -> list:
    """'i' | 'f' per accumulator of an in-order fold: a float neutral or
    element makes it a double, so does an operator that turns it into one
    (Python's int -> float promotion, fixed point over the parameters)."""
    g = _Gen(env or {}, lambda node: 0)
    tys = ["f" if (in_f[j] or ne_f[j]) else "i" for j in range(k)]
    for _ in range(k + 2):
        tenv = {}
        for j, p in enumerate(lam.params):
            tenv[p] = tys[j] if j < k else ("f" if in_f[j - k] else "i")
        r = g.infer(lam.body, tenv)
        rs = r if isinstance(r, list) else [r]
        new = ["f" if "f" in (a, b) else "i" for a, b in zip(tys, rs)]
        if new == tys:
            break
        tys = new
    return tys


def _seq_scan_source(lam, k, in_types, env, site_bits, acc_tys=None):
    """The exact in-order fold (oracle.py:288-292) on one thread over
    shared-memory-staged tiles; accumulators typed int64 or double."""
    acc_tys = acc_tys or ["i"] * k
    g = _Gen(env, site_bits)
    g.depth = 4
    g.on_fail = "failed = 1; goto done;"
    scope = {}
    for j, p in enumerate(lam.params):
        if p != "_":
            scope[p] = f"acc{j}" if j < k else f"el{j - k}"
    for j in range(k):
        if acc_tys[j] == "f":
            g.fty.add(f"acc{j}")
        if in_types[j] == "double":
            g.fty.add(f"el{j}")
    res = g.tuple_expr(lam.body, scope, k)
    ein = ["double" if t == "double" else "long long" for t in in_types]
    ins = [f"const {t}* __restrict__ in{j}" for j, t in enumerate(in_types)]
    params = ins + [f"const {_ctype(t)}* __restrict__ a{j}, long long len{j}" for j, t in enumerate(g.spec.arrays)]
    params += [f"{_CT2[acc_tys[j]]}* __restrict__ out{j}" for j in range(k)]
    params += ["long long n", "int stmt", "ixg_status* st"] + [f"{_CT2[acc_tys[j]]} ne{j}" for j in range(k)]
    params += [_scalar_param(j, v) for j, v in enumerate(g.spec.scalars)]
    params += [f"int pk{j}, long long pt{j}, u64 ps{j}" for j in range(len(g.spec.preds))]
    params += ["unsigned long long* gbud"]
    decl = "\n".join(f"  __shared__ {ein[j]} si{j}[{_SEQ_TILE}];\n  __shared__ {_CT2[acc_tys[j]]} so{j}[{_SEQ_TILE}];"
                     for j in range(k))
    load = "\n".join(f"      si{j}[q] = ({ein[j]})in{j}[base + q];" for j in range(k))
    els = "\n".join(f"        const {ein[j]} el{j} = si{j}[q];" for j in range(k))
    # results are staged in temporaries before any acc is overwritten
    upd_tmp = "\n".join(f"        const {_CT2[acc_tys[j]]} r{j} = {g.conv(r, acc_tys[j])};" for j, r in enumerate(res))
    upd = "\n".join(f"        acc{j} = r{j};\n        so{j}[q] = r{j};" for j in range(k))
    store = "\n".join(f"      out{j}[base + q] = so{j}[q];" for j in range(k))
    src = _PRELUDE + f"""
extern "C" __global__ void __launch_bounds__(256) ixg_scan_seq({", ".join(params)}) {{
{decl}
  __shared__ int failed;
  {" ".join(f"{_CT2[acc_tys[j]]} acc{j} = ne{j};" for j in range(k))}
  if (threadIdx.x == 0) failed = 0;
  for (long long base = 0; base < n; base += {_SEQ_TILE}) {{
    const int cnt = (int)min((long long){_SEQ_TILE}, n - base);
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {{
{load}
    }}
    __syncthreads();
    if (threadIdx.x == 0) {{
      for (int q = 0; q < cnt; ++q) {{
        const long long i = base + q;
{els}
{chr(10).join(g.body)}
{upd_tmp}
{upd}
      }}
      done:;
    }}
    __syncthreads();
    if (failed) return;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {{
{store}
    }}
    __syncthreads();
  }}
}}
"""
    return src, g.spec


def _hist_seq_source(lam, v_type, env, site_bits, acc_ty="i"):
    """hist in index order (oracle.py:313-315) on one thread; the
    destination is filled with ne by the kernel itself."""
    g = _Gen(env, site_bits)
    g.depth = 4
    g.on_fail = "failed = 1; goto done;"
    a, b = lam.params
    scope = {}
    if a != "_":
        scope[a] = "cur"
    if b != "_":
        scope[b] = "v"
    if acc_ty == "f":
        g.fty.add("cur")
    vf = v_type == "double"
    if vf:
        g.fty.add("v")
    res = g.expr(lam.body, scope)
    ct = _CT2[acc_ty]
    vt = "double" if vf else "long long"
    params = ["const long long* __restrict__ is", f"const {v_type}* __restrict__ vs"]
    params += [f"const {_ctype(t)}* __restrict__ a{j}, long long len{j}" for j, t in enumerate(g.spec.arrays)]
    params += [f"{ct}* __restrict__ dst", "long long dlen", "long long m", "int stmt", "ixg_status* st", f"{ct} ne"]
    params += [_scalar_param(j, v) for j, v in enumerate(g.spec.scalars)]
    params += [f"int pk{j}, long long pt{j}, u64 ps{j}" for j in range(len(g.spec.preds))]
    params += ["unsigned long long* gbud"]
    src = _PRELUDE + f"""
extern "C" __global__ void __launch_bounds__(256) ixg_hist_seq({", ".join(params)}) {{
  __shared__ long long si[{_SEQ_TILE}];
  __shared__ {vt} sv[{_SEQ_TILE}];
  __shared__ int failed;
  if (threadIdx.x == 0) failed = 0;
  for (long long q = threadIdx.x; q < dlen; q += blockDim.x) dst[q] = ne;
  __syncthreads();
  for (long long base = 0; base < m; base += {_SEQ_TILE}) {{
    const int cnt = (int)min((long long){_SEQ_TILE}, m - base);
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {{
      si[q] = is[base + q];
      sv[q] = ({vt})vs[base + q];
    }}
    __syncthreads();
    if (threadIdx.x == 0) {{
      for (int q = 0; q < cnt; ++q) {{
        const long long i = base + q;
        const long long bin = si[q];
        if ((unsigned long long)bin >= (unsigned long long)dlen) continue;
        const {ct} cur = dst[bin];
        const {vt} v = sv[q];
        (void)cur; (void)v;
{chr(10).join(g.body)}
        dst[bin] = {g.conv(res, acc_ty)};
      }}
      done:;
    }}
    __syncthreads();
    if (failed) return;
  }}
}}
"""
    return src, g.spec


def _hist_cas_source(lam, v_type):
    """Commutative + associative hist operator as a CAS loop per element.
    Its int64 arithmetic is checked per update: an update that leaves int64
    in THIS order is reported, and the caller re-runs the exact in-order
    fold (the reference's order decides, oracle.py:313-315)."""
    a, b = lam.params
    g = _Gen({}, lambda node: 0)
    g.ovf = "flag"
    g.depth = 3
    res = g.expr(lam.body, {a: "cur", b: "v"})
    _ints_only(g, [res])
    return _PRELUDE + f"""
extern "C" __global__ void __launch_bounds__(256) ixg_hist_cas(const long long* __restrict__ is,
    const {v_type}* __restrict__ vs, long long* __restrict__ dst, long long dlen, long long m, ixg_status* st) {{
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {{
    const long long bin = is[i];
    if ((unsigned long long)bin >= (unsigned long long)dlen) continue;
    const long long v = (long long)vs[i];
    unsigned long long* p = (unsigned long long*)(dst + bin);
    unsigned long long old = *(volatile unsigned long long*)p, seen;
    int ovf_;
    do {{
      seen = old;
      ovf_ = 0;
      const long long cur = (long long)seen;
{chr(10).join(g.body)}
      old = atomicCAS(p, seen, (unsigned long long)({res}));
    }} while (old != seen);
    if (ovf_) fail_ovf(st, 0, i);
  }}
}}
"""


# ---------------------------------------------------------------- launching
def _kernel(src, names):
    key = hashlib.sha1(src.encode()).hexdigest()
    kern = _CACHE.get(key)
    if kern is None:
        kern = _CACHE[key] = _Kernel(src, names)
    return kern


def _launch(kern, name, grid, block, vals, dev):
    from cuda.bindings import driver

    argv = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
    (err,) = driver.cuLaunchKernel(kern.fns[name], grid, 1, 1, block, 1, 1, 0,
                                   torch.cuda.current_stream(dev).cuda_stream, ctypes.addressof(argv), 0)
    _ok(err, "cuLaunchKernel")
    LAUNCHES[0] += 1


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def _captures(spec):
    vals = []
    for t in spec.arrays:
        t = t.contiguous()
        vals += [_p(t), ctypes.c_longlong(t.numel())]
    return vals


def _tail(spec):
    return scalar_args(spec)


def _ints_only(g, res):
    """The fold kernels carry int64 state: float operators are not lowered."""
    if any(g.is_f(r) for r in res):
        raise Unsupported("floating-point scan / hist operator")


def _elem(t: torch.Tensor) -> torch.Tensor:
    return t.view(torch.uint8) if t.dtype == torch.bool else t.contiguous()


def scan(lam, nes: list, arrays: list, env: dict, site_bits, status, device=None, force_seq=False):
    """scan lam nes... arrays... -> (list of k tensors (int64, or float64 for
    a float accumulator), sites, parallel?).  Output length = len(arrays[0])
    (oracle.py:286); the caller checks that the other operands are at least
    as long.  Float folds are never re-associated: the in-order kernel."""
    k = len(nes)
    dev = device or arrays[0].device
    n = arrays[0].numel()
    ins = [_elem(a)[:n] for a in arrays]
    in_types = [_ctype(t) for t in ins]
    acc_tys = fold_types(lam, k, [t.is_floating_point() for t in ins], [isinstance(v, float) for v in nes], env)
    outs = [torch.empty(n, dtype=torch.float64 if ty == "f" else torch.int64, device=dev) for ty in acc_tys]
    nev = [ctypes.c_double(float(v)) if ty == "f" else ctypes.c_longlong(int(v)) for v, ty in zip(nes, acc_tys)]
    par = not force_seq and "f" not in acc_tys and classify_scan(lam, k)
    if par:
        src, ipt = _par_scan_source(lam, k, in_types)
        if n == 0:
            return outs, [], True
        kern = _kernel(src, ("ixg_scan_red", "ixg_scan_top", "ixg_scan_down"))
        tiles = (n + 256 * ipt - 1) // (256 * ipt)
        agg = torch.empty(tiles * k, dtype=torch.int64, device=dev)
        carry = torch.empty(tiles * k, dtype=torch.int64, device=dev)
        _launch(kern, "ixg_scan_red", tiles, 256, [_p(t) for t in ins] + [ctypes.c_longlong(n), _p(agg)], dev)
        _launch(kern, "ixg_scan_top", 1, 1024, [_p(agg), ctypes.c_longlong(tiles)] + nev + [_p(carry)], dev)
        _launch(kern, "ixg_scan_down", tiles, 256,
                [_p(t) for t in ins] + [_p(o) for o in outs] + [ctypes.c_longlong(n), _p(carry), _p(status.t)], dev)
        return outs, [], True
    src, spec = _seq_scan_source(lam, k, in_types, env, site_bits, acc_tys)
    if n == 0:
        return outs, spec.sites, False
    kern = _kernel(src, ("ixg_scan_seq",))
    vals = [_p(t) for t in ins] + _captures(spec) + [_p(o) for o in outs]
    vals += [ctypes.c_longlong(n), ctypes.c_int(0), _p(status.t)] + nev + _tail(spec) + budget_arg(spec, dev)
    _launch(kern, "ixg_scan_seq", 1, 256, vals, dev)
    return outs, spec.sites, False


def hist(lam, ne, dlen: int, is_: torch.Tensor, vs: torch.Tensor, env: dict, site_bits, status,
         force_seq=False):
    """hist lam ne dlen is vs -> (tensor [max(dlen,0)] int64 or float64,
    sites, kind) with kind 'cas' | 'seq' (the named fast paths are the
    caller's).  Float accumulations keep the index order (no CAS)."""
    from . import ops

    dev = is_.device
    m = min(is_.numel(), vs.numel())
    iss, vss = is_.contiguous()[:m], _elem(vs)[:m]
    v_type = _ctype(vss)
    acc_ty = fold_types(lam, 1, [vss.is_floating_point()], [isinstance(ne, float)], env)[0]
    nd = max(int(dlen), 0)
    if not force_seq and acc_ty == "i" and classify_hist(lam) is not None:
        dst = ops.fill(nd, int(ne), torch.int64, dev)
        src = _hist_cas_source(lam, v_type)
        if m and nd:
            kern = _kernel(src, ("ixg_hist_cas",))
            sms = torch.cuda.get_device_properties(dev).multi_processor_count
            grid = max(1, min((m + 255) // 256, sms * 8))
            st = ops.Status(dev)
            _launch(kern, "ixg_hist_cas", grid, 256,
                    [_p(iss), _p(vss), _p(dst), ctypes.c_longlong(nd), ctypes.c_longlong(m), _p(st.t)], dev)
            if not st.read().ok:  # an update left int64 in the atomic order: decide in the reference's order
                return hist(lam, ne, dlen, is_, vs, env, site_bits, status, force_seq=True)
        return dst, [], "cas"
    dst = torch.empty(nd, dtype=torch.float64 if acc_ty == "f" else torch.int64, device=dev)
    src, spec = _hist_seq_source(lam, v_type, env, site_bits, acc_ty)
    if nd:
        kern = _kernel(src, ("ixg_hist_seq",))
        nev = ctypes.c_double(float(ne)) if acc_ty == "f" else ctypes.c_longlong(int(ne))
        vals = [_p(iss), _p(vss)] + _captures(spec)
        vals += [_p(dst), ctypes.c_longlong(nd), ctypes.c_longlong(m), ctypes.c_int(0), _p(status.t), nev]
        _launch(kern, "ixg_hist_seq", 1, 256, vals + _tail(spec) + budget_arg(spec, dev), dev)
    return dst, spec.sites, "seq"
