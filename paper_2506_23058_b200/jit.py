"""Compile a lambda of the reference language straight to a CUDA kernel
(lambda -> CUDA via NVRTC) for the generic `map`.

The register VM (vm.py, csrc/k_vm.cuh) interprets a lambda per element from a
local-memory register file; here the same lambda becomes straight-line C++
with the same evaluation order and semantics -- jumps become `if`, `&&` /
`||` short-circuit (oracle.py:216-219), an IndexE in an untaken branch is
never evaluated, a CHECKED index site records the first failure exactly like
the VM (status [stmt:8][elem:48][site:8], the element's output skipped) --
compiled once per distinct (lambda, element types, checked sites) for sm_100a
with NVRTC and cached.  Captured scalars and predicate descriptors are
kernel parameters, so a cached kernel serves every call of its lambda.

`map_jit` has the signature of `ops.map_vm` plus the compile step; the
executor uses it unless IXG_JIT=0 (then the VM).
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import struct
from dataclasses import dataclass, field

import torch

from . import _lib as L
from . import ir
from .pred import Pred
from .vm import Unsupported

_CMP = {"==": "==", "!=": "!=", "<": "<", "<=": "<=", ">": ">", ">=": ">="}
_ARITH = {"+": "+", "-": "-", "*": "*"}
# Python float arithmetic is IEEE double with no contraction: round-to-nearest
# intrinsics keep NVRTC from fusing a*b+c into an FMA
_FARITH = {"+": "__dadd_rn", "-": "__dsub_rn", "*": "__dmul_rn"}
_CT = {torch.int64: "long long", torch.int32: "int", torch.uint8: "unsigned char", torch.bool: "unsigned char",
       torch.float64: "double"}
BUDGET_SITE = 255  # status site of a loop that ran past the step budget

_PRELUDE = r"""
typedef unsigned long long u64;
struct ixg_status { u64 first; unsigned int codes; unsigned int flags; };
__device__ __forceinline__ u64 mix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
// pred_eval of csrc/common.cuh (oracle.py:327-329 semantics)
__device__ __forceinline__ long long pred(int kind, long long thr, u64 seed, long long x) {
  switch (kind) {
    case 0: return x < thr;
    case 1: return x > thr;
    case 2: return x <= thr;
    case 3: return x >= thr;
    case 4: return x == thr;
    case 5: return x != thr;
    case 6: return (mix64((u64)x ^ seed) >> 63) != 0;
    case 7: return 1;
    default: return 0;
  }
}
__device__ __forceinline__ void fail_oob(ixg_status* st, int stmt, long long elem, int site) {
  const u64 key = ((u64)(stmt & 0xff) << 56) | (((u64)elem & 0xffffffffffffULL) << 8) | (u64)(site & 0xff);
  atomicMin(&st->first, key);
  atomicOr(&st->codes, 1u << 1);
}
// int64 arithmetic of the language, checked: the reference's ints are
// unbounded (oracle.py:214-240), a value leaving int64 is IXG_OVERFLOW at
// site IXG_OVF_SITE (254) instead of a wrapped result
__device__ __forceinline__ void fail_ovf(ixg_status* st, int stmt, long long elem) {
  const u64 key = ((u64)(stmt & 0xff) << 56) | (((u64)elem & 0xffffffffffffULL) << 8) | 254ULL;
  atomicMin(&st->first, key);
  atomicOr(&st->codes, 1u << 6);
}
__device__ __forceinline__ int ck_add(long long a, long long b, long long* r) {
  const long long s = (long long)((u64)a + (u64)b); *r = s; return ((a ^ s) & (b ^ s)) < 0;
}
__device__ __forceinline__ int ck_sub(long long a, long long b, long long* r) {
  const long long s = (long long)((u64)a - (u64)b); *r = s; return ((a ^ b) & (a ^ s)) < 0;
}
__device__ __forceinline__ int ck_mul(long long a, long long b, long long* r) {
  const long long lo = (long long)((u64)a * (u64)b); *r = lo; return __mul64hi(a, b) != (lo >> 63);
}
"""
_CK = {"+": "ck_add", "-": "ck_sub", "*": "ck_mul"}
OVF_SITE = 254  # status site of an int64 overflow (include/ixgpu.h IXG_OVF_SITE)


@dataclass
class _Spec:
    inputs: list = field(default_factory=list)   # per-element tensors
    arrays: list = field(default_factory=list)   # gather sources (tensors)
    scalars: list = field(default_factory=list)  # captured ints / floats
    preds: list = field(default_factory=list)    # Pred
    sites: list = field(default_factory=list)    # IndexE nodes in site order
    out_types: list = field(default_factory=list)  # 'i' | 'f' per output
    need_budget: bool = False  # a loop: the kernel's gbud counter bounds all its iterations


def _size_binds(f, slot_len):
    """Size parameters of an inlined function from its array arguments'
    lengths (oracle.py:137-161: [n] := len, [n+1] := len - 1)."""
    out = {}
    for p in f.params:
        t = p.type
        if ir.kind(t) != "TArray" or p.name not in slot_len:
            continue
        ln = slot_len[p.name]
        sz = t.size
        if sz is None:
            continue
        if ir.kind(sz) == "VarE":
            out.setdefault(sz.name, ln)
        elif (ir.kind(sz) == "BinOp" and sz.op == "+" and ir.kind(sz.lhs) == "VarE" and ir.kind(sz.rhs) == "Const"
              and not isinstance(sz.rhs.value, float)):
            out.setdefault(sz.lhs.name, f"({ln} - {int(sz.rhs.value)}LL)")
    return out


class _Gen:
    """Straight-line C++ for one lambda (or an inlined scalar function).
    Values are `long long` (ints, bools as 0/1) or `double` (Python floats,
    f32/f64 in the language); the type of every expression is inferred
    before it is emitted, mixed arithmetic promotes to double like Python."""

    def __init__(self, env: dict, site_bits, funs=None, bits_for=None, loop_cap: int = 1 << 31):
        self.env, self.site_bits = env, site_bits
        self.funs = funs or {}
        self.bits_for = bits_for
        self.loop_cap = int(loop_cap)
        self.spec = _Spec()
        self.body: list = []
        self.ntmp = 0
        self.depth = 2
        self._arr_slot: dict = {}
        self.fty: set = set()  # C expressions of type double
        self.inlining = 0
        # what a failed CHECKED index site does after recording the failure
        self.on_fail = "goto next;"
        # int64 + - *: "fail" = checked, an overflow fails the element like an
        # index site (needs st / stmt / i in scope); "flag" = checked, ORs into
        # an `ovf_` variable of the enclosing code; "wrap" = modular
        self.ovf = "fail"

    def line(self, s: str):
        self.body.append("  " * self.depth + s)

    def tmp(self) -> str:
        t = f"t{self.ntmp}"
        self.ntmp += 1
        return t

    def is_f(self, s: str) -> bool:
        return s in self.fty

    def as_f(self, s: str) -> str:
        return s if self.is_f(s) else f"(double)({s})"

    def conv(self, s: str, ty: str) -> str:
        return self.as_f(s) if ty == "f" else (f"(long long)({s})" if self.is_f(s) else s)

    def new(self, value: str, ty: str = "i") -> str:
        t = self.tmp()
        self.line(f"const {'double' if ty == 'f' else 'long long'} {t} = {value};")
        if ty == "f":
            self.fty.add(t)
        return t

    def mut(self, ty: str) -> str:
        t = self.tmp()
        self.line(f"{'double' if ty == 'f' else 'long long'} {t};")
        if ty == "f":
            self.fty.add(t)
        return t

    def array_slot(self, t) -> int:
        k = id(t)
        if k not in self._arr_slot:
            self._arr_slot[k] = len(self.spec.arrays)
            self.spec.arrays.append(t)
        return self._arr_slot[k]

    def scalar(self, v) -> str:
        self.spec.scalars.append(v)
        s = f"s{len(self.spec.scalars) - 1}"
        if isinstance(v, float):
            self.fty.add(s)
        return s

    def fconst(self, v: float) -> str:
        bits = struct.unpack("<q", struct.pack("<d", float(v)))[0]
        t = f"__longlong_as_double({bits}LL)"
        self.fty.add(t)
        return t

    # ------------------------------------------------------------ inference
    def _tenv(self, scope: dict) -> dict:
        return {n: ([("f" if self.is_f(x) else "i") for x in c] if isinstance(c, list) else
                    ("f" if self.is_f(c) else "i")) for n, c in scope.items()}

    def infer(self, e, tenv: dict, env=None):
        """'i' | 'f' of a scalar expression, a list of those for a tuple."""
        env = self.env if env is None else env
        k = ir.kind(e)
        if k == "Const":
            return "f" if isinstance(e.value, float) else "i"
        if k == "VarE":
            if e.name in tenv:
                return tenv[e.name]
            b = env.get(e.name)
            return "f" if b is not None and b[0] == "scalar" and isinstance(b[1], float) else "i"
        if k == "BinOp":
            if e.op in _ARITH:
                a, b = self.infer(e.lhs, tenv, env), self.infer(e.rhs, tenv, env)
                return "f" if "f" in (a, b) else "i"
            return "i"
        if k == "NotE":
            return "i"
        if k == "If":
            a, b = self.infer(e.then, tenv, env), self.infer(e.els, tenv, env)
            if isinstance(a, list):
                return ["f" if "f" in (x, y) else "i" for x, y in zip(a, b)]
            return "f" if "f" in (a, b) else "i"
        if k == "Let":
            r = self.infer(e.rhs, tenv, env)
            inner = dict(tenv)
            if len(e.names) == 1:
                inner[e.names[0]] = r
            else:
                for n, t in zip(e.names, r if isinstance(r, list) else [r] * len(e.names)):
                    inner[n] = t
            return self.infer(e.body, inner, env)
        if k == "TupleE":
            return [self.infer(x, tenv, env) for x in e.items]
        if k == "IndexE":
            b = env.get(e.arr.name) if ir.kind(e.arr) == "VarE" else None
            return "f" if b is not None and b[0] == "array" and b[1].is_floating_point() else "i"
        if k == "Loop":
            return self._loop_types(e, tenv, env)
        if k == "App" and ir.kind(e.fun) == "VarE" and e.fun.name in self.funs:
            f = self.funs[e.fun.name]
            if self.inlining > 16:
                raise Unsupported("recursive function")
            cenv, ct = {}, {}
            for p, a in zip(f.params, e.args):
                pk = ir.kind(p.type)
                if pk in ("TArray", "TFun"):
                    if ir.kind(a) == "VarE" and a.name in env:
                        cenv[p.name] = env[a.name]
                else:
                    ct[p.name] = self.infer(a, tenv, env)
            for s in f.sizes:
                ct.setdefault(s, "i")
            self.inlining += 1
            try:
                return self.infer(f.body, ct, cenv)
            finally:
                self.inlining -= 1
        return "i"

    def _loop_types(self, e, tenv, env):
        pts = [self.infer(x, tenv, env) for x in e.inits]
        for _ in range(len(pts) + 2):
            inner = dict(tenv)
            for p, t in zip(e.params, pts):
                inner[p.name] = t
            if e.kind == "for" and e.counter:
                inner[e.counter] = "i"
            r = self.infer(e.body, inner, env)
            rs = r if isinstance(r, list) else [r]
            new = ["f" if "f" in (a, b) else "i" for a, b in zip(pts, rs)]
            if new == pts:
                break
            pts = new
        return pts if len(pts) > 1 else pts[0]

    # -------------------------------------------------------------- codegen
    def expr(self, e, scope: dict) -> str:
        k = ir.kind(e)
        if k == "Const":
            if isinstance(e.value, float):
                return self.fconst(e.value)
            return f"{int(e.value)}LL"
        if k == "VarE":
            if e.name in scope:
                if isinstance(scope[e.name], list):
                    raise Unsupported(f"tuple {e.name} in a scalar position")
                return scope[e.name]
            b = self.env.get(e.name)
            if b is None:
                raise Unsupported(f"free name {e.name}")
            if b[0] == "scalar":
                return self.scalar(b[1])
            raise Unsupported(f"{e.name} used as a scalar")
        if k == "BinOp":
            if e.op in ("&&", "||"):
                r = self.mut("i")
                a = self.expr(e.lhs, scope)
                self.line(f"{r} = ({a}) != 0;")
                self.line(f"if ({'' if e.op == '&&' else '!'}{r}) {{")
                self.depth += 1
                b = self.expr(e.rhs, scope)
                self.line(f"{r} = ({b}) != 0;")
                self.depth -= 1
                self.line("}")
                return r
            a = self.expr(e.lhs, scope)
            b = self.expr(e.rhs, scope)
            fl = self.is_f(a) or self.is_f(b)
            if e.op in _ARITH:
                if fl:
                    return self.new(f"{_FARITH[e.op]}({self.as_f(a)}, {self.as_f(b)})", "f")
                if self.ovf == "wrap":
                    return self.new(f"(long long)((u64)({a}) {_ARITH[e.op]} (u64)({b}))")
                r = self.mut("i")
                ck = f"{_CK[e.op]}({a}, {b}, &{r})"
                if self.ovf == "flag":
                    self.line(f"ovf_ |= {ck};")
                else:
                    self.line(f"if ({ck}) {{ fail_ovf(st, stmt, i); {self.on_fail} }}")
                return r
            if e.op in _CMP:
                if fl:
                    return self.new(f"(long long)(({self.as_f(a)}) {_CMP[e.op]} ({self.as_f(b)}))")
                return self.new(f"(long long)(({a}) {_CMP[e.op]} ({b}))")
            raise Unsupported(f"operator {e.op}")
        if k == "NotE":
            a = self.expr(e.arg, scope)
            return self.new(f"(long long)(({a}) == 0)")
        if k == "If":
            ty = self.infer(e, self._tenv(scope))
            if isinstance(ty, list):
                raise Unsupported("tuple-valued if in a scalar position")
            c = self.expr(e.cond, scope)
            r = self.mut(ty)
            self.line(f"if (({c}) != 0) {{")
            self.depth += 1
            t = self.expr(e.then, scope)
            self.line(f"{r} = {self.conv(t, ty)};")
            self.depth -= 1
            self.line("} else {")
            self.depth += 1
            f = self.expr(e.els, scope)
            self.line(f"{r} = {self.conv(f, ty)};")
            self.depth -= 1
            self.line("}")
            return r
        if k == "Let":
            inner = dict(scope)
            if len(e.names) != 1:
                vs = self.tuple_expr(e.rhs, scope, len(e.names))
                for n, v in zip(e.names, vs):
                    if n != "_":
                        inner[n] = v
                return self.expr(e.body, inner)
            r = self.expr(e.rhs, scope)
            v = self.new(r, "f" if self.is_f(r) else "i")
            if e.names[0] != "_":
                inner[e.names[0]] = v
            return self.expr(e.body, inner)
        if k == "IndexE":
            if ir.kind(e.arr) != "VarE" or e.arr.name in scope:
                raise Unsupported("indexing a computed array")
            b = self.env.get(e.arr.name)
            if b is None or b[0] != "array":
                raise Unsupported(f"indexing non-array {e.arr.name}")
            ix = self.expr(e.idx, scope)
            if self.is_f(ix):
                raise Unsupported("float index")
            i = self.new(ix)
            slot = self.array_slot(b[1])
            site = len(self.spec.sites)
            self.spec.sites.append(e)
            if self.site_bits(e) & L.V_BOUNDS:
                self.line(f"if ((u64){i} >= (u64)len{slot}) {{ fail_oob(st, stmt, i, {site}); {self.on_fail} }}")
            if b[1].is_floating_point():
                return self.new(f"(double)a{slot}[{i}]", "f")
            return self.new(f"(long long)a{slot}[{i}]")
        if k == "Loop":
            r = self.loop(e, scope)
            if len(r) != 1:
                raise Unsupported("tuple-valued loop in a scalar position")
            return r[0]
        if k == "App" and ir.kind(e.fun) == "VarE":
            b = self.env.get(e.fun.name)
            if b is not None and b[0] == "pred" and len(e.args) == 1:
                a = self.expr(e.args[0], scope)
                p: Pred = b[1]
                if p not in self.spec.preds:
                    self.spec.preds.append(p)
                j = self.spec.preds.index(p)
                return self.new(f"pred(pk{j}, pt{j}, ps{j}, {self.conv(a, 'i')})")
            if e.fun.name == "length" and len(e.args) == 1 and ir.kind(e.args[0]) == "VarE":
                b = self.env.get(e.args[0].name)
                if b is not None and b[0] == "array":
                    return f"len{self.array_slot(b[1])}"
            if e.fun.name in self.funs:
                r = self.inline(e, scope, 1)
                return r[0]
        raise Unsupported(f"{k} inside a lambda: {ir.expr_str(e)}")

    def tuple_expr(self, e, scope: dict, k: int) -> list:
        """The k components of a tuple-valued body (a k-ary scan operator,
        oracle.py:286-290, a multi-parameter loop, a tuple-returning
        function), evaluated left to right like TupleE (oracle.py:199-200);
        Let and If may wrap the tuple."""
        kd = ir.kind(e)
        if kd == "VarE" and isinstance(scope.get(e.name), list):  # an element of an array of tuples
            if len(scope[e.name]) != k:
                raise Unsupported("tuple arity")
            return list(scope[e.name])
        if k == 1:
            return [self.expr(e, scope)]
        if kd == "TupleE":
            if len(e.items) != k:
                raise Unsupported("operator result arity")
            out = []
            for x in e.items:
                r = self.expr(x, scope)
                out.append(self.new(r, "f" if self.is_f(r) else "i"))
            return out
        if kd == "Let":
            inner = dict(scope)
            if len(e.names) != 1:
                vs = self.tuple_expr(e.rhs, scope, len(e.names))
                for n, v in zip(e.names, vs):
                    if n != "_":
                        inner[n] = v
                return self.tuple_expr(e.body, inner, k)
            r = self.expr(e.rhs, scope)
            v = self.new(r, "f" if self.is_f(r) else "i")
            if e.names[0] != "_":
                inner[e.names[0]] = v
            return self.tuple_expr(e.body, inner, k)
        if kd == "If":
            tys = self.infer(e, self._tenv(scope))
            if not isinstance(tys, list) or len(tys) != k:
                raise Unsupported("operator result arity")
            c = self.expr(e.cond, scope)
            rs = [self.mut(t) for t in tys]
            self.line(f"if (({c}) != 0) {{")
            for branch in (e.then, e.els):
                self.depth += 1
                vs = self.tuple_expr(branch, scope, k)
                for r, v, t in zip(rs, vs, tys):
                    self.line(f"{r} = {self.conv(v, t)};")
                self.depth -= 1
                self.line("} else {" if branch is e.then else "}")
            return rs
        if kd == "Loop":
            r = self.loop(e, scope)
            if len(r) != k:
                raise Unsupported("loop arity")
            return r
        if kd == "App" and ir.kind(e.fun) == "VarE" and e.fun.name in self.funs:
            return self.inline(e, scope, k)
        raise Unsupported(f"{kd} as a tuple-valued operator body")

    def loop(self, e, scope: dict) -> list:
        """`loop (ps) = (inits) for j < bound do body` / `while cond do body`
        (oracle.py:242-262): the bound is evaluated once, the parameters are
        rebound from the body's results after every iteration.  A loop that
        runs past the step budget records BUDGET_SITE (StepBudgetExceeded)."""
        inits = [self.expr(x, scope) for x in e.inits]
        pts = self._loop_types(e, self._tenv(scope), self.env)
        pts = pts if isinstance(pts, list) else [pts]
        lps = []
        for v, t in zip(inits, pts):
            lp = self.mut(t)
            self.line(f"{lp} = {self.conv(v, t)};")
            lps.append(lp)
        inner = dict(scope)
        for p, lp in zip(e.params, lps):
            inner[p.name] = lp
        it = self.mut("i")
        self.line(f"{it} = 0;")
        cap = self.scalar(self.loop_cap)
        self.spec.need_budget = True
        # the step budget bounds one loop instance AND, through the shared
        # counter (256 iterations at a time), all loops of the launch -- a
        # never-ending loop over many elements fails fast instead of running
        # budget x elements iterations
        guard = (f"if (++{it} > {cap} || (({it} & 255) == 0 && atomicAdd(gbud, 256ULL) + 256ULL > (u64){cap})) "
                 f"{{ fail_oob(st, stmt, i, {BUDGET_SITE}); {self.on_fail} }}")
        if e.kind == "for":
            bound = self.new(self.conv(self.expr(e.bound, scope), "i"))
            c = self.tmp()
            self.line(f"for (long long {c} = 0; {c} < {bound}; ++{c}) {{")
            if e.counter:
                inner[e.counter] = c
            self.depth += 1
            self.line(guard)
        else:
            self.line("for (;;) {")
            self.depth += 1
            cond = self.expr(e.cond, inner)
            self.line(f"if (!({cond})) break;")
            self.line(guard)
        rs = self.tuple_expr(e.body, inner, len(lps))
        staged = [self.new(self.conv(r, t), t) for r, t in zip(rs, pts)]
        for lp, r in zip(lps, staged):
            self.line(f"{lp} = {r};")
        self.depth -= 1
        self.line("}")
        return lps

    def inline(self, e, scope: dict, k: int) -> list:
        """A call of a program function inside a kernel: its body inlined
        with its scalar parameters bound to the evaluated arguments (left to
        right, oracle.py:325), array and predicate parameters to the
        caller's captured bindings and its size parameters to the arrays'
        lengths; its index sites carry its own verifier verdicts."""
        f = self.funs[e.fun.name]
        if len(e.args) != len(f.params):
            raise Unsupported("call arity")
        if self.inlining > 16:
            raise Unsupported("recursive function")
        cenv, cscope, lens = {}, {}, {}
        for p, a in zip(f.params, e.args):
            pk = ir.kind(p.type)
            if pk in ("TArray", "TFun"):
                if ir.kind(a) != "VarE" or a.name in scope or a.name not in self.env:
                    raise Unsupported("array argument must be a captured array")
                cenv[p.name] = self.env[a.name]
                if pk == "TArray":
                    lens[p.name] = f"len{self.array_slot(self.env[a.name][1])}"
            else:
                cscope[p.name] = self.expr(a, scope)
        cscope.update({s: v for s, v in _size_binds(f, lens).items() if s not in cscope})
        saved = (self.env, self.site_bits)
        self.env = cenv
        if self.bits_for is not None:
            self.site_bits = self.bits_for(f.name)
        self.inlining += 1
        try:
            return self.tuple_expr(f.body, cscope, k)
        finally:
            self.inlining -= 1
            self.env, self.site_bits = saved


class TupleCols:
    """An array of k-tuples (`map` with a tuple-valued lambda, oracle.py:280
    returns a list of tuples) held as k device columns."""

    def __init__(self, cols: list):
        self.cols = list(cols)

    def numel(self) -> int:
        return self.cols[0].numel() if self.cols else 0

    def __len__(self) -> int:
        return self.numel()


def tuple_arity(e, funs=None) -> int:
    """k of a tuple-valued expression (TupleE, through let / if / loops /
    calls of tuple-returning functions), 1 for a scalar."""
    k = ir.kind(e)
    if k == "TupleE":
        return len(e.items)
    if k == "Let":
        return tuple_arity(e.body, funs)
    if k == "If":
        return tuple_arity(e.then, funs)
    if k == "Loop":
        return len(e.params)
    if k == "App" and ir.kind(e.fun) == "VarE" and funs and e.fun.name in funs:
        rt = funs[e.fun.name].result_type
        return len(rt.items) if ir.kind(rt) == "TTuple" else 1
    return 1


def _ctype(t: torch.Tensor) -> str:
    if t.dtype not in _CT:
        raise Unsupported(f"element type {t.dtype}")
    return _CT[t.dtype]


def _scalar_param(j: int, v) -> str:
    return f"double s{j}" if isinstance(v, float) else f"long long s{j}"


def generate(lam, arrays: list, env: dict, site_bits=lambda node: L.V_BOUNDS, out_dtype=None, funs=None,
             bits_for=None, loop_cap: int = 1 << 31, k_out: int = 1):
    """-> (CUDA source, _Spec).  The source depends on the lambda, the
    element types and which index sites are checked -- not on the values of
    captured scalars or predicates (kernel parameters).  out_dtype None:
    int64, or float64 when the body is float-valued; k_out > 1 for a
    tuple-valued body (one output array per component)."""
    if len(lam.params) != len(arrays):
        raise Unsupported("lambda arity")
    g = _Gen(env, site_bits, funs, bits_for, loop_cap)
    flat = []  # per-element input columns (an array of tuples contributes one per component)
    scope = {}
    loads = []
    for p, a in zip(lam.params, arrays):
        cols = a.cols if isinstance(a, TupleCols) else [a]
        names = []
        for t in cols:
            j = len(flat)
            flat.append(t)
            _ctype(t)
            if t.is_floating_point():
                loads.append(f"    const double x{j} = in{j}[i];")
                g.fty.add(f"x{j}")
            else:
                loads.append(f"    const long long x{j} = (long long)in{j}[i];")
            names.append(f"x{j}")
        if p != "_":
            scope[p] = names if isinstance(a, TupleCols) else names[0]
    arrays = flat
    g.spec.inputs = list(flat)
    res = g.tuple_expr(lam.body, scope, k_out)
    tys = ["f" if g.is_f(r) else "i" for r in res]
    if out_dtype is not None and k_out == 1:
        tys = ["f" if out_dtype == torch.float64 else "i"]
    g.spec.out_types = tys
    ots = [out_dtype if (out_dtype is not None and k_out == 1) else (torch.float64 if t == "f" else torch.int64)
           for t in tys]
    params = [f"const {_ctype(t)}* __restrict__ in{j}" for j, t in enumerate(arrays)]
    params += [f"const {_ctype(t)}* __restrict__ a{j}, long long len{j}" for j, t in enumerate(g.spec.arrays)]
    params += [f"{_CT[o]}* __restrict__ out{j}" for j, o in enumerate(ots)]
    params += ["long long n", "int stmt", "ixg_status* st"]
    params += [_scalar_param(j, v) for j, v in enumerate(g.spec.scalars)]
    params += [f"int pk{j}, long long pt{j}, u64 ps{j}" for j in range(len(g.spec.preds))]
    params += ["unsigned long long* gbud"]
    stores = []
    for j, (r, o) in enumerate(zip(res, ots)):
        if o in (torch.uint8, torch.bool):
            stores.append(f"    out{j}[i] = ({_CT[o]})(({r}) != 0);")
        elif o == torch.float64:
            stores.append(f"    out{j}[i] = {g.as_f(r)};")
        else:
            stores.append(f"    out{j}[i] = ({_CT[o]})({g.conv(r, 'i')});")
    src = (_PRELUDE + 'extern "C" __global__ void __launch_bounds__(256) ixg_jit_map(' + ", ".join(params) + ") {\n"
           "  const long long stride = (long long)gridDim.x * blockDim.x;\n"
           "  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {\n"
           "   {\n" + "\n".join(loads) + "\n" + "\n".join(g.body) + "\n" + "\n".join(stores) + "\n   }\n"
           "  next:;\n  }\n}\n")
    g.spec.out_dtypes = ots
    return src, g.spec


class _Kernel:
    def __init__(self, src: str, names=("ixg_jit_map",)):
        from cuda.bindings import driver, nvrtc

        err, prog = nvrtc.nvrtcCreateProgram(src.encode(), b"ixg_jit_map.cu", 0, [], [])
        _ok(err, "nvrtcCreateProgram")
        opts = [b"--gpu-architecture=sm_100a", b"-std=c++17", b"-default-device"]
        (err,) = nvrtc.nvrtcCompileProgram(prog, len(opts), opts)
        if err != nvrtc.nvrtcResult.NVRTC_SUCCESS:
            _, size = nvrtc.nvrtcGetProgramLogSize(prog)
            log = b" " * size
            nvrtc.nvrtcGetProgramLog(prog, log)
            raise RuntimeError("NVRTC failed on a generated kernel:\n" + log.decode(errors="replace") + "\n" + src)
        err, size = nvrtc.nvrtcGetCUBINSize(prog)
        _ok(err, "nvrtcGetCUBINSize")
        cubin = b" " * size
        (err,) = nvrtc.nvrtcGetCUBIN(prog, cubin)
        _ok(err, "nvrtcGetCUBIN")
        nvrtc.nvrtcDestroyProgram(prog)
        (err,) = driver.cuInit(0)
        _ok(err, "cuInit")
        torch.cuda.synchronize()  # the runtime's primary context is current on this thread
        err, self.module = driver.cuModuleLoadData(cubin)
        _ok(err, "cuModuleLoadData")
        self.fns = {}
        for name in names:
            err, self.fns[name] = driver.cuModuleGetFunction(self.module, name.encode())
            _ok(err, "cuModuleGetFunction")
        self.fn = self.fns[names[0]]


def _ok(err, what):
    if int(err) != 0:
        raise RuntimeError(f"{what} failed: {err}")


_CACHE: dict = {}
LAUNCHES = [0]


def scalar_args(spec) -> list:
    vals = []
    for v in spec.scalars:
        vals.append(ctypes.c_double(v) if isinstance(v, float) else ctypes.c_longlong(int(v)))
    for p in spec.preds:
        vals += [ctypes.c_int(p.kind), ctypes.c_longlong(p.thr), ctypes.c_ulonglong(p.seed & ((1 << 64) - 1))]
    return vals


_BUDGET_KEEP: list = []  # the counters of launches in flight (freed by the caching allocator later)


def budget_arg(spec, dev) -> list:
    """the kernel's shared loop counter: a zeroed device word when the
    generated code has a loop, else a null pointer"""
    if not spec.need_budget:
        return [ctypes.c_void_p(0)]
    t = torch.zeros(1, dtype=torch.int64, device=dev)
    _BUDGET_KEEP.append(t)
    del _BUDGET_KEEP[:-64]
    return [ctypes.c_void_p(t.data_ptr())]


def map_jit(lam, arrays: list, env: dict, site_bits, n: int, status, out_dtype=None, device=None, funs=None,
            bits_for=None, loop_cap: int = 1 << 31, k_out: int = 1):
    """map lam arrays... on the GPU through a generated, cached kernel;
    returns (out, sites) -- out a list of k_out tensors when k_out > 1.
    Raises Unsupported for lambdas outside the language subset (the caller
    then uses the VM)."""
    from cuda.bindings import driver

    src, spec = generate(lam, arrays, env, site_bits, out_dtype, funs, bits_for, loop_cap, k_out)
    key = hashlib.sha1(src.encode()).hexdigest()
    kern = _CACHE.get(key)
    if kern is None:
        kern = _CACHE[key] = _Kernel(src)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    outs = [torch.empty(n, dtype=o, device=dev) for o in spec.out_dtypes]
    ret = outs if k_out > 1 else outs[0]
    if n == 0:
        return ret, spec.sites
    ins = [t.contiguous() for t in spec.inputs]
    arrs = [t.contiguous() for t in spec.arrays]
    vals = [ctypes.c_void_p(t.data_ptr()) for t in ins]
    for t in arrs:
        vals += [ctypes.c_void_p(t.data_ptr()), ctypes.c_longlong(t.numel())]
    vals += [ctypes.c_void_p(o.data_ptr()) for o in outs]
    vals += [ctypes.c_longlong(n), ctypes.c_int(0), ctypes.c_void_p(status.t.data_ptr())]
    vals += scalar_args(spec)
    vals += budget_arg(spec, dev)
    argv = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    grid = max(1, min((n + 255) // 256, sms * 8))
    (err,) = driver.cuLaunchKernel(kern.fn, grid, 1, 1, 256, 1, 1, 0, torch.cuda.current_stream(dev).cuda_stream,
                                   ctypes.addressof(argv), 0)
    _ok(err, "cuLaunchKernel")
    LAUNCHES[0] += 1
    return ret, spec.sites


def enabled() -> bool:
    return os.environ.get("IXG_JIT", "1") != "0"
