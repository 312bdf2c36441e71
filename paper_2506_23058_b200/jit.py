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
from dataclasses import dataclass, field

import torch

from . import _lib as L
from . import ir
from .pred import Pred
from .vm import Unsupported

_CMP = {"==": "==", "!=": "!=", "<": "<", "<=": "<=", ">": ">", ">=": ">="}
_ARITH = {"+": "+", "-": "-", "*": "*"}
_CT = {torch.int64: "long long", torch.int32: "int", torch.uint8: "unsigned char", torch.bool: "unsigned char"}

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
"""


@dataclass
class _Spec:
    inputs: list = field(default_factory=list)   # per-element tensors
    arrays: list = field(default_factory=list)   # gather sources (tensors)
    scalars: list = field(default_factory=list)  # captured ints
    preds: list = field(default_factory=list)    # Pred
    sites: list = field(default_factory=list)    # IndexE nodes in site order


class _Gen:
    def __init__(self, env: dict, site_bits):
        self.env, self.site_bits = env, site_bits
        self.spec = _Spec()
        self.body: list = []
        self.ntmp = 0
        self.depth = 2
        self._arr_slot: dict = {}
        # what a failed CHECKED index site does after recording the failure
        self.on_fail = "goto next;"

    def line(self, s: str):
        self.body.append("  " * self.depth + s)

    def tmp(self) -> str:
        t = f"t{self.ntmp}"
        self.ntmp += 1
        return t

    def new(self, value: str) -> str:
        t = self.tmp()
        self.line(f"const long long {t} = {value};")
        return t

    def array_slot(self, t) -> int:
        k = id(t)
        if k not in self._arr_slot:
            self._arr_slot[k] = len(self.spec.arrays)
            self.spec.arrays.append(t)
        return self._arr_slot[k]

    def scalar(self, v: int) -> str:
        self.spec.scalars.append(int(v))
        return f"s{len(self.spec.scalars) - 1}"

    def expr(self, e, scope: dict) -> str:
        k = ir.kind(e)
        if k == "Const":
            if isinstance(e.value, float):
                raise Unsupported("floating point lambda")
            return f"{int(e.value)}LL"
        if k == "VarE":
            if e.name in scope:
                return scope[e.name]
            b = self.env.get(e.name)
            if b is None:
                raise Unsupported(f"free name {e.name}")
            if b[0] == "scalar":
                if isinstance(b[1], float):
                    raise Unsupported("floating point scalar")
                return self.scalar(b[1])
            raise Unsupported(f"{e.name} used as a scalar")
        if k == "BinOp":
            if e.op in ("&&", "||"):
                r = self.tmp()
                self.line(f"long long {r};")
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
            if e.op in _ARITH:
                # two's-complement wrap like the VM's long long arithmetic
                return self.new(f"(long long)((u64)({a}) {_ARITH[e.op]} (u64)({b}))")
            if e.op in _CMP:
                return self.new(f"(long long)(({a}) {_CMP[e.op]} ({b}))")
            raise Unsupported(f"operator {e.op}")
        if k == "NotE":
            a = self.expr(e.arg, scope)
            return self.new(f"(long long)(({a}) == 0)")
        if k == "If":
            c = self.expr(e.cond, scope)
            r = self.tmp()
            self.line(f"long long {r};")
            self.line(f"if (({c}) != 0) {{")
            self.depth += 1
            t = self.expr(e.then, scope)
            self.line(f"{r} = {t};")
            self.depth -= 1
            self.line("} else {")
            self.depth += 1
            f = self.expr(e.els, scope)
            self.line(f"{r} = {f};")
            self.depth -= 1
            self.line("}")
            return r
        if k == "Let":
            if len(e.names) != 1:
                raise Unsupported("tuple let inside a lambda")
            v = self.new(self.expr(e.rhs, scope))
            inner = dict(scope)
            if e.names[0] != "_":
                inner[e.names[0]] = v
            return self.expr(e.body, inner)
        if k == "IndexE":
            if ir.kind(e.arr) != "VarE" or e.arr.name in scope:
                raise Unsupported("indexing a computed array")
            b = self.env.get(e.arr.name)
            if b is None or b[0] != "array":
                raise Unsupported(f"indexing non-array {e.arr.name}")
            i = self.new(self.expr(e.idx, scope))
            slot = self.array_slot(b[1])
            site = len(self.spec.sites)
            self.spec.sites.append(e)
            if self.site_bits(e) & L.V_BOUNDS:
                self.line(f"if ((u64){i} >= (u64)len{slot}) {{ fail_oob(st, stmt, i, {site}); {self.on_fail} }}")
            return self.new(f"(long long)a{slot}[{i}]")
        if k == "App" and ir.kind(e.fun) == "VarE":
            b = self.env.get(e.fun.name)
            if b is not None and b[0] == "pred" and len(e.args) == 1:
                a = self.expr(e.args[0], scope)
                p: Pred = b[1]
                if p not in self.spec.preds:
                    self.spec.preds.append(p)
                j = self.spec.preds.index(p)
                return self.new(f"pred(pk{j}, pt{j}, ps{j}, {a})")
            if e.fun.name == "length" and len(e.args) == 1 and ir.kind(e.args[0]) == "VarE":
                b = self.env.get(e.args[0].name)
                if b is not None and b[0] == "array":
                    return f"len{self.array_slot(b[1])}"
        raise Unsupported(f"{k} inside a lambda: {ir.expr_str(e)}")

    def tuple_expr(self, e, scope: dict, k: int) -> list:
        """The k components of a tuple-valued body (a k-ary scan operator,
        oracle.py:286-290), evaluated left to right like TupleE
        (oracle.py:199-200); Let and If may wrap the tuple."""
        if k == 1:
            return [self.expr(e, scope)]
        kd = ir.kind(e)
        if kd == "TupleE":
            if len(e.items) != k:
                raise Unsupported("operator result arity")
            return [self.new(self.expr(x, scope)) for x in e.items]
        if kd == "Let":
            if len(e.names) != 1:
                raise Unsupported("tuple let inside a lambda")
            v = self.new(self.expr(e.rhs, scope))
            inner = dict(scope)
            if e.names[0] != "_":
                inner[e.names[0]] = v
            return self.tuple_expr(e.body, inner, k)
        if kd == "If":
            c = self.expr(e.cond, scope)
            rs = [self.tmp() for _ in range(k)]
            self.line("long long " + ", ".join(rs) + ";")
            self.line(f"if (({c}) != 0) {{")
            for branch in (e.then, e.els):
                self.depth += 1
                vs = self.tuple_expr(branch, scope, k)
                for r, v in zip(rs, vs):
                    self.line(f"{r} = {v};")
                self.depth -= 1
                self.line("} else {" if branch is e.then else "}")
            return rs
        raise Unsupported(f"{kd} as a tuple-valued operator body")


def _ctype(t: torch.Tensor) -> str:
    if t.dtype not in _CT:
        raise Unsupported(f"element type {t.dtype}")
    return _CT[t.dtype]


def generate(lam, arrays: list, env: dict, site_bits=lambda node: L.V_BOUNDS, out_dtype=torch.int64):
    """-> (CUDA source, _Spec).  The source depends on the lambda, the
    element types and which index sites are checked -- not on the values of
    captured scalars or predicates (kernel parameters)."""
    if len(lam.params) != len(arrays):
        raise Unsupported("lambda arity")
    g = _Gen(env, site_bits)
    g.spec.inputs = list(arrays)
    scope = {}
    for j, p in enumerate(lam.params):
        if p != "_":
            scope[p] = f"x{j}"
    res = g.expr(lam.body, scope)
    params = [f"const {_ctype(t)}* __restrict__ in{j}" for j, t in enumerate(arrays)]
    params += [f"const {_ctype(t)}* __restrict__ a{j}, long long len{j}" for j, t in enumerate(g.spec.arrays)]
    params += [f"{_CT[out_dtype]}* __restrict__ out", "long long n", "int stmt", "ixg_status* st"]
    params += [f"long long s{j}" for j in range(len(g.spec.scalars))]
    params += [f"int pk{j}, long long pt{j}, u64 ps{j}" for j in range(len(g.spec.preds))]
    loads = [f"    const long long x{j} = (long long)in{j}[i];" for j in range(len(arrays))]
    store = f"({_CT[out_dtype]})(({res}) != 0)" if out_dtype in (torch.uint8, torch.bool) else \
        f"({_CT[out_dtype]})({res})"
    src = (_PRELUDE + 'extern "C" __global__ void __launch_bounds__(256) ixg_jit_map(' + ", ".join(params) + ") {\n"
           "  const long long stride = (long long)gridDim.x * blockDim.x;\n"
           "  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {\n"
           "   {\n" + "\n".join(loads) + "\n" + "\n".join(g.body) + f"\n    out[i] = {store};\n   }}\n"
           "  next:;\n  }\n}\n")
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


def map_jit(lam, arrays: list, env: dict, site_bits, n: int, status, out_dtype=torch.int64, device=None):
    """map lam arrays... on the GPU through a generated, cached kernel;
    returns (out, sites).  Raises Unsupported for lambdas outside the
    language subset (the caller then uses the VM)."""
    from cuda.bindings import driver

    src, spec = generate(lam, arrays, env, site_bits, out_dtype)
    key = hashlib.sha1(src.encode()).hexdigest()
    kern = _CACHE.get(key)
    if kern is None:
        kern = _CACHE[key] = _Kernel(src)
    dev = device or torch.device("cuda", torch.cuda.current_device())
    out = torch.empty(n, dtype=out_dtype, device=dev)
    if n == 0:
        return out, spec.sites
    ins = [t.contiguous() for t in spec.inputs]
    arrs = [t.contiguous() for t in spec.arrays]
    vals = [ctypes.c_void_p(t.data_ptr()) for t in ins]
    for t in arrs:
        vals += [ctypes.c_void_p(t.data_ptr()), ctypes.c_longlong(t.numel())]
    vals += [ctypes.c_void_p(out.data_ptr()), ctypes.c_longlong(n), ctypes.c_int(0), ctypes.c_void_p(status.t.data_ptr())]
    vals += [ctypes.c_longlong(v) for v in spec.scalars]
    for p in spec.preds:
        vals += [ctypes.c_int(p.kind), ctypes.c_longlong(p.thr), ctypes.c_ulonglong(p.seed & ((1 << 64) - 1))]
    argv = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    grid = max(1, min((n + 255) // 256, sms * 8))
    (err,) = driver.cuLaunchKernel(kern.fn, grid, 1, 1, 256, 1, 1, 0, torch.cuda.current_stream(dev).cuda_stream,
                                   ctypes.addressof(argv), 0)
    _ok(err, "cuLaunchKernel")
    LAUNCHES[0] += 1
    return out, spec.sites


def enabled() -> bool:
    return os.environ.get("IXG_JIT", "1") != "0"
