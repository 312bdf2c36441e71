"""Program representation at the drop-in boundary.

``eval_program`` receives the reference's normalized AST
(``ixverify.ast``, /root/reference/pkg/src/ixverify/ast.py; produced by
``parser.parse_program`` + ``normalize.normalize``).  Everything here walks
that AST by *class name and field name only*, so it works on the reference's
own objects and on the light mirror nodes below, which are what a program
snapshot (JSON, ``data/programs.json``) turns back into on a machine without
the reference installed (the GPU box).

Also here: ``expr_str`` (the reference's diagnostic printer, ast.py
``expr_str``, restated -- it is the ``site`` text of ``OutOfBounds``) and
``fingerprint`` (a structural hash of a normalized function that ignores
source positions and the fresh ``%aN`` names normalization invents, so
pipelines and frozen verifier verdicts can be matched without the
reference's global name counter).
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from typing import Any, Optional


# ----------------------------------------------------------------- mirror nodes
# Same class and field names as ixverify.ast (the data model is the
# interface; behaviour lives in the executor).
@dataclass(frozen=True)
class TBase:
    name: str


@dataclass(frozen=True)
class TArray:
    size: Any
    elem: Any


@dataclass(frozen=True)
class TTuple:
    items: tuple


@dataclass(frozen=True)
class TFun:
    arg: Any
    res: Any


@dataclass
class Node:
    pos: tuple = (0, 0)


def _mk(name, fields):
    ns = {"__annotations__": {f: Any for f in fields}}
    if fields[-1] == "pos":
        ns["pos"] = (0, 0)
    cls = dataclass(type(name, (), ns))
    return cls


Const = _mk("Const", ["value", "pos"])
VarE = _mk("VarE", ["name", "pos"])
BinOp = _mk("BinOp", ["op", "lhs", "rhs", "pos"])
NotE = _mk("NotE", ["arg", "pos"])
IndexE = _mk("IndexE", ["arr", "idx", "pos"])
If = _mk("If", ["cond", "then", "els", "pos"])
Let = _mk("Let", ["names", "rhs", "body", "pos"])
TupleE = _mk("TupleE", ["items", "pos"])
Lambda = _mk("Lambda", ["params", "body", "pos"])
App = _mk("App", ["fun", "args", "pos"])
LoopParam = _mk("LoopParam", ["name", "type", "pre"])
Loop = _mk("Loop", ["params", "inits", "kind", "cond", "counter", "bound", "body", "pos"])
Param = _mk("Param", ["name", "type", "pre", "pos"])
FunDef = _mk("FunDef", ["name", "sizes", "params", "result_type", "post", "body", "pos"])
Program = _mk("Program", ["defs", "path"])

_CLASSES = {c.__name__: c for c in (TBase, TArray, TTuple, TFun, Const, VarE, BinOp, NotE, IndexE, If, Let, TupleE,
                                    Lambda, App, LoopParam, Loop, Param, FunDef, Program)}
_FIELDS = {
    "TBase": ["name"], "TArray": ["size", "elem"], "TTuple": ["items"], "TFun": ["arg", "res"],
    "Const": ["value", "pos"], "VarE": ["name", "pos"], "BinOp": ["op", "lhs", "rhs", "pos"],
    "NotE": ["arg", "pos"], "IndexE": ["arr", "idx", "pos"], "If": ["cond", "then", "els", "pos"],
    "Let": ["names", "rhs", "body", "pos"], "TupleE": ["items", "pos"], "Lambda": ["params", "body", "pos"],
    "App": ["fun", "args", "pos"], "LoopParam": ["name", "type", "pre"],
    "Loop": ["params", "inits", "kind", "cond", "counter", "bound", "body", "pos"],
    "Param": ["name", "type", "pre", "pos"],
    "FunDef": ["name", "sizes", "params", "result_type", "post", "body", "pos"], "Program": ["defs", "path"],
}


def kind(node) -> str:
    return type(node).__name__


# ----------------------------------------------------------------- JSON
def to_json(x):
    """Serialize a reference (or mirror) AST to plain JSON data."""
    if x is None or isinstance(x, (bool, str)):
        return x
    if isinstance(x, float):
        if x != x or x in (float("inf"), float("-inf")):
            return {"$float": repr(x)}
        return {"$float": repr(x)}
    if isinstance(x, int):
        return x
    if isinstance(x, (tuple, list)):
        return [to_json(v) for v in x]
    k = kind(x)
    if k not in _FIELDS:
        raise TypeError(f"cannot serialize {k}")
    return {"$": k, **{f: to_json(getattr(x, f)) for f in _FIELDS[k]}}


def from_json(d):
    if d is None or isinstance(d, (bool, int, str)):
        return d
    if isinstance(d, list):
        return tuple(from_json(v) for v in d)
    if "$float" in d:
        return float(d["$float"])
    k = d["$"]
    cls = _CLASSES[k]
    return cls(**{f: from_json(d[f]) for f in _FIELDS[k]})


def dumps(program) -> str:
    return json.dumps(to_json(program))


def loads(text: str):
    return from_json(json.loads(text))


# ----------------------------------------------------------------- expr_str
def expr_str(e) -> str:
    """The reference's diagnostic text of an expression (ixverify/ast.py
    expr_str); OutOfBounds(site) carries exactly this string."""
    k = kind(e)
    if k == "Const":
        v = e.value
        if v is True:
            return "true"
        if v is False:
            return "false"
        return str(v)
    if k == "VarE":
        return e.name
    if k == "BinOp":
        return f"{expr_str(e.lhs)} {e.op} {expr_str(e.rhs)}"
    if k == "NotE":
        return f"!{expr_str(e.arg)}"
    if k == "IndexE":
        base = expr_str(e.arr)
        if kind(e.arr) not in ("VarE", "IndexE"):
            base = f"({base})"
        return f"{base}[{expr_str(e.idx)}]"
    if k == "If":
        return f"if {expr_str(e.cond)} then {expr_str(e.then)} else {expr_str(e.els)}"
    if k == "Let":
        pat = e.names[0] if len(e.names) == 1 else "(" + ", ".join(e.names) + ")"
        return f"let {pat} = {expr_str(e.rhs)} in {expr_str(e.body)}"
    if k == "TupleE":
        return "(" + ", ".join(expr_str(x) for x in e.items) + ")"
    if k == "Lambda":
        return "\\" + " ".join(e.params) + " -> " + expr_str(e.body)
    if k == "App":
        parts = [expr_str(e.fun)] + [
            f"({expr_str(a)})" if kind(a) not in ("VarE", "Const") else expr_str(a) for a in e.args
        ]
        return " ".join(parts)
    if k == "Loop":
        return "loop ..."
    return repr(e)


# ----------------------------------------------------------------- traversal
def children(e):
    k = kind(e)
    if k in ("Const", "VarE"):
        return []
    if k == "BinOp":
        return [e.lhs, e.rhs]
    if k == "NotE":
        return [e.arg]
    if k == "IndexE":
        return [e.arr, e.idx]
    if k == "If":
        return [e.cond, e.then, e.els]
    if k == "Let":
        return [e.rhs, e.body]
    if k == "TupleE":
        return list(e.items)
    if k == "Lambda":
        return [e.body]
    if k == "App":
        return [e.fun, *e.args]
    if k == "Loop":
        out = list(e.inits)
        if e.cond is not None:
            out.append(e.cond)
        if e.bound is not None:
            out.append(e.bound)
        out.append(e.body)
        return out
    return []


def sites(fundef):
    """Checkable sites of a function in evaluation order: IndexE (bounds) and
    App scatter (scatter-safety).  Returns [(kind, pos, node)]."""
    out = []

    def walk(e):
        for c in children(e):
            walk(c)
        k = kind(e)
        if k == "IndexE":
            out.append(("bounds", tuple(e.pos), e))
        elif k == "App" and kind(e.fun) == "VarE" and e.fun.name == "scatter":
            out.append(("scatter-safety", tuple(e.pos), e))

    # evaluation order: Let rhs before body (children order), post-order
    walk(fundef.body)
    return out


# ----------------------------------------------------------------- fingerprint
def canonical(fundef, contract: bool = False) -> str:
    """Position-free, alpha-normalised text of a normalized function: bound
    names (params, lets, lambda params, loop variables) become v0, v1, ...
    in binding order; free names (builtins, other functions) stay.

    contract=False: the body only (what a pipeline must compute -- the
    registry's key).  contract=True adds everything the verifier ASSUMES or
    PROVES about the function: the parameter preconditions (``Param.pre``,
    assumed by infer.py:231-338 ``_bind_param`` / ``_assume_cond``), loop
    parameter types and preconditions, the result type and the
    postcondition (``FunDef.post``) -- two functions with the same body but
    different annotations get different verdicts, so the frozen verdict
    table is keyed by this form (``closure_fingerprint``)."""
    names: dict = {}

    def bind(n):
        if n == "_":
            return "_"
        names[n] = f"v{len(names)}"
        return names[n]

    def ref(n):
        return names.get(n, n)

    def ty(t):
        if t is None:
            return "?"
        k = kind(t)
        if k == "TBase":
            return t.name
        if k == "TArray":
            return f"[{ex(t.size) if t.size is not None else ''}]{ty(t.elem)}"
        if k == "TTuple":
            return "(" + ",".join(ty(x) for x in t.items) + ")"
        if k == "TFun":
            return f"({ty(t.arg)}->{ty(t.res)})"
        return k

    def ex(e):
        k = kind(e)
        if k == "Const":
            return f"#{e.value!r}"
        if k == "VarE":
            return ref(e.name)
        if k == "BinOp":
            return f"({e.op} {ex(e.lhs)} {ex(e.rhs)})"
        if k == "NotE":
            return f"(! {ex(e.arg)})"
        if k == "IndexE":
            return f"(idx {ex(e.arr)} {ex(e.idx)})"
        if k == "If":
            return f"(if {ex(e.cond)} {ex(e.then)} {ex(e.els)})"
        if k == "Let":
            rhs = ex(e.rhs)
            pat = " ".join(bind(n) for n in e.names)
            return f"(let ({pat}) {rhs} {ex(e.body)})"
        if k == "TupleE":
            return "(tup " + " ".join(ex(x) for x in e.items) + ")"
        if k == "Lambda":
            saved = dict(names)
            ps = " ".join(bind(p) for p in e.params)
            body = ex(e.body)
            names.clear()
            names.update(saved)
            return f"(lam ({ps}) {body})"
        if k == "App":
            return "(app " + " ".join(ex(x) for x in (e.fun, *e.args)) + ")"
        if k == "Loop":
            inits = " ".join(ex(x) for x in e.inits)
            bound = ex(e.bound) if e.bound is not None else ""
            ps = " ".join(bind(p.name) for p in e.params)
            if contract:
                ps += " | " + " ".join(f"{ty(p.type)}:{ex(p.pre) if p.pre is not None else '-'}" for p in e.params)
            cnt = bind(e.counter) if e.counter else ""
            cond = ex(e.cond) if e.cond is not None else ""
            return f"(loop {e.kind} ({ps}) ({inits}) {cnt} {bound} {cond} {ex(e.body)})"
        return k

    sizes = " ".join(bind(s) for s in fundef.sizes)
    params = " ".join(f"{bind(p.name)}:{ty(p.type)}" for p in fundef.params)
    if not contract:
        return f"(def ({sizes}) ({params}) {ex(fundef.body)})"
    # every parameter is bound before any precondition is printed (a
    # precondition may name a later parameter)
    pres = " ".join(ex(p.pre) if p.pre is not None else "-" for p in fundef.params)
    post = ex(fundef.post) if fundef.post is not None else "-"
    return (f"(def ({sizes}) ({params}) (pre {pres}) (res {ty(fundef.result_type)}) (post {post}) "
            f"{ex(fundef.body)})")


_FP_CACHE: dict = {}  # id(fundef) -> (fundef, fingerprint): programs are immutable values


def fingerprint(fundef) -> str:
    hit = _FP_CACHE.get(id(fundef))
    if hit is not None and hit[0] is fundef:
        return hit[1]
    fp = hashlib.sha256(canonical(fundef).encode()).hexdigest()[:16]
    if len(_FP_CACHE) > 4096:
        _FP_CACHE.clear()
    _FP_CACHE[id(fundef)] = (fundef, fp)
    return fp


def callees(fundef, names) -> list:
    """Program functions (from `names`) that `fundef` applies, sorted."""
    out = set()

    def walk(e):
        if kind(e) == "App" and kind(e.fun) == "VarE" and e.fun.name in names:
            out.add(e.fun.name)
        for c in children(e):
            walk(c)

    walk(fundef.body)
    return sorted(out)


def closure_fingerprint(program, fundef) -> str:
    """Key of a function's verifier verdicts: its contract form (body +
    annotations, ``canonical(contract=True)``) together with the closure
    fingerprints of every program function it calls, transitively -- the
    verifier proves a caller's sites from its callees' analysis results
    (infer.py:1387-1420 applies a callee's gamma and postcondition), so a
    redefined helper must change the caller's key.  Recursion is cut by
    naming the cycle."""
    defs = {f.name: f for f in program.defs}
    memo: dict = {}

    def fp(f, stack):
        if f.name in memo:
            return memo[f.name]
        if f.name in stack:
            return f"rec:{f.name}"
        parts = [canonical(f, contract=True)]
        for c in callees(f, defs):
            if c == f.name:
                parts.append(f"{c}=self")
            else:
                parts.append(f"{c}={fp(defs[c], stack | {f.name})}")
        h = hashlib.sha256("\n".join(parts).encode()).hexdigest()[:16]
        memo[f.name] = h
        return h

    return fp(fundef, frozenset())


def find_def(program, name: str):
    for f in program.defs:
        if f.name == name:
            return f
    raise KeyError(name)
