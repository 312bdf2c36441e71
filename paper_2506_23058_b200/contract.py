"""Runtime check of a function's preconditions before ELIDED variants run.

The verifier proves a site's dynamic check unnecessary *under the function's
parameter annotations*: ``Analyzer._bind_param`` / ``_assume_cond`` /
``_assume_prop`` (/root/reference/pkg/src/ixverify/infer.py:231-338) ASSUME
``Range``, ``Inj``, ``Bij``, ``Mono`` and plain boolean conditions, they are
never proved for an entry point.  The reference interpreter ignores them
(``Interp.call``, oracle.py:127-135): a call that violates an annotation
still gets the program's own answer -- an ``OutOfBounds``, a
``NonIdempotentScatter`` or a value.  So the drop-in executor checks an
entry function's annotations on the device first and runs the CHECKED
variants when one fails (or cannot be checked), which reproduces the
reference exactly; only calls that satisfy the contract run ELIDED.

Each property restates the reference's own concrete predicate
(oracle.py:712-734 ``_check_pre_atom``; ``chk_range`` / ``chk_mono`` /
``chk_inj`` / ``chk_bij`` :478-520) as one streaming device pass
(csrc/k_contract.cuh).  ``Equiv``, ``FiltPart``, ``InvFiltPart`` and
``OrthogPreds`` have no cheap check: a function assuming them runs CHECKED.
"""

from __future__ import annotations

import math

import torch

from . import ir
from . import ops

PROPERTY_HEADS = {"Range", "Equiv", "Mono", "Inj", "Bij", "FiltPart", "InvFiltPart", "OrthogPreds"}
_MONO_OPS = {"le": 0, "lt": 1, "ge": 2, "gt": 3}


class Unknown(Exception):
    """An annotation that cannot be evaluated here (treated as violated)."""


def conjuncts(e):
    if ir.kind(e) == "BinOp" and e.op == "&&":
        yield from conjuncts(e.lhs)
        yield from conjuncts(e.rhs)
    else:
        yield e


def has_preconditions(fdef, required=None) -> bool:
    """any annotation to check (required: see check)?"""
    if required is not None:
        return bool(required)
    return any(p.pre is not None for p in fdef.params)


def bind_sizes(fdef, values: dict) -> dict:
    """oracle.py:137-161 on the values at hand: [n] := len(arg), [n+1] := len(arg) - 1."""
    env = dict(values)
    for p in fdef.params:
        t = p.type
        if p.name not in env:
            continue
        v = env[p.name]
        if ir.kind(t) != "TArray" or not (isinstance(v, torch.Tensor) or hasattr(v, "__len__")):
            continue
        n = v.numel() if isinstance(v, torch.Tensor) else len(v)
        sz = t.size
        if sz is None:
            continue
        if ir.kind(sz) == "VarE":
            env.setdefault(sz.name, n)
        elif (ir.kind(sz) == "BinOp" and sz.op == "+" and ir.kind(sz.lhs) == "VarE"
              and ir.kind(sz.rhs) == "Const"):
            env.setdefault(sz.lhs.name, n - sz.rhs.value)
    return env


def scalar(e, env):
    """Host value of a scalar annotation expression (sizes, scalar params, inf)."""
    k = ir.kind(e)
    if k == "Const":
        return e.value
    if k == "VarE":
        v = env.get(e.name)
        if v is None or isinstance(v, torch.Tensor) or not isinstance(v, (bool, int, float)):
            raise Unknown(e.name)
        return v
    if k == "NotE":
        return not scalar(e.arg, env)
    if k == "BinOp":
        if e.op == "&&":
            return bool(scalar(e.lhs, env)) and bool(scalar(e.rhs, env))
        if e.op == "||":
            return bool(scalar(e.lhs, env)) or bool(scalar(e.rhs, env))
        a, b = scalar(e.lhs, env), scalar(e.rhs, env)
        ops_ = {"+": lambda: a + b, "-": lambda: a - b, "*": lambda: a * b, "==": lambda: a == b,
                "!=": lambda: a != b, "<": lambda: a < b, "<=": lambda: a <= b, ">": lambda: a > b,
                ">=": lambda: a >= b}
        if e.op not in ops_:
            raise Unknown(e.op)
        try:
            return ops_[e.op]()
        except (TypeError, ValueError) as ex:  # inf - inf and friends
            raise Unknown(str(ex)) from None
    raise Unknown(k)


def _interval(e, env):
    if ir.kind(e) != "TupleE" or len(e.items) != 2:
        raise Unknown("interval")
    return scalar(e.items[0], env), scalar(e.items[1], env)


def _int_array(v) -> torch.Tensor:
    if not isinstance(v, torch.Tensor) or v.is_floating_point():
        raise Unknown("not an integer array")
    return v.view(torch.uint8) if v.dtype == torch.bool else v


def _clamp_int(lo, hi, mn: int, mx: int):
    """[lo, hi] (ints or +-inf) intersected with [mn, mx] as ints."""
    lo2 = mn if (isinstance(lo, float) and math.isinf(lo) and lo < 0) else max(mn, math.ceil(lo))
    hi2 = mx if (isinstance(hi, float) and math.isinf(hi) and hi > 0) else min(mx, math.floor(hi))
    return int(lo2), int(hi2)


def _atom(atom, env) -> bool:
    if ir.kind(atom) == "App" and ir.kind(atom.fun) == "VarE" and atom.fun.name in PROPERTY_HEADS:
        head = atom.fun.name
        if not atom.args or ir.kind(atom.args[0]) != "VarE" or atom.args[0].name not in env:
            raise Unknown(head)
        x = env[atom.args[0].name]
        if head == "Range":
            lo, hi = _interval(atom.args[1], env)
            if not isinstance(x, torch.Tensor):
                return bool(lo <= scalar(atom.args[0], env) <= hi)
            a = _int_array(x)
            if a.numel() == 0:
                return True
            mn, mx = ops.minmax(a).tolist()
            return bool(lo <= mn and mx <= hi)
        if head == "Mono":
            a = _int_array(x)
            op = atom.args[1].name if len(atom.args) > 1 and ir.kind(atom.args[1]) == "VarE" else "le"
            if op not in _MONO_OPS:
                raise Unknown(f"Mono {op}")
            return a.numel() < 2 or int(ops.mono_violations(a, _MONO_OPS[op]).item()) == 0
        if head in ("Inj", "Bij"):
            a = _int_array(x)
            lo, hi = _interval(atom.args[1], env)
            if head == "Bij":
                if len(atom.args) != 3:
                    raise Unknown("segmented Bij")
                ilo, ihi = _interval(atom.args[2], env)
                if not all(isinstance(v, int) for v in (ilo, ihi)):
                    raise Unknown("Bij image")
            else:
                ilo, ihi = None, None
            if a.numel() == 0:
                return head == "Inj" or ihi < ilo
            mn, mx = ops.minmax(a).tolist()
            clo, chi = _clamp_int(lo, hi, mn, mx)
            if clo > chi:  # no value inside the codomain interval
                return head == "Inj" or ihi < ilo
            r = ops.inj_check(a, clo, chi, clo if ilo is None else ilo, chi if ihi is None else ihi)
            if r is None:
                raise Unknown(f"{head}: value range too wide for a claim bitmap")
            cnt, rep, out_img = r.tolist()
            if rep:
                return False
            if head == "Inj":
                return True
            return out_img == 0 and cnt == max(0, ihi - ilo + 1)
        raise Unknown(head)  # Equiv / FiltPart / InvFiltPart / OrthogPreds
    return bool(scalar(atom, env))


def check(fdef, values: dict, required=None):
    """Do `fdef`'s parameter annotations hold for `values` (param name ->
    device tensor / host scalar)?  Returns (ok, reason).  `required`: the
    "param|atom" keys the verdicts depend on (select.required_atoms); the
    other conjuncts back no elided check and are not evaluated.  None: all."""
    from .select import atom_key

    need = None if required is None else set(required)
    env = bind_sizes(fdef, values)
    for p in fdef.params:
        if p.pre is None:
            continue
        for atom in conjuncts(p.pre):
            if need is not None and atom_key(p.name, atom) not in need:
                continue
            try:
                ok = _atom(atom, env)
            except Unknown as ex:
                return False, f"{p.name}: cannot check {ir.expr_str(atom)} ({ex})"
            if not ok:
                return False, f"{p.name}: {ir.expr_str(atom)} does not hold"
    return True, ""
