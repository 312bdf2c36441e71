"""Compile a lambda of the reference language into an ixg_map register
program (include/ixgpu.h, csrc/k_vm.cuh).

The reference evaluates ``map f xs ys ...`` by calling a Closure per element
(oracle.py:274-280, 94-107).  Here the lambda body -- already in ANF after
``normalize`` -- is compiled once into straight-line register code with
jumps for ``if`` and short-circuit ``&&``/``||`` (oracle.py:214-219), so an
IndexE inside an untaken branch is never evaluated, exactly like the
interpreter.  Captured scalars become constants, captured arrays become
gather sources, predicate parameters become device predicate descriptors.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

from . import _lib as L
from . import ir
from .pred import Pred

_BIN = {"+": L.VM_ADD, "-": L.VM_SUB, "*": L.VM_MUL, "==": L.VM_EQ, "!=": L.VM_NE, "<": L.VM_LT, "<=": L.VM_LE,
        ">": L.VM_GT, ">=": L.VM_GE}


class Unsupported(Exception):
    pass


@dataclass
class Compiled:
    insns: list = field(default_factory=list)  # (op, dst, a, b, c, imm)
    inputs: list = field(default_factory=list)  # per-element arrays then gather sources (tensors)
    preds: list = field(default_factory=list)
    sites: list = field(default_factory=list)   # IndexE nodes in site order (c operand)


class _Compiler:
    def __init__(self, env: dict, site_bits):
        self.env = env          # name -> ("scalar", int) | ("array", tensor) | ("pred", Pred)
        self.site_bits = site_bits  # IndexE node -> bits (V_BOUNDS)
        self.c = Compiled()
        self.nreg = 0
        self.arrays: dict = {}  # id(tensor) -> input slot

    def reg(self) -> int:
        r = self.nreg
        self.nreg += 1
        if r >= L.VM_REGS:
            raise Unsupported("lambda needs too many registers")
        return r

    def emit(self, op, dst=0, a=0, b=0, c=0, imm=0) -> int:
        self.c.insns.append([op, dst, a, b, c, imm])
        return len(self.c.insns) - 1

    def array_slot(self, t) -> int:
        k = id(t)
        if k not in self.arrays:
            if len(self.c.inputs) >= L.VM_MAX_IN:
                raise Unsupported("too many arrays in one lambda")
            self.arrays[k] = len(self.c.inputs)
            self.c.inputs.append(t)
        return self.arrays[k]

    def expr(self, e, scope: dict) -> int:
        k = ir.kind(e)
        if k == "Const":
            v = e.value
            if isinstance(v, float):
                raise Unsupported("floating point lambda")
            r = self.reg()
            self.emit(L.VM_CONST, r, imm=int(v))
            return r
        if k == "VarE":
            if e.name in scope:
                return scope[e.name]
            b = self.env.get(e.name)
            if b is None:
                raise Unsupported(f"free name {e.name}")
            if b[0] == "scalar":
                if isinstance(b[1], float):
                    raise Unsupported("floating point scalar")
                r = self.reg()
                self.emit(L.VM_CONST, r, imm=int(b[1]))
                return r
            raise Unsupported(f"{e.name} used as a scalar")
        if k == "BinOp":
            if e.op in ("&&", "||"):
                # short-circuit (oracle.py:216-219): bool(lhs) and/or bool(rhs)
                r = self.reg()
                a = self.expr(e.lhs, scope)
                z = self.reg()
                self.emit(L.VM_CONST, z, imm=0)
                self.emit(L.VM_NE, r, a, z)
                if e.op == "&&":
                    j = self.emit(L.VM_JZ, a=r)
                else:
                    nr = self.reg()
                    self.emit(L.VM_NOT, nr, r)
                    j = self.emit(L.VM_JZ, a=nr)
                b = self.expr(e.rhs, scope)
                self.emit(L.VM_NE, r, b, z)
                self.c.insns[j][4] = len(self.c.insns)
                return r
            if e.op not in _BIN:
                raise Unsupported(f"operator {e.op}")
            a = self.expr(e.lhs, scope)
            b = self.expr(e.rhs, scope)
            r = self.reg()
            self.emit(_BIN[e.op], r, a, b)
            return r
        if k == "NotE":
            a = self.expr(e.arg, scope)
            r = self.reg()
            self.emit(L.VM_NOT, r, a)
            return r
        if k == "If":
            c = self.expr(e.cond, scope)
            r = self.reg()
            j = self.emit(L.VM_JZ, a=c)
            t = self.expr(e.then, scope)
            self.emit(L.VM_MOV, r, t)
            jend = self.emit(L.VM_JMP)
            self.c.insns[j][4] = len(self.c.insns)
            f = self.expr(e.els, scope)
            self.emit(L.VM_MOV, r, f)
            self.c.insns[jend][4] = len(self.c.insns)
            return r
        if k == "Let":
            v = self.expr(e.rhs, scope)
            if len(e.names) != 1:
                raise Unsupported("tuple let inside a lambda")
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
            i = self.expr(e.idx, scope)
            slot = self.array_slot(b[1])
            site = len(self.c.sites)
            self.c.sites.append(e)
            r = self.reg()
            check = 1 if (self.site_bits(e) & L.V_BOUNDS) else 0
            self.emit(L.VM_IDX, r, i, slot, site, check)
            return r
        if k == "App":
            if ir.kind(e.fun) == "VarE":
                b = self.env.get(e.fun.name)
                if b is not None and b[0] == "pred" and len(e.args) == 1:
                    a = self.expr(e.args[0], scope)
                    if b[1] not in self.c.preds:
                        if len(self.c.preds) >= L.VM_MAX_PRED:
                            raise Unsupported("too many predicates")
                        self.c.preds.append(b[1])
                    r = self.reg()
                    self.emit(L.VM_PRED, r, a, self.c.preds.index(b[1]))
                    return r
                if e.fun.name == "length" and len(e.args) == 1 and ir.kind(e.args[0]) == "VarE":
                    b = self.env.get(e.args[0].name)
                    if b is not None and b[0] == "array":
                        r = self.reg()
                        self.emit(L.VM_LEN, r, 0, self.array_slot(b[1]))
                        return r
            raise Unsupported(f"application {ir.expr_str(e)} inside a lambda")
        raise Unsupported(k)


def compile_map(lam, arrays: list, env: dict, site_bits=lambda node: L.V_BOUNDS) -> Compiled:
    """lam: Lambda node; arrays: per-element device tensors (one per lambda
    parameter); env: captured names.  Returns the program with input slots
    0..len(arrays)-1 holding the per-element arrays and one output."""
    if len(lam.params) != len(arrays):
        raise Unsupported("lambda arity")
    comp = _Compiler(env, site_bits)
    for t in arrays:
        comp.c.inputs.append(t)
    scope = {}
    for i, p in enumerate(lam.params):
        r = comp.reg()
        comp.emit(L.VM_IN, r, i)
        if p != "_":
            scope[p] = r
    res = comp.expr(lam.body, scope)
    comp.emit(L.VM_OUT, 0, res, 0)
    if len(comp.c.insns) > L.VM_MAX_INSN:
        raise Unsupported("lambda too long")
    return comp.c
