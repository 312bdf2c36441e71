"""Predicate descriptors: the reproducible stand-in for predicate arguments.

The reference passes Python callables for ``p : i64 -> bool`` parameters and
calls them from the interpreter (``oracle.py:327-329``); its random-input
generator draws ``x < thr``, ``x > thr`` or a memoised random table
(``oracle.py:686-696``).  A :class:`Pred` is *both*: a Python callable with
exactly those semantics (so the reference interpreter can run it) and a
by-value descriptor the CUDA kernels evaluate (``ixg_pred``).  The random
table becomes ``HASH``: one bit of a 64-bit mix of ``x`` and a seed,
bit-identical in Python, in ``oracle/ixoracle.c`` and on the device.
"""

from __future__ import annotations

from dataclasses import dataclass

MASK64 = (1 << 64) - 1

LT, GT, LE, GE, EQ, NE, HASH, TRUE, FALSE = range(9)
_NAMES = {LT: "<", GT: ">", LE: "<=", GE: ">=", EQ: "==", NE: "!="}


def mix64(z: int) -> int:
    """splitmix64 finaliser (== ixo_mix64 / ixg::mix64)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


@dataclass(frozen=True)
class Pred:
    kind: int
    thr: int = 0
    seed: int = 0

    def __call__(self, x) -> bool:
        k = self.kind
        if k == LT:
            return x < self.thr
        if k == GT:
            return x > self.thr
        if k == LE:
            return x <= self.thr
        if k == GE:
            return x >= self.thr
        if k == EQ:
            return x == self.thr
        if k == NE:
            return x != self.thr
        if k == HASH:
            return (mix64((int(x) & MASK64) ^ self.seed) >> 63) == 1
        return k == TRUE

    @classmethod
    def lt(cls, thr: int) -> "Pred":
        return cls(LT, thr)

    @classmethod
    def gt(cls, thr: int) -> "Pred":
        return cls(GT, thr)

    @classmethod
    def le(cls, thr: int) -> "Pred":
        return cls(LE, thr)

    @classmethod
    def ge(cls, thr: int) -> "Pred":
        return cls(GE, thr)

    @classmethod
    def hash(cls, seed: int) -> "Pred":
        return cls(HASH, 0, seed & MASK64)

    def to_json(self) -> dict:
        return {"pred": self.kind, "thr": self.thr, "seed": self.seed}

    @classmethod
    def from_json(cls, d: dict) -> "Pred":
        return cls(int(d["pred"]), int(d.get("thr", 0)), int(d.get("seed", 0)))

    def __repr__(self) -> str:
        if self.kind in _NAMES:
            return f"Pred(x {_NAMES[self.kind]} {self.thr})"
        if self.kind == HASH:
            return f"Pred(hash {self.seed:#x})"
        return f"Pred({'true' if self.kind == TRUE else 'false'})"
