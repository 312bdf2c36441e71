"""Record whether the reference's own evaluation produced an integer outside
int64 (generator-side instrumentation, used by make_golden.py and
make_fuzz.py; the reference is unmodified -- Interp._binop is wrapped only
inside these scripts).

The reference's ints are unbounded (oracle.py:214-240); the GPU path
computes in int64 and raises IntegerOverflow rather than return a wrapped
value.  A case whose reference run never left int64 must match exactly on
the GPU; one that did ("big": true) may raise IntegerOverflow instead (and
must, when a result itself does not fit)."""

from __future__ import annotations

import contextlib

I64_MIN, I64_MAX = -(1 << 63), (1 << 63) - 1


def fits(v) -> bool:
    if isinstance(v, bool) or not isinstance(v, int):
        if isinstance(v, (list, tuple)):
            return all(fits(x) for x in v)
        return True
    return I64_MIN <= v <= I64_MAX


@contextlib.contextmanager
def tracking():
    """yields a one-element list; [0] becomes True when a + - * result of the
    reference interpreter leaves int64"""
    from ixverify import oracle as O

    flag = [False]
    orig = O.Interp._binop

    def _binop(self, e, env):
        r = orig(self, e, env)
        if not flag[0] and isinstance(r, int) and not isinstance(r, bool) and not I64_MIN <= r <= I64_MAX:
            flag[0] = True
        return r

    O.Interp._binop = _binop
    try:
        yield flag
    finally:
        O.Interp._binop = orig
