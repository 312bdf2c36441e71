"""The reference interpreter's exception classes (oracle.py:51-77).

When ``ixverify`` is importable the executor raises the reference's own
classes, so callers that catch ``ixverify.oracle.OutOfBounds`` keep working
unchanged (drop-in).  Otherwise classes with the same names, constructor
signatures, messages and attributes are defined here.
"""

from __future__ import annotations

import os
import sys

_REF = os.environ.get("IXVERIFY_SRC", "/root/reference/pkg/src")


def _load_reference():
    try:
        if os.path.isdir(_REF) and _REF not in sys.path:
            sys.path.insert(0, _REF)
        from ixverify import oracle as _o  # noqa: F401

        return _o
    except Exception:
        return None


_ref = _load_reference()

if _ref is not None:
    OracleError = _ref.OracleError
    OutOfBounds = _ref.OutOfBounds
    NonIdempotentScatter = _ref.NonIdempotentScatter
    StepBudgetExceeded = _ref.StepBudgetExceeded
    UnboundFree = _ref.UnboundFree
    REFERENCE_CLASSES = True
else:
    REFERENCE_CLASSES = False

    class OracleError(Exception):
        pass

    class OutOfBounds(OracleError):
        def __init__(self, site, pos=None):
            super().__init__(f"out of bounds: {site}")
            self.site = site
            self.pos = pos

    class NonIdempotentScatter(OracleError):
        def __init__(self, pos=None):
            super().__init__("scatter writes conflicting values to one index")
            self.pos = pos

    class StepBudgetExceeded(OracleError):
        pass

    class UnboundFree(OracleError):
        pass


class NarrowingOverflow(OracleError):
    """A result did not fit the i32 storage the caller asked for (the
    reference's ints are unbounded; raise rather than return a wrapped value)."""


class IntegerOverflow(OracleError):
    """An integer value left int64.  The reference's ints are unbounded
    (oracle.py:214-240: a scan of [2^62, 2^62, 2^62] returns 3 * 2^62); the
    device computes in int64 and checks every result exactly, so instead of
    returning a wrapped value the executor raises this at the first element
    (in the reference's order) whose value does not fit."""

    def __init__(self, what: str = "", elem=None):
        super().__init__(f"integer overflow: a value left int64{': ' + what if what else ''}")
        self.elem = elem
