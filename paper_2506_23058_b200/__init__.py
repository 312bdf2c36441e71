"""paper_2506_23058_b200 -- B200 (sm_100a) execution path for the
index-array combinators of arXiv 2506.23058 (reference: ``ixverify``).

``eval_program`` keeps the signature of ``ixverify.oracle.eval_program``
(/root/reference/pkg/src/ixverify/oracle.py:332) and runs the program's
combinators as CUDA kernels (libixgpu.so), choosing per source site the
CHECKED or ELIDED kernel variant from the reference verifier's obligations.
"""

from .pred import Pred  # noqa: F401


def __getattr__(name):
    # lazy: importing the package must not require torch or a GPU
    if name in ("eval_program", "Interp"):
        from . import executor

        return getattr(executor, name)
    if name == "select":
        from .select import select

        return select
    raise AttributeError(name)


__all__ = ["Pred", "eval_program", "Interp", "select"]
