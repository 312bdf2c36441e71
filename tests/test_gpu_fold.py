"""scan / hist with generic operators (jit_fold.py) beyond the golden sizes:
the tiled parallel scan against numpy and against the in-order device fold
at sizes with many tiles, and the CAS hist against the in-order hist.  The
small-size parity with the reference interpreter itself is the golden replay
(test_gpu_executor.py over corpus/scanops.ixl)."""

import json
import os

import numpy as np
import pytest

from oracle import ixoracle as O
from paper_2506_23058_b200 import ir
from paper_2506_23058_b200 import gen

pytestmark = pytest.mark.gpu

V = ir.VarE


def lam(params, body):
    return ir.Lambda(tuple(params), body)


MIN = lam("ab", ir.If(ir.BinOp("<", V("a"), V("b")), V("a"), V("b")))
MAX = lam("ab", ir.If(ir.BinOp(">=", V("b"), V("a")), V("b"), V("a")))
MUL = lam("ab", ir.BinOp("*", V("a"), V("b")))
AND = lam("ab", ir.BinOp("&&", V("a"), V("b")))
PAIR = lam(("a1", "a2", "b1", "b2"),
           ir.TupleE((ir.BinOp("+", V("a1"), V("b1")), ir.If(ir.BinOp(">", V("a2"), V("b2")), V("a2"), V("b2")))))
SEGMIN = lam(("f1", "v1", "f2", "v2"),
             ir.TupleE((ir.BinOp("||", V("f1"), V("f2")),
                        ir.If(V("f2"), V("v2"), ir.If(ir.BinOp("<=", V("v1"), V("v2")), V("v1"), V("v2"))))))
CLIP = lam("ab", ir.If(ir.BinOp(">", V("a"), ir.Const(20)), V("b"), ir.BinOp("+", V("a"), V("b"))))
HORNER = lam("ab", ir.BinOp("+", ir.BinOp("*", V("a"), ir.Const(3)), V("b")))
LAST = lam("ab", V("b"))

SIZES = [1, 255, 2049, (1 << 20) + 3, 3 << 21]


def _scan(cuda, op, nes, arrs, force_seq=False):
    import torch

    from paper_2506_23058_b200 import jit_fold, ops

    st = ops.Status(cuda)
    ts = [torch.from_numpy(a).to(cuda) for a in arrs]
    outs, sites, par = jit_fold.scan(op, nes, ts, {}, lambda node: 0, st, device=cuda, force_seq=force_seq)
    assert st.read().ok
    return [o.cpu().numpy() for o in outs], par


@pytest.mark.parametrize("n", SIZES)
def test_parallel_scans_vs_numpy(cuda, n):
    xs = gen.uniform(n, n, -(1 << 40), 1 << 40, np.int64)
    (got,), par = _scan(cuda, MIN, [7], [xs])
    assert par and np.array_equal(got, np.minimum.accumulate(np.concatenate([[7], xs]))[1:])
    (got,), _ = _scan(cuda, MAX, [-(1 << 50)], [xs])
    assert np.array_equal(got, np.maximum.accumulate(xs))
    sg = np.where(gen.uniform(n + 1, n, 0, 9, np.int64) == 0, -1, 1).astype(np.int64)
    (got,), _ = _scan(cuda, MUL, [3], [sg])
    assert np.array_equal(got, 3 * np.cumprod(sg))
    cs = (gen.uniform(n + 2, n, 0, 5000, np.int64) != 0).astype(np.uint8)
    (got,), _ = _scan(cuda, AND, [1], [cs])
    assert np.array_equal(got, np.logical_and.accumulate(cs.astype(bool)).astype(np.int64))
    ys = gen.uniform(n + 3, n, -1000, 1000, np.int64)
    (g1, g2), _ = _scan(cuda, PAIR, [3, -100], [xs, ys])
    assert np.array_equal(g1, 3 + np.cumsum(xs))
    assert np.array_equal(g2, np.maximum.accumulate(np.concatenate([[-100], ys]))[1:])


@pytest.mark.parametrize("n", [1, 4097, 1 << 16])
def test_parallel_matches_inorder_fold(cuda, n):
    """The tiled scan and the in-order device fold agree, and both agree
    with the reference's fold restated (oracle fold_scan) where that is
    cheap; covers the segmented lift with a non-(+) operator."""
    fs = (gen.uniform(n, n, 0, 6, np.int64) == 0).astype(np.uint8)
    xs = gen.uniform(n + 1, n, -500, 500, np.int64)
    par, p1 = _scan(cuda, SEGMIN, [0, 9], [fs, xs])
    seq, p2 = _scan(cuda, SEGMIN, [0, 9], [fs, xs], force_seq=True)
    assert p1 and not p2
    assert np.array_equal(par[0], seq[0]) and np.array_equal(par[1], seq[1])
    want = O.fold_scan(lambda f1, v1, f2, v2: (int(bool(f1) or bool(f2)), v2 if f2 else (v1 if v1 <= v2 else v2)),
                       [0, 9], [fs.tolist(), xs.tolist()])
    assert par[0].tolist() == want[0] and par[1].tolist() == want[1]


@pytest.mark.parametrize("n", [0, 5, 1025, 1 << 16])
def test_inorder_fold_non_associative(cuda, n):
    xs = gen.uniform(n + 7, n, -9, 9, np.int64)
    (got,), par = _scan(cuda, CLIP, [0], [xs])
    assert not par
    assert got.tolist() == O.fold_scan(lambda a, b: b if a > 20 else a + b, [0], [xs.tolist()])


def _hist(cuda, op, ne, dlen, is_, vs, force_seq=False):
    import torch

    from paper_2506_23058_b200 import jit_fold, ops

    st = ops.Status(cuda)
    dst, _, kind = jit_fold.hist(op, ne, dlen, torch.from_numpy(is_).to(cuda), torch.from_numpy(vs).to(cuda), {},
                                 lambda node: 0, st, force_seq=force_seq)
    assert st.read().ok
    return dst.cpu().numpy(), kind


@pytest.mark.parametrize("m", [1, 1000, 1 << 20])
def test_hist_cas_and_inorder(cuda, m):
    dlen = max(1, m // 8)
    is_ = gen.uniform(m, m, -3, dlen + 3, np.int64)
    vs = np.where(gen.uniform(m + 1, m, 0, 3, np.int64) == 0, -1, 1).astype(np.int64)
    cas, k1 = _hist(cuda, MUL, 5, dlen, is_, vs)
    seq, k2 = _hist(cuda, MUL, 5, dlen, is_, vs, force_seq=True)
    assert (k1, k2) == ("cas", "seq") and np.array_equal(cas, seq)
    ok = (is_ >= 0) & (is_ < dlen)
    neg = np.bincount(is_[ok & (vs < 0)], minlength=dlen)[:dlen]
    assert np.array_equal(cas, 5 * np.where(neg % 2 == 1, -1, 1))
    # order-dependent operators: the in-order fold against the reference's fold
    small = min(m, 1 << 14)
    v2 = gen.uniform(m + 2, small, -3, 3, np.int64)
    for op, f in ((LAST, lambda a, b: b), (HORNER, lambda a, b: a * 3 + b)):
        got, kind = _hist(cuda, op, 0, 4 * dlen, is_[:small], v2)
        assert kind == "seq"
        assert got.tolist() == O.fold_hist(f, 0, 4 * dlen, is_[:small].tolist(), v2.tolist())


def test_never_ending_loop_fails_fast(cuda):
    """A while loop that never ends, mapped over many elements, stops at the
    step budget for the whole launch (the shared counter), not after
    budget x elements iterations."""
    import time

    from paper_2506_23058_b200 import errors
    from paper_2506_23058_b200.executor import eval_program

    prog = ir.from_json(json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                    "paper_2506_23058_b200", "data", "programs.json")))
                        ["own:kmeans_rows.ixl"]["program"])
    xs = [-1] * (1 << 16)  # every element loops forever
    t0 = time.time()
    with pytest.raises(errors.StepBudgetExceeded):
        eval_program(prog, "countdown", [xs], step_budget=10**6, variant="checked")
    assert time.time() - t0 < 30
