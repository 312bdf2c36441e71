"""The drop-in boundary on the GPU: paper_2506_23058_b200.eval_program on
every golden case the Python reference produced (tests/golden/cases.json),
for the verifier-selected variants, the all-CHECKED variants and the generic
combinator path (one kernel per builtin, lambdas through the map VM).
Results, exception classes, OutOfBounds site text and positions must match
the reference exactly."""

import json
import os

import pytest

from paper_2506_23058_b200 import errors, ir
from paper_2506_23058_b200 import select as sel

from test_oracle_golden import CASES, dec

import bigtrack

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
PROGRAMS = json.load(open(os.path.join(HERE, "..", "paper_2506_23058_b200", "data", "programs.json")))
_CACHE = {}

GENERIC_UNSUPPORTED = set()  # kmeans_ker: the function-level loop compiles to a one-thread kernel


def program(key):
    if key not in _CACHE:
        _CACHE[key] = ir.from_json(PROGRAMS[key]["program"])
    return _CACHE[key]


def _same(got, want):
    if isinstance(want, float) or isinstance(got, float):
        return float(got).hex() == float(want).hex()
    if isinstance(want, (list, tuple)) and isinstance(got, (list, tuple)):
        return len(got) == len(want) and all(_same(g, w) for g, w in zip(got, want))
    return got == want


def expected_entry_bits(prog, fun, mode, pre):
    """The variant bits the executor must run the entry function's sites
    with: the verifier's (frozen, closure-keyed) verdicts in selected mode
    when the reference's own predicates say the annotations hold
    (cases.json "pre", make_golden.ref_pre_holds), else every check."""
    f = ir.find_def(prog, fun)
    chk = sel.checked_selection(f)
    if mode == "checked":
        return tuple(s.bits for s in chk.sites)
    fs = sel.selection_for(prog, f)
    if pre is False and fs.elides:
        return tuple(s.bits for s in chk.sites)
    return tuple(s.bits for s in fs.sites)


@pytest.mark.parametrize("mode", ["selected", "checked", "generic"])
@pytest.mark.parametrize("idx", range(len(CASES)))
def test_eval_program_matches_reference(cuda, idx, mode):
    """Every golden case in every mode -- including inputs that violate the
    annotations the verifier relied on: selected mode checks them on the
    device and runs CHECKED, so it must raise / answer exactly like the
    reference -- and the variant bits actually used for the entry function's
    sites are asserted, not just the values."""
    from paper_2506_23058_b200.executor import Interp

    case = CASES[idx]
    if mode == "generic" and case["fun"] in GENERIC_UNSUPPORTED:
        pytest.skip("loop body: pipeline only")
    prog = program(case["program"])
    args = dec(case["args"])
    kw = {"variant": "checked" if mode == "checked" else "selected", "generic_only": mode == "generic"}
    if "error" in case and mode == "generic":
        kw["variant"] = "checked"  # generic path with the reference's own checks
    it = Interp(prog, case.get("budget", 10**6), **kw)
    if case.get("big"):
        # the reference held an integer outside int64 (tests/golden/bigtrack.py):
        # IntegerOverflow -- mandatory when a result does not fit -- or its answer
        try:
            got = it.call(case["fun"], args)
        except errors.IntegerOverflow:
            return
        except errors.OracleError as ex:
            assert "error" in case and type(ex).__name__ == case["error"], ex
            return
        want = dec(case["result"])
        assert "result" in case and bigtrack.fits(want) and _same(got, want), (got, case)
        return
    if "error" in case:
        cls = getattr(errors, case["error"])
        with pytest.raises(cls) as ei:
            it.call(case["fun"], args)
        if "site" in case:
            assert ei.value.site == case["site"]
        if "pos" in case:
            assert list(ei.value.pos) == case["pos"]
    else:
        got = it.call(case["fun"], args)
        want = dec(case["result"])
        assert _same(got, want), (got, want)
    used = [t[3] for t in it.trace if t[0] == "select" and t[1] == case["fun"]]
    if used and ir.sites(ir.find_def(prog, case["fun"])):
        assert used[0] == expected_entry_bits(prog, case["fun"], kw["variant"], case.get("pre")), it.trace


def test_opaque_callable_rejected(cuda):
    from paper_2506_23058_b200.executor import eval_program

    prog = program("ref:filter.ixl")
    with pytest.raises(TypeError):
        eval_program(prog, "filter", [lambda x: x < 3, [1, 2, 5]])


@pytest.mark.parametrize("m", [1, 1000, 40_000])
def test_partition2l_pipeline_large(cuda, m):
    """partition2L's registered pipeline at up to ~1.2M elements against the
    C restatement (oracle/ixoracle.c ixo_partition2l)."""
    import numpy as np

    from oracle import ixoracle as O
    from paper_2506_23058_b200 import gen
    from paper_2506_23058_b200.executor import eval_program

    prog = ir.from_json(PROGRAMS["own:partition2l.ixl"]["program"])
    shp = gen.uniform(m, m, 0, 60, np.int64)
    shp[::5] = 0
    n = int(shp.sum())
    cs = gen.uniform(m + 1, n, 0, 2, np.int64) == 0
    xs = gen.uniform(m + 2, n, -1000, 1000, np.int64)
    want = O.partition2l(shp, cs.astype(np.int64), xs)
    got = eval_program(prog, "partition2L", [shp.tolist(), cs.tolist(), xs.tolist()], as_tensors=True)
    assert np.array_equal(got.cpu().numpy(), want)


@pytest.mark.parametrize("mode", ["selected", "checked", "generic"])
def test_drop_in_at_scale(cuda, mode):
    """The drop-in eval_program on the reference's own corpus at 2^22 int64
    elements (device tensors in, device tensors out), every execution mode
    against the C restatement: partition2, filter, partition3, C2."""
    import numpy as np
    import torch

    from oracle import ixoracle as O
    from paper_2506_23058_b200 import gen
    from paper_2506_23058_b200.executor import eval_program
    from paper_2506_23058_b200.pred import Pred

    n = 1 << 22
    xs_h = gen.uniform(41, n, -(1 << 40), 1 << 40, np.int64)
    xs = torch.from_numpy(xs_h).to(cuda)
    kw = {"variant": "checked" if mode == "checked" else "selected", "generic_only": mode == "generic",
          "as_tensors": True}
    p, q = Pred.lt(0), Pred.hash(0xC0FFEE)
    nt, ys = eval_program(program("ref:partition2.ixl"), "partition2", [p, xs], **kw)
    wnt, wys = O.partition2(p, xs_h)
    assert nt == wnt and np.array_equal(ys.cpu().numpy(), wys)
    ys = eval_program(program("ref:filter.ixl"), "filter", [q, xs], **kw)
    assert np.array_equal(ys.cpu().numpy(), O.filter_(q, xs_h))
    m1, m2, ys = eval_program(program("ref:partition3.ixl"), "partition3", [p, q, xs], **kw)
    w1, w2, wys = O.partition3(p, q, xs_h)
    assert (m1, m2) == (w1, w2) and np.array_equal(ys.cpu().numpy(), wys)
    small = gen.uniform(42, n, -128, 127, np.int64)
    k = int(np.count_nonzero(small >= 0))
    shape = gen.segment_shape(43, 1 << 14, k)
    ys, zs = eval_program(program("own:c2_filter_sgmsum.ixl"), "c2",
                          [Pred.ge(0), torch.from_numpy(small).to(cuda), torch.from_numpy(shape).to(cuda)], **kw)
    wys, wzs = O.c2(Pred.ge(0), small, shape)
    assert np.array_equal(ys.cpu().numpy(), wys) and np.array_equal(zs.cpu().numpy(), wzs)
