"""GPU: the device precondition checks (csrc/k_contract.cuh via contract.py)
against the reference's own concrete predicates restated in numpy
(oracle.py:478-520 chk_range / chk_mono / chk_inj / chk_bij), and the
executor's use of them: annotated entry points run ELIDED only when their
annotations hold, CHECKED (the reference's answer) otherwise."""

import numpy as np
import pytest

from paper_2506_23058_b200 import gen

pytestmark = pytest.mark.gpu


def _t(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("n", [1, 7, 4096, 100_003, 1 << 22])
@pytest.mark.parametrize("dtype", [np.int32, np.int64, np.uint8])
def test_minmax(cuda, n, dtype):
    from paper_2506_23058_b200 import ops

    lo, hi = (0, 255) if dtype == np.uint8 else (-(1 << 30), 1 << 30)
    xs = gen.uniform(n, n, lo, hi, np.int64).astype(dtype)
    mm = ops.minmax(_t(xs, cuda)).tolist()
    assert mm == [int(xs.min()), int(xs.max())]
    assert ops.minmax(_t(xs[:0], cuda)).tolist() == [(1 << 63) - 1, -(1 << 63)]


@pytest.mark.parametrize("n", [0, 1, 2, 5000, 1 << 20])
def test_mono(cuda, n):
    from paper_2506_23058_b200 import ops

    xs = np.sort(gen.uniform(n + 3, n, -1000, 1000, np.int64))
    for op, f in ((0, np.less_equal), (1, np.less), (2, np.greater_equal), (3, np.greater)):
        want = int(np.count_nonzero(~f(xs[:-1], xs[1:]))) if n > 1 else 0
        assert int(ops.mono_violations(_t(xs, cuda), op).item()) == want


@pytest.mark.parametrize("n", [1, 100, 65_537, 1 << 21])
def test_inj_bij(cuda, n):
    from paper_2506_23058_b200 import ops

    perm = np.random.default_rng(n).permutation(n).astype(np.int64)
    r = ops.inj_check(_t(perm, cuda), 0, n - 1, 0, n - 1).tolist()
    assert r == [n, 0, 0]
    dup = perm.copy()
    dup[n // 2] = dup[0] if n > 1 else dup[0]
    r = ops.inj_check(_t(dup, cuda), 0, n - 1, 0, n - 1).tolist()
    assert r[1] == (1 if n > 1 else 0)
    # values outside [lo, hi] are ignored; outside the image are counted
    shifted = perm - 3
    r = ops.inj_check(_t(shifted, cuda), -3, n - 4, 0, n - 4).tolist()
    assert r == [n, 0, min(3, n)]
    assert ops.inj_check(_t(perm, cuda), 0, 1 << 40, 0, 1) is None  # too wide for a bitmap


def _prog(key):
    import json
    import os

    from paper_2506_23058_b200 import ir

    here = os.path.dirname(os.path.abspath(__file__))
    progs = json.load(open(os.path.join(here, "..", "paper_2506_23058_b200", "data", "programs.json")))
    return ir.from_json(progs[key]["program"])


def _entry_bits(it, fn):
    return [t[3] for t in it.trace if t[0] == "select" and t[1] == fn][0]


def test_csrg_runs_elided_only_under_its_range(cuda):
    """csrg at 2^20 nnz: Range indices holds -> ELIDED bits and the right
    products; one index == num_cols -> CHECKED, OutOfBounds x[c] like the
    reference (a row of corpus/c4_csr_gather.ixl)."""
    import torch

    from paper_2506_23058_b200 import errors
    from paper_2506_23058_b200 import _lib as L
    from paper_2506_23058_b200.executor import Interp

    prog = _prog("own:c4_csr_gather.ixl")
    n, ncols = 1 << 20, 1000
    x = gen.uniform(1, ncols, -99, 99, np.int64)
    v = gen.uniform(2, n, -99, 99, np.int64)
    c = gen.uniform(3, n, 0, ncols - 1, np.int64)
    it = Interp(prog, as_tensors=True)
    got = it.call("csrg", [_t(x, cuda), _t(v, cuda), _t(c, cuda)])
    assert torch.equal(got.cpu(), torch.from_numpy(v * x[c]))
    assert _entry_bits(it, "csrg") == (0,)
    c[n - 7] = ncols
    it = Interp(prog, as_tensors=True)
    with pytest.raises(errors.OutOfBounds) as ei:
        it.call("csrg", [_t(x, cuda), _t(v, cuda), _t(c, cuda)])
    assert ei.value.site == "x[c]"
    assert _entry_bits(it, "csrg") == (L.V_BOUNDS,)
    # the caller's contract: trusted, the ELIDED bits run regardless
    c[n - 7] = 0
    it = Interp(prog, as_tensors=True, preconditions="trust")
    it.call("csrg", [_t(x, cuda), _t(v, cuda), _t(c, cuda)])
    assert _entry_bits(it, "csrg") == (0,) and not [t for t in it.trace if t[0] == "pre"]


def test_sc_bij_checked_when_not_a_bijection(cuda):
    """sc_bij with a permutation: Sc1 (no init, no checks); with a repeated
    index carrying two values: CHECKED -> NonIdempotentScatter."""
    from paper_2506_23058_b200 import errors
    from paper_2506_23058_b200 import _lib as L
    from paper_2506_23058_b200.executor import Interp

    prog = _prog("own:c3_scatter.ixl")
    n = 1 << 18
    perm = np.random.default_rng(5).permutation(n).astype(np.int64)
    vs = gen.uniform(6, n, -50, 50, np.int64)
    it = Interp(prog, as_tensors=True)
    got = it.call("sc_bij", [_t(np.zeros(n, np.int64), cuda), _t(perm, cuda), _t(vs, cuda)]).cpu().numpy()
    want = np.zeros(n, np.int64)
    want[perm] = vs
    assert np.array_equal(got, want) and _entry_bits(it, "sc_bij") == (0,)
    perm[10] = perm[11]
    vs[10], vs[11] = 1, 2
    it = Interp(prog, as_tensors=True)
    with pytest.raises(errors.NonIdempotentScatter):
        it.call("sc_bij", [_t(np.zeros(n, np.int64), cuda), _t(perm, cuda), _t(vs, cuda)])
    assert _entry_bits(it, "sc_bij") == (L.V_CONFLICT | L.V_INIT,)


def test_stripped_kmeans_checks_every_site(cuda):
    """kmeans_ker without its Range annotations (corpus/kmeans_noann.ixl):
    all five sites CHECKED, row = n + 1 raises OutOfBounds(pointers[row])."""
    from paper_2506_23058_b200 import errors
    from paper_2506_23058_b200 import _lib as L
    from paper_2506_23058_b200.executor import Interp

    prog = _prog("own:kmeans_noann.ixl")
    args = [[0, 1, 2], [1.5, 2.5], [0.5, 1.0], [0, 1]]
    it = Interp(prog)
    with pytest.raises(errors.OutOfBounds) as ei:
        it.call("kmeans_ker", [3] + args)
    assert ei.value.site == "pointers[row]"
    assert _entry_bits(it, "kmeans_ker") == (L.V_BOUNDS,) * 5
