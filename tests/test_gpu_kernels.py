"""GPU parity: every libixgpu.so entry point against the CPU oracle
(oracle/ixoracle.c, itself pinned to the Python reference by
tests/test_oracle_golden.py) on the same seeded inputs.  Integer work, so
the bar is bit-exact."""

import numpy as np
import pytest

from oracle import ixoracle as O
from paper_2506_23058_b200 import _lib as L
from paper_2506_23058_b200 import gen
from paper_2506_23058_b200.pred import Pred

pytestmark = pytest.mark.gpu

SIZES = [0, 1, 5, 4095, 4096, 4097, 12_345, 300_001]
VARIANTS = [L.VARIANT_ELIDED, L.VARIANT_CHECKED]
PREDS = [Pred.lt(0), Pred.ge(3), Pred.hash(0xABCDEF), Pred(7)]  # 7 = TRUE


def _t(a, dev):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


def _np(t):
    return t.cpu().numpy()


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("variant", VARIANTS)
def test_partition2(cuda, n, dtype, variant):
    from paper_2506_23058_b200 import ops

    xs = gen.uniform(n + 1, n, -50, 50, dtype)
    for p in PREDS:
        nt, ys = O.partition2(p, xs)
        st = ops.Status(cuda)
        gys, dnt = ops.partition2(_t(xs, cuda), p, variant, st)
        assert int(dnt.item()) == nt
        assert np.array_equal(_np(gys).astype(np.int64), ys)
        assert st.read().ok


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("variant", VARIANTS)
def test_partition3(cuda, n, dtype, variant):
    from paper_2506_23058_b200 import ops

    xs = gen.uniform(n + 2, n, -50, 50, dtype)
    p, q = Pred.lt(-10), Pred.hash(99)
    m1, m2, ys = O.partition3(p, q, xs)
    st = ops.Status(cuda)
    gys, dm = ops.partition3(_t(xs, cuda), p, q, variant, st)
    assert _np(dm).tolist() == [m1, m2]
    assert np.array_equal(_np(gys).astype(np.int64), ys)
    assert st.read().ok


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
@pytest.mark.parametrize("variant", VARIANTS)
def test_filter(cuda, n, dtype, variant):
    from paper_2506_23058_b200 import ops

    xs = gen.uniform(n + 3, n, -1000, 1000, dtype)
    for p in PREDS:
        want = O.filter_(p, xs)
        st = ops.Status(cuda)
        gys, dk = ops.filter(_t(xs, cuda), p, variant, st)
        k = int(dk.item())
        assert k == len(want)
        assert np.array_equal(_np(gys)[:k].astype(np.int64), want)
        assert st.read().ok
    cs = (gen.uniform(n + 4, n, 0, 3, np.int64) == 0).astype(np.uint8)
    want = O.filter_by(cs, xs)
    st = ops.Status(cuda)
    gys, dk = ops.filter_by(_t(cs, cuda), _t(xs, cuda), variant, st)
    k = int(dk.item())
    assert np.array_equal(_np(gys)[:k].astype(np.int64), want)


EDGE_THR = [-(1 << 63), -(1 << 31) - 1, -(1 << 31), -1, 0, 1, (1 << 31) - 1, 1 << 31, (1 << 63) - 1]


@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_filter_pred_edges(cuda, dtype):
    """comparison predicates with thresholds at and beyond the element
    type's range (the kernels test them as a clamped interval in T's width)."""
    from paper_2506_23058_b200 import ops
    from paper_2506_23058_b200 import pred as P

    n = 100_000  # several full tiles + a ragged one
    info = np.iinfo(dtype)
    xs = gen.uniform(77, n, int(info.min), int(info.max), dtype)
    xs[:12] = [info.min, info.min + 1, -2, -1, 0, 1, 2, info.max - 1, info.max, -(1 << 31), (1 << 31) - 1, 0]
    for kind in (P.LT, P.GT, P.LE, P.GE, P.EQ, P.NE):
        for thr in EDGE_THR + [int(xs[500]), int(info.min), int(info.max)]:
            p = Pred(kind, thr)
            want = O.filter_(p, xs)
            st = ops.Status(cuda)
            gys, dk = ops.filter(_t(xs, cuda), p, L.VARIANT_ELIDED, st)
            k = int(dk.item())
            assert k == len(want), (kind, thr)
            assert np.array_equal(_np(gys)[:k].astype(np.int64), want), (kind, thr)
            nt, ys = O.partition2(p, xs)
            gys, dnt = ops.partition2(_t(xs, cuda), p, L.VARIANT_ELIDED, st)
            assert int(dnt.item()) == nt and np.array_equal(_np(gys).astype(np.int64), ys), (kind, thr)


@pytest.mark.parametrize("head", [-(1 << 20), 0])
def test_c2_narrow_exact(cuda, head):
    """int32 zs: NARROW is raised iff an exact sgmSum value leaves int32.  A
    segment crossing a tile boundary whose tile-local prefix overflows while
    the exact value (with the preceding tile's carry) stays in range must
    not raise it (head < 0); with no negative head it must (head = 0)."""
    import torch

    from paper_2506_23058_b200 import ops

    tile = 3 * 8192  # a multiple of the k_filter_b<int32> tile (12288 or 24576 elements)
    n = 3 * tile + 100
    xs = np.zeros(n, np.int32)
    xs[:2047] = head
    xs[tile:tile + 2100] = 1 << 20
    shape = np.array([30_000, n - 30_000], np.int64)
    want_ys, want_zs = O.c2(Pred(7), xs, shape)
    st = ops.Status(cuda)
    ys, zs, dk = ops.c2(_t(xs, cuda), Pred(7), _t(shape, cuda), L.VARIANT_ELIDED, st, z_dtype=torch.int32)
    s = st.read()
    assert s.ok
    overflow = bool(np.any(want_zs != want_zs.astype(np.int32)))
    assert overflow == (head == 0)
    assert s.narrow == overflow
    if not overflow:
        assert np.array_equal(_np(zs).astype(np.int64), want_zs)


@pytest.mark.parametrize("n", SIZES + [1 << 21])
@pytest.mark.parametrize("zdt", ["i32", "i64"])
@pytest.mark.parametrize("variant", VARIANTS + [0x2000])  # 0x2000: only mkFlags' conflict check on
def test_c2(cuda, n, zdt, variant):
    import torch

    from paper_2506_23058_b200 import ops

    xs = gen.uniform(n + 5, n, -128, 127, np.int32)
    p = Pred.ge(0)
    k = int((xs >= 0).sum())
    for m in (0, 1, 7, 1000):
        shape = gen.segment_shape(m + n, m, k) if m else np.zeros(0, np.int64)
        want_ys, want_zs = O.c2(p, xs, shape)
        st = ops.Status(cuda)
        zt = torch.int32 if zdt == "i32" else torch.int64
        ys, zs, dk = ops.c2(_t(xs, cuda), p, _t(shape, cuda), variant, st, z_dtype=zt)
        kk = int(dk.item())
        assert kk == len(want_ys)
        assert np.array_equal(_np(ys)[:kk].astype(np.int64), want_ys)
        assert np.array_equal(_np(zs)[:kk].astype(np.int64), want_zs)
        assert st.read().ok


def test_c2_sum_below_k(cuda):
    """shape sums to less / more than k: flags past k are dropped (OOB)."""
    from paper_2506_23058_b200 import ops

    n = 20_000
    xs = gen.uniform(11, n, -128, 127, np.int32)
    p = Pred.ge(0)
    k = int((xs >= 0).sum())
    for tot in (k // 2, 3 * k):
        shape = gen.segment_shape(12, 100, tot)
        want_ys, want_zs = O.c2(p, xs, shape)
        for variant in VARIANTS:
            st = ops.Status(cuda)
            ys, zs, dk = ops.c2(_t(xs, cuda), p, _t(shape, cuda), variant, st)
            kk = int(dk.item())
            assert np.array_equal(_np(zs)[:kk].astype(np.int64), want_zs)


def test_c2_shape_prefix_past_int64(cuda):
    """A segment shape whose running sum leaves int64 (the reference's ints
    are unbounded, its starts past n are simply dropped): the ELIDED mkFlags
    scan (and the CHECKED pipeline's materialised starts) record IXG_OVERFLOW
    instead of setting a flag at a wrapped start."""
    from paper_2506_23058_b200 import ops

    n = 10_000
    xs = gen.uniform(17, n, -128, 127, np.int32)
    shape = np.array([5, 1 << 62, 1 << 62, 3, 7], np.int64)
    for variant in VARIANTS:
        st = ops.Status(cuda)
        ops.c2(_t(xs, cuda), Pred.ge(0), _t(shape, cuda), variant, st)
        s = st.read()
        assert not s.ok and s.codes & (1 << L.OVERFLOW), variant


def _flag_bits_ref(shape, nbits):
    """mkFlags as a bitmap: bit scn[i] for every shape[i] > 0 whose start
    scn[i] (exclusive prefix of shape) lies in [0, nbits)."""
    scn = np.concatenate([[0], np.cumsum(shape)[:-1]]).astype(np.int64) if len(shape) else np.zeros(0, np.int64)
    words = np.zeros((nbits + 31) // 32 + 1, np.uint32)
    for s_, st_ in zip(shape, scn):
        if s_ > 0 and 0 <= st_ < nbits:
            words[st_ >> 5] |= np.uint32(1 << (int(st_) & 31))
    return words[: (nbits + 31) // 32]


@pytest.mark.parametrize("m", [0, 1, 7, 4095, 4096, 4097, 12_345, 300_001])
@pytest.mark.parametrize("kind", ["segments", "unit", "negatives", "past_nbits"])
@pytest.mark.parametrize("on_device", [False, True])
def test_flag_bitmap(cuda, m, kind, on_device):
    """ixg_flag_bitmap (the C2 mkFlags: bitmap clear + big-tile scan) against
    the definition, with empty and negative segments (starts that move
    backwards), starts at or past nbits, and nbits read from the device."""
    import torch

    from paper_2506_23058_b200 import ops

    rng = np.random.default_rng(m + len(kind))
    if kind == "unit":
        shape = np.ones(m, np.int64)
    elif kind == "negatives":
        shape = rng.integers(-3, 9, m).astype(np.int64)
    else:
        shape = rng.integers(0, 6, m).astype(np.int64)
    total = int(shape[shape > 0].sum()) if m else 0
    nbits = max(1, total // 2) if kind == "past_nbits" else total + 70
    cap = nbits + 4096 if on_device else nbits
    d_nbits = torch.tensor([nbits], dtype=torch.int64, device=cuda) if on_device else None
    bits = torch.full((int(ops._lib().ixg_bitmap_words(cap)),), -1, dtype=torch.int32, device=cuda)  # stale words
    ops.flag_bitmap(_t(shape, cuda), cap, d_nbits=d_nbits, bits=bits)
    got = _np(bits).view(np.uint32)[: (nbits + 31) // 32].copy()
    if nbits % 32:
        got[-1] &= np.uint32((1 << (nbits % 32)) - 1)
    assert np.array_equal(got, _flag_bits_ref(shape, nbits))


@pytest.mark.parametrize("m", [1, 7, 4097, 300_001])
@pytest.mark.parametrize("kind", ["segments", "unit", "negatives"])
@pytest.mark.parametrize("win", [(0, 1000), (37, 5000), (100_003, 77_777), (10 ** 9, 64)])
def test_flag_bitmap_window(cuda, m, kind, win):
    """ixg_flag_bitmap_window (a shard's window of mkFlags: the sharded C2
    step): bit j = the flag of global position lo + j, j < nb (nb on the
    device), the rest of the buffer's words cleared."""
    import torch

    from paper_2506_23058_b200 import ops

    rng = np.random.default_rng(m + 3 * len(kind))
    if kind == "unit":
        shape = np.ones(m, np.int64)
    elif kind == "negatives":
        shape = rng.integers(-3, 9, m).astype(np.int64)
    else:
        shape = rng.integers(0, 6, m).astype(np.int64)
    lo, nb = win
    full = _flag_bits_ref(shape, lo + nb)
    want = np.array([(full[(lo + j) >> 5] >> np.uint32((lo + j) & 31)) & 1 for j in range(nb)], np.uint32)
    cap = nb + 4096
    bits = torch.full((int(ops._lib().ixg_bitmap_words(cap)),), -1, dtype=torch.int32, device=cuda)  # stale words
    ops.flag_bitmap(_t(shape, cuda), cap, d_nbits=torch.tensor([nb], dtype=torch.int64, device=cuda), bits=bits,
                    d_lo=torch.tensor([lo], dtype=torch.int64, device=cuda))
    got_w = _np(bits).view(np.uint32)
    got = np.array([(got_w[j >> 5] >> np.uint32(j & 31)) & 1 for j in range(nb)], np.uint32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("n", SIZES)
def test_scan_add(cuda, n):
    from paper_2506_23058_b200 import ops

    for dtype in (np.int32, np.int64, np.uint8):
        xs = gen.uniform(n, n, 0, 200, np.int64).astype(dtype)
        for ne in (0, 5, -7):
            want = O.scan_add(xs, ne)
            got = _np(ops.scan_add(_t(xs, cuda), ne))
            assert np.array_equal(got, want)
            got = _np(ops.scan_add(_t(xs, cuda), ne, exclusive=True))
            assert np.array_equal(got, want - xs.astype(np.int64))


@pytest.mark.parametrize("n", SIZES)
def test_segscan(cuda, n):
    from paper_2506_23058_b200 import ops

    flags = (gen.uniform(n + 9, n, 0, 9, np.int64) == 0).astype(np.uint8)
    xs = gen.uniform(n + 10, n, -100, 100, np.int64)
    want = O.sgmsum(flags, xs)
    assert np.array_equal(_np(ops.segscan_add(_t(flags, cuda), _t(xs, cuda))), want)


@pytest.mark.parametrize("case", ["local_overflow_carried_back", "overflow", "wide_carry_flag_first",
                                  "wide_carry_no_flag", "random"])
def test_segsum_int32_narrow_exact(cuda, case):
    """ixg_segsum int32 -> int32 (the sharded C2 sgmSum): values exact, and
    NARROW iff an exact value (the carry of earlier shards included) leaves
    int32 -- the kernel carries the run in 32 bits from an in-range start
    and in 64 bits from a start outside int32."""
    import torch

    from paper_2506_23058_b200 import ops

    tile = 12288
    n = 3 * tile + 100
    xs = np.zeros(n, np.int32)
    starts = [0, 30_000]
    carry_v, carry_f = 0, False
    if case == "local_overflow_carried_back":  # a tile-local prefix past int32, the exact value back in range
        xs[:2047] = -(1 << 20)
        xs[tile:tile + 2100] = 1 << 20
    elif case == "overflow":
        xs[tile:tile + 2100] = 1 << 20
    elif case == "wide_carry_flag_first":  # an earlier shard's carry outside int32, a flag at 0 resets it
        carry_v, carry_f = 1 << 33, True
        xs[:] = gen.uniform(3, n, -1000, 1000, np.int32)
    elif case == "wide_carry_no_flag":  # the same carry reaches the first elements: NARROW
        carry_v, carry_f = 1 << 33, True
        starts = [30_000]
        xs[:] = gen.uniform(4, n, -1000, 1000, np.int32)
    else:
        xs[:] = gen.uniform(5, n, -(1 << 31), (1 << 31) - 1, np.int32)
        carry_v, carry_f = -(1 << 31), True
        starts = sorted(set([0] + list(gen.uniform(6, 400, 1, n - 1, np.int64))))
    # this array's flags start `base` bits into the mkFlags bitmap (a shard
    # that begins inside a segment: no flag at its position 0)
    base = 5 if case == "wide_carry_no_flag" else 0
    gstarts = [0] + [q + base for q in starts if q + base > 0]
    shape = np.diff(np.array(gstarts + [n + base], np.int64))
    flags = np.zeros(n, bool)
    flags[np.array([q - base for q in gstarts if q >= base])] = True
    want = np.zeros(n, np.int64)
    run = carry_v
    for i in range(n):  # segmented inclusive sum after the carry, in Python ints
        run = int(xs[i]) if flags[i] else run + int(xs[i])
        want[i] = run
    overflow = bool(np.any((want < -(1 << 31)) | (want > (1 << 31) - 1)))
    bits = ops.flag_bitmap(_t(shape, cuda), n + base)
    zs = torch.empty(n, dtype=torch.int32, device=cuda)
    tot = torch.empty(2, dtype=torch.int64, device=cuda)
    st = ops.Status(cuda)
    ops.segsum(_t(xs, cuda), n, bits, base, zs, carry_v, carry_f, tot, st)
    s = st.read()
    assert s.narrow == overflow, case
    if case in ("local_overflow_carried_back", "wide_carry_flag_first"):
        assert not overflow
    if case in ("overflow", "wide_carry_no_flag"):
        assert overflow
    if not overflow:
        assert np.array_equal(_np(zs).astype(np.int64), want), case


@pytest.mark.parametrize("n", [0, 1, 1000, 1 << 20])
def test_scatter_perm(cuda, n):
    """Injective scatter (a partition2 permutation): all variants agree."""
    from paper_2506_23058_b200 import ops

    xs = gen.uniform(21, n, -(1 << 31), (1 << 31) - 1, np.int64)
    is_ = np.argsort(np.argsort(xs, kind="stable"), kind="stable").astype(np.int64)
    vs = gen.uniform(22, n, -1000, 1000, np.int64)
    dst = np.zeros(n, np.int64)
    want = O.scatter(dst, is_, vs)
    for bits in (0, L.V_INIT, L.V_CONFLICT | L.V_INIT):
        st = ops.Status(cuda)
        out = _t(dst, cuda).clone()
        ops.scatter(out, _t(is_, cuda), _t(vs, cuda), bits, st)
        assert np.array_equal(_np(out), want)
        assert st.read().ok


def test_scatter_semantics(cuda):
    """Appendix A of SURVEY.md: zip truncation, OOB ignore, equal dups, conflicts."""
    from paper_2506_23058_b200 import ops

    cases = [
        ([0, 0, 0], [0, 1, 2], [7, 8], [7, 8, 0]),
        ([0, 0, 0], [-1, 3, 2, 100], [5, 6, 9, 1], [0, 0, 9]),
        ([0, 0, 0], [1, 1], [5, 5], [0, 5, 0]),
        ([0, 0], [5, 5], [1, 2], [0, 0]),  # conflicting but out of bounds
    ]
    for dst, is_, vs, want in cases:
        st = ops.Status(cuda)
        out = _t(np.array(dst, np.int64), cuda)
        ops.scatter(out, _t(np.array(is_, np.int64), cuda), _t(np.array(vs, np.int64), cuda),
                    L.V_CONFLICT | L.V_INIT, st, stmt=0, site=3)
        assert _np(out).tolist() == want
        assert st.read().ok
    st = ops.Status(cuda)
    out = _t(np.zeros(4, np.int64), cuda)
    ops.scatter(out, _t(np.array([0, 2, 0], np.int64), cuda), _t(np.array([1, 2, 3], np.int64), cuda),
                L.V_CONFLICT | L.V_INIT, st, stmt=0, site=3)
    s = st.read()
    assert not s.ok and s.codes & (1 << L.CONFLICT) and s.site == 3
    # large random scatter with one injected conflict
    n = 1 << 20
    is_ = np.random.default_rng(0).permutation(n).astype(np.int64)
    vs = np.arange(n, dtype=np.int64)
    is_[n // 2] = is_[n // 3]
    st = ops.Status(cuda)
    out = _t(np.zeros(n, np.int64), cuda)
    ops.scatter(out, _t(is_, cuda), _t(vs, cuda), L.V_CONFLICT | L.V_INIT, st)
    assert not st.read().ok
    # same duplicate, equal values: no conflict, same result as the oracle
    vs2 = vs.copy()
    vs2[n // 2] = vs2[n // 3]
    st = ops.Status(cuda)
    out = _t(np.zeros(n, np.int64), cuda)
    ops.scatter(out, _t(is_, cuda), _t(vs2, cuda), L.V_CONFLICT | L.V_INIT, st)
    assert st.read().ok
    assert np.array_equal(_np(out), O.scatter(np.zeros(n, np.int64), is_, vs2))


def test_gather_checked(cuda):
    from paper_2506_23058_b200 import ops

    arr = np.arange(10, dtype=np.int64) * 3
    idx = np.array([0, 9, 4, 10, 2, -1], np.int64)
    st = ops.Status(cuda)
    ops.gather(_t(arr, cuda), _t(idx, cuda), L.V_BOUNDS, st, stmt=2, site=4)
    s = st.read()
    assert not s.ok and s.elem == 3 and s.site == 4 and s.stmt == 2
    idx = np.array([0, 9, 4, 2], np.int64)
    for bits in (0, L.V_BOUNDS):
        st = ops.Status(cuda)
        got = ops.gather(_t(arr, cuda), _t(idx, cuda), bits, st)
        assert _np(got).tolist() == O.gather(arr, idx).tolist()
        assert st.read().ok


def test_hist(cuda):
    from paper_2506_23058_b200 import ops

    assert _np(ops.hist(L.HIST_MIN, 99, 3, _t(np.array([0, 0, 2, 5, -1]), cuda),
                        _t(np.array([4, 2, 7, 1, 1]), cuda))).tolist() == [2, 99, 7]
    n = 100_000
    is_ = gen.uniform(1, n, -5, 1000, np.int64)
    vs = gen.uniform(2, n, -(1 << 40), 1 << 40, np.int64)
    for op in (L.HIST_MIN, L.HIST_MAX, L.HIST_ADD):
        want = O.hist(op, 7, 990, is_, vs)
        assert np.array_equal(_np(ops.hist(op, 7, 990, _t(is_, cuda), _t(vs, cuda))), want)
    assert ops.hist(L.HIST_MIN, 1, -3, _t(is_, cuda), _t(vs, cuda)).numel() == 0


@pytest.mark.parametrize("nnz", [0, 1, 7, 4096, 1_000_003])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_csr_gather(cuda, nnz, dtype):
    from paper_2506_23058_b200 import ops

    ncols = 5000
    x = gen.uniform(31, ncols, -(1 << 15), (1 << 15) - 1, dtype)
    vals = gen.uniform(32, nnz, -(1 << 15), (1 << 15) - 1, dtype)
    idx = gen.uniform(33, nnz, 0, ncols - 1, np.int64)
    want = O.csrg(x, vals, idx)
    for variant in VARIANTS:
        st = ops.Status(cuda)
        got = ops.csr_gather(_t(x, cuda), _t(vals, cuda), _t(idx, cuda), variant, st)
        assert np.array_equal(_np(got).astype(np.int64), want)
        assert st.read().ok
    if nnz > 10:
        bad = idx.copy()
        bad[nnz // 2] = ncols
        bad[nnz - 2] = -4
        st = ops.Status(cuda)
        ops.csr_gather(_t(x, cuda), _t(vals, cuda), _t(bad, cuda), L.VARIANT_CHECKED, st)
        s = st.read()
        assert not s.ok and s.elem == nnz // 2


def test_kmeans(cuda):
    import torch

    from paper_2506_23058_b200 import ops

    rng = np.random.default_rng(5)
    nrows, ncols = 300, 50
    lens = rng.integers(0, 40, nrows)
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    nnz = int(ptr[-1])
    vals = np.round(rng.uniform(-4, 9, nnz), 2)
    cols = rng.integers(0, ncols, nnz).astype(np.int64)
    cl = np.round(rng.uniform(-4, 9, ncols), 2)
    rows = np.arange(nrows, dtype=np.int64)
    st = ops.Status(cuda)
    got = _np(ops.kmeans_ker(_t(rows, cuda), _t(ptr, cuda), torch.from_numpy(cl).to(cuda),
                             torch.from_numpy(vals).to(cuda), _t(cols, cuda), L.VARIANT_CHECKED, st))
    want = np.array([O.kmeans_ker(int(r), ptr, cl, vals, cols) for r in rows])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))  # bit-exact f64
    st = ops.Status(cuda)
    ops.kmeans_ker(_t(np.array([nrows], np.int64), cuda), _t(ptr, cuda), torch.from_numpy(cl).to(cuda),
                   torch.from_numpy(vals).to(cuda), _t(cols, cuda), L.VARIANT_CHECKED, st)
    s = st.read()
    assert not s.ok and s.site == 1  # pointers[row+1] fails first


def test_mksgmdescr(cuda):
    from paper_2506_23058_b200 import ops

    for shape, xs in [([0, 2, 1, 0, 3], [1, 2, 3, 4, 5]), ([], []), ([0, 0], [4, 5])]:
        st = ops.Status(cuda)
        got = ops.mksgmdescr(_t(np.array(shape, np.int64), cuda), _t(np.array(xs, np.int64), cuda),
                             L.VARIANT_CHECKED, st)
        assert _np(got).tolist() == O.mksgmdescr(shape, xs).tolist()
    m = 10_000
    shape = gen.uniform(3, m, 0, 9, np.int64)
    xs = gen.uniform(4, m, -9, 9, np.int64)
    st = ops.Status(cuda)
    got = ops.mksgmdescr(_t(shape, cuda), _t(xs, cuda), L.VARIANT_CHECKED, st)
    assert np.array_equal(_np(got), O.mksgmdescr(shape, xs))
    # negative shapes violate the precondition; the checked scatter must flag conflicts
    shape = np.array([3, -3, 4, 1], np.int64)
    xs = np.array([1, 2, 3, 4], np.int64)
    with pytest.raises(O.OracleFail):
        O.mksgmdescr(shape, xs)
    st = ops.Status(cuda)
    ops.mksgmdescr(_t(shape, cuda), _t(xs, cuda), L.VARIANT_CHECKED, st)
    assert st.read().codes & (1 << L.CONFLICT)


def test_gen_uniform(cuda):
    import torch

    from paper_2506_23058_b200 import ops

    for dtype, tdt, lo, hi in [(np.int32, torch.int32, -(1 << 31), (1 << 31) - 1), (np.int64, torch.int64, -5, 17),
                               (np.int32, torch.int32, -128, 127)]:
        got = _np(ops.gen_uniform(100_003, lo, hi, 42, dtype=tdt, offset=77, device=cuda))
        assert np.array_equal(got, gen.uniform(42, 100_003, lo, hi, dtype, offset=77))


def test_workspace_reuse(cuda):
    """Self-resetting look-back state: many launches, changing sizes."""
    from paper_2506_23058_b200 import ops

    for rep in range(40):
        n = [5000, 123_456, 4096, 1][rep % 4]
        xs = gen.uniform(rep, n, -9, 9, np.int32)
        st = ops.Status(cuda)
        gys, dnt = ops.partition2(_t(xs, cuda), Pred.lt(0), L.VARIANT_ELIDED, st)
        nt, ys = O.partition2(Pred.lt(0), xs)
        assert int(dnt.item()) == nt and np.array_equal(_np(gys).astype(np.int64), ys)


@pytest.mark.parametrize("pred", [Pred(7), Pred(8), Pred.ge(120)])  # all, none, ~3 %
@pytest.mark.parametrize("seg", ["one", "unit", "sparse"])
def test_c2_extremes(cuda, pred, seg):
    """C2 at 2^22 with the selectivity and flag density at their extremes:
    every element kept / none / few; one segment, every output its own
    segment (all flags set), or a few long segments."""
    import torch

    from paper_2506_23058_b200 import ops

    n = 1 << 22
    xs = gen.uniform(71, n, -128, 127, np.int32)
    k = len(O.filter_(pred, xs))
    if seg == "one":
        shape = np.array([k], np.int64)
    elif seg == "unit":
        shape = np.ones(k, np.int64)
    else:
        shape = gen.segment_shape(5, 3, k)
    want_ys, want_zs = O.c2(pred, xs, shape)
    for zt in (torch.int32, torch.int64):
        st = ops.Status(cuda)
        ys, zs, dk = ops.c2(_t(xs, cuda), pred, _t(shape, cuda), L.VARIANT_ELIDED, st, z_dtype=zt)
        kk = int(dk.item())
        assert kk == k
        assert np.array_equal(_np(ys)[:kk].astype(np.int64), want_ys)
        assert np.array_equal(_np(zs)[:kk].astype(np.int64), want_zs)
        s = st.read()
        assert s.ok and not s.narrow


# ----------------------------------------------------------------- int64 overflow (the reference's ints are unbounded)
@pytest.mark.parametrize("n", [3, 5000, 1 << 20])
def test_scan_overflow_exact(cuda, n):
    """scan (+) over int64: IXG_OVERFLOW exactly at the first prefix leaving
    int64 (both scan kernels), never for sums that stay inside -- including
    prefixes that touch INT64_MAX/MIN and come back."""
    import torch

    from paper_2506_23058_b200 import ops

    big = 1 << 62
    xs = np.zeros(n, np.int64)
    xs[0], xs[1] = big, big - 1            # 2^63 - 1: fits
    if n > 2:
        xs[2] = -big
    st = ops.Status(cuda)
    got = ops.scan_add(_t(xs, cuda), 0, status=st)
    assert st.read().ok and np.array_equal(_np(got), np.cumsum(xs))
    for at in sorted({2, n // 2, n - 1}):
        ys = xs.copy()
        ys[2] = 0
        ys[at] += 1                        # the prefix at `at` becomes 2^63
        for exclusive in (False, True):
            st = ops.Status(cuda)
            ops.scan_add(_t(ys, cuda), 0, exclusive=exclusive, status=st)
            s = st.read()
            assert not s.ok and s.site == L.OVF_SITE and s.elem == at, (at, s)
    # via the ne seed (int32 input path too)
    st = ops.Status(cuda)
    ops.scan_add(torch.ones(n, dtype=torch.int32, device=cuda), (1 << 63) - 2, status=st)
    s = st.read()
    assert not s.ok and s.elem == 1


def test_segscan_overflow_resets_at_flags(cuda):
    from paper_2506_23058_b200 import ops

    big = 1 << 62
    xs = np.array([big, big - 1, big, big, 5, -big, -big, -1], np.int64)
    fl = np.array([1, 0, 1, 0, 1, 0, 0, 0], np.uint8)
    st = ops.Status(cuda)
    ops.segscan_add(_t(fl, cuda), _t(xs, cuda), status=st)
    s = st.read()
    assert not s.ok and s.elem == 3  # big + big in the second segment
    xs[3] = big - 1
    xs[4] = -5
    st = ops.Status(cuda)
    ops.segscan_add(_t(fl, cuda), _t(xs, cuda), status=st)
    s = st.read()
    assert not s.ok and s.elem == 6  # -5 - 2^62 - 2^62 < -2^63
    xs[4], xs[7] = 5, 0  # 5 - 2^63: fits
    st = ops.Status(cuda)
    got = ops.segscan_add(_t(fl, cuda), _t(xs, cuda), status=st)
    assert st.read().ok and _np(got).tolist() == O.sgmsum(fl.astype(np.int64), xs).tolist()


def test_hist_add_128bit_bins(cuda):
    """hist (+): bins hold exact 128-bit sums; only a FINAL value outside
    int64 is an overflow (atomic order does not matter)."""
    from paper_2506_23058_b200 import ops

    big = 1 << 62
    is_ = np.array([0, 0, 0, 1, 1, 1, 2], np.int64)
    vs = np.array([big, big, -big, big, big, big, -5], np.int64)
    st = ops.Status(cuda)
    got = ops.hist(L.HIST_ADD, 0, 3, _t(is_, cuda), _t(vs, cuda), status=st)
    s = st.read()
    assert not s.ok and s.elem == 1  # bin 1 = 3 * 2^62
    assert _np(got)[0] == big and _np(got)[2] == -5
    n = 1 << 20
    is2 = (np.arange(n, dtype=np.int64) // 2) % 100
    vs2 = np.where(np.arange(n) % 2 == 0, big, -big).astype(np.int64)  # the atomic order's partial sums swing
    st = ops.Status(cuda)
    got = ops.hist(L.HIST_ADD, 7, 100, _t(is2, cuda), _t(vs2, cuda), status=st)
    assert st.read().ok and np.array_equal(_np(got), O.hist(L.HIST_ADD, 7, 100, is2, vs2))


# ----------------------------------------------------------------- generic scatter: privatised claims, binning
def _scatter_case(n, dtype, kind, seed):
    rng = np.random.default_rng(seed)
    if kind == "streams":  # partition2 indices: two monotone streams (C3)
        c = rng.random(n) < 0.5
        t = np.cumsum(c)
        is_ = np.where(c, t - 1, t[-1] + (np.arange(1, n + 1) - t) - 1).astype(np.int64)
    else:
        is_ = rng.permutation(n).astype(np.int64)
    vs = rng.integers(-1000, 1000, n).astype(dtype)
    return is_, vs


@pytest.mark.parametrize("layout", ["direct", "binned"])
@pytest.mark.parametrize("kind", ["streams", "random"])
@pytest.mark.parametrize("n", [1000, 65_537, 1 << 20])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_scatter_layouts(cuda, monkeypatch, layout, kind, n, dtype):
    """ELIDED (Sc1), injective-only and CHECKED scatters in both layouts
    (IXG_BIN_SHIFT=12: 4096-destination windows, so small sizes bin into many
    windows) against the C restatement of oracle.py:294-305: permutations,
    out-of-range indices (ignored), equal-valued duplicates (legal) and a
    conflicting duplicate (NonIdempotentScatter)."""
    from paper_2506_23058_b200 import ops

    monkeypatch.setenv("IXG_BIN_SHIFT", "12")
    lay = L.SCATTER_BINNED if layout == "binned" else L.SCATTER_DIRECT
    is_, vs = _scatter_case(n, dtype, kind, n)
    want = O.scatter(np.zeros(n, np.int64), is_, vs)
    for bits in (0, L.V_INIT, L.V_CONFLICT | L.V_INIT):
        st = ops.Status(cuda)
        out = _t(np.zeros(n, dtype), cuda)
        ops.scatter(out, _t(is_, cuda), _t(vs, cuda), bits, st, layout=lay)
        assert st.read().ok and np.array_equal(_np(out).astype(np.int64), want), bits
    # CHECKED with out-of-range indices, equal duplicates, into a larger dst
    is2 = is_.copy()
    is2[::7] = -1
    is2[3::11] = n + 5
    is2[1::13] = is_[2]  # many duplicates of one destination ...
    vs2 = vs.copy()
    vs2[1::13] = vs[2]  # ... all with its value (position 2 keeps it too): legal
    dst = np.full(n + 3, 9, dtype)
    want2 = O.scatter(dst.astype(np.int64), is2, vs2)
    st = ops.Status(cuda)
    out = _t(dst, cuda)
    ops.scatter(out, _t(is2, cuda), _t(vs2, cuda), L.V_CONFLICT | L.V_INIT, st, layout=lay)
    assert st.read().ok and np.array_equal(_np(out).astype(np.int64), want2)
    vs2[1 + 13 * (len(vs2[1::13]) // 2)] += 1  # one conflicting value
    st = ops.Status(cuda)
    out = _t(dst, cuda)
    ops.scatter(out, _t(is2, cuda), _t(vs2, cuda), L.V_CONFLICT | L.V_INIT, st, layout=lay)
    s = st.read()
    assert not s.ok and s.codes & (1 << L.CONFLICT)


def test_scatter_probe_and_auto(cuda):
    """the locality probe: C3's two monotone streams stay direct, a random
    permutation bins (and the auto layout still scatters exactly)."""
    from paper_2506_23058_b200 import ops

    n = 1 << 23
    for kind, want in (("streams", L.SCATTER_DIRECT), ("random", L.SCATTER_BINNED)):
        is_, vs = _scatter_case(n, np.int32, kind, 3)
        assert ops.scatter_layout(_t(is_, cuda), (1 << 23) + 1) == want
    is_, vs = _scatter_case(n, np.int32, "random", 4)
    out = _t(np.zeros(n, np.int32), cuda)
    st = ops.Status(cuda)
    ops.scatter(out, _t(is_, cuda), _t(vs, cuda), 0, st)
    w = np.zeros(n, np.int32)
    w[is_] = vs
    assert st.read().ok and np.array_equal(_np(out), w)


def test_two_streams_concurrently(cuda):
    """the same ops on two streams at once (per-stream workspaces: look-back
    slots and tile tickets are never shared) -- both results exact."""
    import torch

    from paper_2506_23058_b200 import ops

    n = 1 << 22
    xa = gen.uniform(1, n, -128, 127, np.int32)
    xb = gen.uniform(2, n, -128, 127, np.int32)
    p = Pred.ge(0)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    ta, tb = _t(xa, cuda), _t(xb, cuda)
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(sa):
            sta = ops.Status(cuda)
            ya, dka = ops.filter(ta, p, L.VARIANT_CHECKED, sta)
            ca = ops.scan_add(ta, 5)
        with torch.cuda.stream(sb):
            stb = ops.Status(cuda)
            yb, dkb = ops.filter(tb, p, L.VARIANT_CHECKED, stb)
            cb = ops.scan_add(tb, 5)
        torch.cuda.synchronize()
        res = (ya[: int(dka.item())], yb[: int(dkb.item())], ca, cb)
        assert np.array_equal(_np(res[0]), O.filter_(p, xa)) and np.array_equal(_np(res[1]), O.filter_(p, xb))
        assert np.array_equal(_np(res[2]), O.scan_add(xa, 5)) and np.array_equal(_np(res[3]), O.scan_add(xb, 5))


def test_back_to_back_launches(cuda):
    """Consecutive big-tile kernels on one stream overlap their launch with
    programmatic dependent launch (each waits for its predecessor in-kernel;
    C2's fused kernel only before it reads the bitmap): 48 pipelines queued
    without a host sync, on one shared workspace per op, every result exact."""
    import torch

    from paper_2506_23058_b200 import ops

    n, m = 300_001, 700
    runs = []
    for i in range(16):
        xs = gen.uniform(100 + i, n, -128, 127, np.int32)
        k = int((xs >= 0).sum())
        shape = gen.segment_shape(200 + i, m, k)
        runs.append((xs, shape, _t(xs, cuda), _t(shape, cuda)))
    torch.cuda.synchronize()
    outs = []
    st = ops.Status(cuda)
    for xs, shape, xd, sd in runs:
        p2 = ops.partition2(xd, Pred.lt(0), L.VARIANT_ELIDED, st)
        f = ops.filter(xd, Pred.ge(3), L.VARIANT_ELIDED, st)
        c = ops.c2(xd, Pred.ge(0), sd, L.VARIANT_ELIDED, st)
        outs.append((p2, f, c))
    torch.cuda.synchronize()
    assert st.read().ok
    for (xs, shape, _, _), ((ys, dnt), (fy, fk), (cy, cz, ck)) in zip(runs, outs):
        nt, want = O.partition2(Pred.lt(0), xs)
        assert int(dnt.item()) == nt and np.array_equal(_np(ys).astype(np.int64), want)
        kf = int(fk.item())
        assert np.array_equal(_np(fy[:kf]).astype(np.int64), O.filter_(Pred.ge(3), xs))
        wy, wz = O.c2(Pred.ge(0), xs, shape)
        kc = int(ck.item())
        assert np.array_equal(_np(cy[:kc]).astype(np.int64), wy) and np.array_equal(_np(cz[:kc]).astype(np.int64), wz)
