"""GPU parity at BASELINE.json's full sizes.

Where the CPU port finishes in seconds the result is compared bit for bit
with it (C2 at 2^28, C4 at 2^28 nnz); at 2^29 / 2^32 the checks are
size-independent properties that pin the result exactly:

* C3 scatter of a permutation: out[is[i]] == vs[i] for every i (torch gather
  as the checker) and every destination written once.
* C5 partition2 at 2^32: the input is a bijection of the index,
  xs[i] = i * A mod 2^32 (A odd), so every output value names its source
  index; the result is the stable partition iff the decoded indices of the
  true run are the true positions in increasing order, and the same for the
  false run.
"""

import numpy as np
import pytest

from oracle import ixoracle as O
from paper_2506_23058_b200 import _lib as L
from paper_2506_23058_b200 import gen
from paper_2506_23058_b200.pred import Pred

pytestmark = pytest.mark.gpu


def test_c2_full_size(cuda):
    import torch

    from paper_2506_23058_b200 import ops

    n, m = 1 << 28, 1 << 20
    xs_h = gen.uniform(0, n, -128, 127, np.int32)
    k = int(np.count_nonzero(xs_h >= 0))
    shape = gen.segment_shape(1, m, k)
    want_ys, want_zs = O.par_c2_i32(Pred.ge(0), xs_h, shape)
    want_k = len(want_ys)
    st = ops.Status(cuda)
    ys, zs, dk = ops.c2(torch.from_numpy(xs_h).to(cuda), Pred.ge(0), torch.from_numpy(shape).to(cuda),
                        L.VARIANT_ELIDED, st)
    kk = int(dk.item())
    assert kk == want_k == k
    assert torch.equal(ys[:kk].cpu(), torch.from_numpy(want_ys[:kk]))
    assert torch.equal(zs[:kk].cpu(), torch.from_numpy(want_zs[:kk]))
    s = st.read()
    assert s.ok and not s.narrow


def test_c3_scatter_full_size(cuda):
    import torch

    from paper_2506_23058_b200 import ops

    n = 1 << 29
    xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 11, torch.int32)
    c = xs < 0
    t = torch.cumsum(c, 0, dtype=torch.int64)
    nt = t[-1]
    i1 = torch.arange(1, n + 1, device=cuda, dtype=torch.int64)
    is_ = torch.where(c, t - 1, nt + (i1 - t) - 1)
    del xs, c, t, i1
    vs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 12, torch.int32)
    out = torch.full((n,), 7, dtype=torch.int32, device=cuda)
    st = ops.Status(cuda)
    ops.scatter(out, is_, vs, 0, st)  # ELIDED (Sc1)
    assert torch.equal(out[is_], vs)
    assert int(torch.bincount(is_, minlength=n).max().item()) == 1
    assert st.read().ok
    # CHECKED at full size: dst init + OOB test + the privatised claims, no
    # conflict on a permutation; then one duplicate index with another value
    out2 = torch.full((n,), 7, dtype=torch.int32, device=cuda)
    st = ops.Status(cuda)
    ops.scatter(out2, is_, vs, L.V_CONFLICT | L.V_INIT, st)
    assert st.read().ok and torch.equal(out2, out)
    is_[n // 3] = is_[2 * n // 3]
    vs[n // 3] = vs[2 * n // 3] + 1
    st = ops.Status(cuda)
    ops.scatter(out2, is_, vs, L.V_CONFLICT | L.V_INIT, st)
    s = st.read()
    assert not s.ok and s.codes & (1 << L.CONFLICT)


@pytest.mark.parametrize("checked", [False, True])
def test_c3_random_permutation_full_size(cuda, checked):
    """C3's secondary at 2^29: a random permutation, binned by destination
    window (the probe must choose it), ELIDED and CHECKED."""
    import torch

    from paper_2506_23058_b200 import ops

    n = 1 << 29
    g = torch.Generator(device=cuda)
    g.manual_seed(5)
    is_ = torch.randperm(n, generator=g, device=cuda, dtype=torch.int64)
    assert ops.scatter_layout(is_, n) == L.SCATTER_BINNED
    vs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 13, torch.int32)
    out = torch.full((n,), 7, dtype=torch.int32, device=cuda)
    st = ops.Status(cuda)
    ops.scatter(out, is_, vs, (L.V_CONFLICT | L.V_INIT) if checked else 0, st)
    assert st.read().ok and torch.equal(out[is_], vs)


def test_c4_csr_full_size(cuda):
    import torch

    from paper_2506_23058_b200 import ops

    nnz, ncols = 1 << 28, 1 << 20
    x = ops.gen_uniform(ncols, -(1 << 15), (1 << 15) - 1, 3, torch.int32, device=cuda)
    vals = ops.gen_uniform(nnz, -(1 << 15), (1 << 15) - 1, 4, torch.int32, device=cuda)
    idx = ops.gen_uniform(nnz, 0, ncols - 1, 5, torch.int64, device=cuda)
    st = ops.Status(cuda)
    out = ops.csr_gather(x, vals, idx, L.VARIANT_ELIDED, st)
    # torch as the checker over the full size; the C oracle over a 2^22 prefix
    want = vals.to(torch.int64) * x.to(torch.int64)[idx]
    assert torch.equal(out.to(torch.int64), want)
    pre = 1 << 22
    w = O.csrg(x.cpu().numpy(), vals[:pre].cpu().numpy(), idx[:pre].cpu().numpy())
    assert np.array_equal(out[:pre].cpu().numpy().astype(np.int64), w)
    assert st.read().ok


def test_c5_partition2_full_size(cuda):
    import torch

    from paper_2506_23058_b200 import ops

    n = 1 << 32
    A = 0x9E3779B1  # odd: i -> i * A mod 2^32 is a bijection
    inv = pow(A, -1, 1 << 32)
    xs = torch.empty(n, dtype=torch.int32, device=cuda)
    chunk = 1 << 28
    for s in range(0, n, chunk):  # xs[i] = (i * A) mod 2^32 as int32
        i = torch.arange(s, s + chunk, device=cuda, dtype=torch.int64)
        v = (i * A) & 0xFFFFFFFF
        xs[s:s + chunk] = torch.where(v >= (1 << 31), v - (1 << 32), v).to(torch.int32)
    st = ops.Status(cuda)
    ys, dnt = ops.partition2(xs, Pred.lt(0), L.VARIANT_ELIDED, st)
    nt = int(dnt.item())
    assert nt == int((xs < 0).sum().item())
    del xs
    prev_t, prev_f = -1, -1
    seen = 0
    for s in range(0, n, chunk):
        v = ys[s:s + chunk].to(torch.int64) & 0xFFFFFFFF
        src = (v * inv) & 0xFFFFFFFF  # the source index of every output
        in_true = torch.arange(s, s + chunk, device=cuda) < nt
        neg = v >= (1 << 31)
        assert torch.equal(neg, in_true)  # class of every output matches its run
        for mask, name in ((in_true, "t"), (~in_true, "f")):
            idx = src[mask]
            if idx.numel() == 0:
                continue
            assert bool((idx[1:] > idx[:-1]).all())  # stable: increasing source order
            first = int(idx[0].item())
            if name == "t":
                assert first > prev_t
                prev_t = int(idx[-1].item())
            else:
                assert first > prev_f
                prev_f = int(idx[-1].item())
            seen += idx.numel()
    assert seen == n
    assert st.read().ok
