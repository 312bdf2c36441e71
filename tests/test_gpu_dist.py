"""GPU side of the sharded path: the per-rank kernels of dist.GpuC2Local
(ixg_filter, ixg_flag_bitmap, ixg_segsum with flag offset and carry,
ixg_seg_carry), driven for G simulated ranks one after the other on one GPU
(no kernel waits on another rank), with the same all-gather arithmetic as
dist.c2_sharded.  The concatenated result must equal the single-process C2."""

import numpy as np
import pytest

from oracle import ixoracle as O
from paper_2506_23058_b200 import dist as D
from paper_2506_23058_b200 import gen
from paper_2506_23058_b200.pred import Pred

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G,n,m", [(2, 100_000, 300), (4, 1_000_003, 5000), (8, 3_000_000, 20_000), (3, 50, 7)])
def test_c2_sharded_kernels(cuda, G, n, m):
    import torch

    xs = gen.uniform(G * 1000 + n, n, -128, 127, np.int32)
    p = Pred.ge(0)
    k_total = int((xs >= 0).sum())
    shape = gen.segment_shape(G, m, k_total)
    want_ys, want_zs = O.c2(p, xs, shape)
    locs = []
    for r in range(G):
        lo, hi = r * n // G, (r + 1) * n // G
        locs.append(D.GpuC2Local(torch.from_numpy(xs[lo:hi].copy()).to(cuda), p, torch.from_numpy(shape).to(cuda)))
    ks = [loc.filter() for loc in locs]                      # all-gather #1: counts
    K = D.exclusive_offsets(ks)
    assert sum(ks) == k_total
    for loc in locs:
        loc.flag_bitmap(k_total)
    aggs = [loc.segsum(K[r]) for r, loc in enumerate(locs)]  # all-gather #2: aggregates
    for r, (loc, c) in enumerate(zip(locs, D.seg_carries(aggs))):
        if c[0] != 0:
            loc.seg_carry(K[r], c[0])
    ys = np.concatenate([loc.ys[: loc.k].cpu().numpy() for loc in locs]).astype(np.int64)
    zs = np.concatenate([loc.zs[: loc.k].cpu().numpy() for loc in locs]).astype(np.int64)
    assert np.array_equal(ys, want_ys)
    assert np.array_equal(zs, want_zs)
    for loc in locs:
        assert loc.st.read().ok


@pytest.mark.parametrize("G,n", [(2, 100_000), (4, 1_000_003), (8, 3_000_001), (3, 50)])
def test_partition2_sharded_kernels(cuda, G, n):
    """dist.GpuPart2Local per simulated rank + dist.partition2_runs: each
    shard's [trues | falses] lands at its global runs; the assembly equals
    the single-process partition2."""
    import torch

    xs = gen.uniform(G * 7 + n, n, -(1 << 31), (1 << 31) - 1, np.int32)
    p = Pred.lt(0)
    want_nt, want = O.partition2(p, xs)
    locs, tc, sizes = [], [], []
    for r in range(G):
        lo, hi = r * n // G, (r + 1) * n // G
        loc = D.GpuPart2Local(torch.from_numpy(xs[lo:hi].copy()).to(cuda), p)
        t, size = loc.partition2()
        locs.append(loc)
        tc.append(t)
        sizes.append(size)
    out = np.zeros(n, np.int64)
    for r, loc in enumerate(locs):
        nt, runs = D.partition2_runs(tc, sizes, r)
        assert nt == want_nt
        ys = loc.ys.cpu().numpy().astype(np.int64)
        off = 0
        for s, ln in zip(runs.starts, runs.lengths):
            out[s:s + ln] = ys[off:off + ln]
            off += ln
        assert loc.st.read().ok
    assert np.array_equal(out, want)


@pytest.mark.parametrize("G,n", [(2, 100_000), (4, 1_000_003), (3, 50)])
def test_sharded_scan_filter_partition3_kernels(cuda, G, n):
    """the per-rank GPU locals of dist.scan_sharded / filter_sharded /
    partition3_sharded, driven rank by rank with the same offset arithmetic."""
    import torch

    from paper_2506_23058_b200 import ops

    xs = gen.uniform(G + n, n, -1000, 1000, np.int64)
    bounds = [(r * n // G, (r + 1) * n // G) for r in range(G)]
    # reduce_add == the shard sums (i32 / i64 / u8 inputs)
    for dt in (np.int32, np.int64, np.uint8):
        a = (xs % 200).astype(dt) if dt == np.uint8 else xs.astype(dt)
        assert int(ops.reduce_add(torch.from_numpy(a).to(cuda)).item()) == int(a.astype(np.int64).sum())
    # scan: totals first, then one seeded scan per rank
    locs = [D.GpuScanLocal(torch.from_numpy(xs[lo:hi].copy()).to(cuda)) for lo, hi in bounds]
    ts = [loc.total() for loc in locs]
    for exclusive in (False, True):
        for loc, seed in zip(locs, D.exclusive_offsets(ts)):
            loc.scan(-3 + seed, exclusive)
        got = np.concatenate([loc.out.cpu().numpy() for loc in locs])
        want = O.scan_add(xs, -3) - (xs if exclusive else 0)
        assert np.array_equal(got, want)
    # filter
    fl = [D.GpuFilterLocal(torch.from_numpy(xs[lo:hi].copy()).to(cuda), Pred.gt(100)) for lo, hi in bounds]
    ks = [f.filter() for f in fl]
    got = np.concatenate([f.ys[:k].cpu().numpy() for f, k in zip(fl, ks)])
    assert np.array_equal(got, O.filter_(Pred.gt(100), xs))
    # partition3
    p, q = Pred.lt(-300), Pred.hash(17)
    pl = [D.GpuPart3Local(torch.from_numpy(xs[lo:hi].copy()).to(cuda), p, q) for lo, hi in bounds]
    rows = [loc.partition3() for loc in pl]
    counts = [[m1, m2, size - m1 - m2] for m1, m2, size in rows]
    out = np.zeros(n, np.int64)
    for r, loc in enumerate(pl):
        totals, runs = D.partition_runs(counts, r)
        ys = loc.ys.cpu().numpy()
        off = 0
        for s, ln in zip(runs.starts, runs.lengths):
            out[s:s + ln] = ys[off:off + ln]
            off += ln
    wm1, wm2, wys = O.partition3(p, q, xs)
    assert totals[:2] == [wm1, wm2]
    assert np.array_equal(out, wys)


@pytest.mark.parametrize("G,per,thr", [(2, 100_000, 0), (4, 300_000, 0), (8, 40_000, 0), (3, 4, 0),
                                        (5, 70_004, -(1 << 30)), (2, 1 << 20, (1 << 31) - 2), (3, 8_196, -(1 << 31))])
@pytest.mark.parametrize("dtype", [np.int32, np.int64])
def test_partition2_peer_kernel(cuda, G, per, thr, dtype):
    """ixg_partition2_peer for G simulated ranks in one process: every rank's
    kernel stores its runs straight into the G destination shards (the
    pointer table a rank gets from CUDA IPC); the shards concatenate to the
    single-process partition2."""
    import torch

    from paper_2506_23058_b200 import ops

    n = G * per
    xs = gen.uniform(G * 31 + per, n, -(1 << 31), (1 << 31) - 1, dtype)
    p = Pred.lt(thr)  # 50 %, 25 %, ~all and no trues
    want_nt, want = O.partition2(p, xs)
    tdt = torch.int32 if dtype == np.int32 else torch.int64
    bufs = [torch.full((per,), -7, dtype=tdt, device=cuda) for _ in range(G)]
    ptrs = [b.data_ptr() for b in bufs]
    shards = [torch.from_numpy(xs[r * per:(r + 1) * per].copy()).to(cuda) for r in range(G)]
    ts = [int(ops.partition_counts(x, p).item()) for x in shards]
    assert sum(ts) == want_nt
    d_counts = torch.tensor(ts, dtype=torch.int64, device=cuda)  # what the device all-gather delivers
    for r in range(G):
        ops.partition2_peer(shards[r], p, ptrs, per, d_counts, r)
        assert ops.rank_offsets(d_counts, G, r).tolist() == [sum(ts[:r]), want_nt]
    got = torch.cat(bufs).cpu().numpy().astype(np.int64)
    assert np.array_equal(got, want)


def _ipc_worker(rank, world, port, per, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = world * per
        xs = gen.uniform(99, n, -(1 << 31), (1 << 31) - 1, np.int32)
        loc = D.GpuPart2PeerLocal(torch.from_numpy(xs[rank * per:(rank + 1) * per].copy()).cuda(), Pred.lt(0))
        nt = int(loc.step()[1].item())
        want_nt, want = O.partition2(Pred.lt(0), xs)
        ok = nt == want_nt and np.array_equal(loc.out.cpu().numpy().astype(np.int64), want[rank * per:(rank + 1) * per])
        dist.barrier()
        loc.close()
        oks = [None] * world
        dist.all_gather_object(oks, bool(ok))
        if rank == 0:
            q.put(all(oks))
    finally:
        dist.destroy_process_group()


def test_partition2_peer_ipc_two_processes(cuda):
    """the CUDA-IPC plumbing of GpuPart2PeerLocal: two processes on one GPU
    map each other's shard and store into it (the kernels never wait on each
    other; the host barrier orders the reads)."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, 200_000, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(300)
        assert pr.exitcode == 0
    assert q.get() is True


def _c2_worker(rank, world, port, per, m, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = world * per
        xs = gen.uniform(7, n, -128, 127, np.int32)
        k_total = int((xs >= 0).sum())
        shape = gen.segment_shape(8, m, k_total)
        loc = D.GpuC2Local(torch.from_numpy(xs[rank * per:(rank + 1) * per].copy()).cuda(), Pred.ge(0),
                           torch.from_numpy(shape).cuda())
        for _ in range(2):  # twice: the bitmap / workspaces are reused
            loc.step_device()
        k, off = int(loc.dk.item()), int(loc.d_off[0].item())
        want_ys, want_zs = O.c2(Pred.ge(0), xs, shape)
        ok = (np.array_equal(loc.ys[:k].cpu().numpy().astype(np.int64), want_ys[off:off + k])
              and np.array_equal(loc.zs[:k].cpu().numpy().astype(np.int64), want_zs[off:off + k])
              and int(loc.d_off[1].item()) == k_total and loc.st.read().ok)
        oks = [None] * world
        dist.all_gather_object(oks, bool(ok))
        if rank == 0:
            q.put(all(oks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_c2_step_device_processes(cuda, world):
    """GpuC2Local.step_device -- the sharded C2 with every count, offset and
    carry on the device -- in `world` processes sharing one GPU (gloo for the
    tiny exchanges; NCCL on a multi-GPU box): each rank's slice equals the
    single-process C2 at its global offset."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=_c2_worker, args=(r, world, port, 150_001, 3000, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(300)
        assert pr.exitcode == 0
    assert q.get() is True
