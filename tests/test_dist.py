"""Multi-rank host logic of the sharded path (paper_2506_23058_b200.dist) on
CPU: world_size 2 and 3 over gloo, each rank running a numpy stand-in for
its GPU's local kernels, results compared with the single-process oracle.
The same orchestration code drives the CUDA kernels on the GPU box."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import ixoracle as O
from paper_2506_23058_b200 import dist as D
from paper_2506_23058_b200 import gen
from paper_2506_23058_b200.pred import Pred


def test_arithmetic():
    assert D.exclusive_offsets([3, 0, 5]) == [0, 3, 3]
    assert D.seg_combine((5, False), (2, False)) == (7, False)
    assert D.seg_combine((5, True), (2, True)) == (2, True)
    assert D.seg_carries([(4, False), (3, True), (1, False)]) == [(0, False), (4, False), (3, True)]
    nt, runs = D.partition2_runs([2, 1], [5, 4], 1)
    assert nt == 3 and runs.starts == [2, 3 + 3] and runs.lengths == [1, 3]


class NpC2Local:
    def __init__(self, xs, pred, shape):
        self.xs, self.pred, self.shape = xs, pred, shape

    def filter(self):
        self.ys = np.array([x for x in self.xs if self.pred(int(x))], dtype=np.int64)
        return len(self.ys)

    def flag_bitmap(self, k_total):
        self.flags = O.mkflags(k_total, self.shape)

    def segsum(self, flag_base):
        fl = self.flags[flag_base:flag_base + len(self.ys)]
        self.zs = O.sgmsum(fl, self.ys) if len(self.ys) else np.zeros(0, np.int64)
        f = bool(fl.any())
        last = int(np.nonzero(fl)[0][-1]) if f else 0
        v = int(self.ys[last:].sum()) if len(self.ys) else 0
        return v, f

    def seg_carry(self, flag_base, carry_v):
        fl = self.flags[flag_base:flag_base + len(self.ys)]
        first = int(np.nonzero(fl)[0][0]) if fl.any() else len(self.ys)
        self.zs[:first] += carry_v


class NpPart2Local:
    def __init__(self, xs, pred):
        self.xs, self.pred = xs, pred

    def partition2(self):
        nt, ys = O.partition2(self.pred, self.xs)
        self.ys = ys
        return nt, len(self.xs)

    def ys_tensor(self):
        import torch

        return torch.from_numpy(np.asarray(self.ys, dtype=np.int64))


def _worker(rank, world, port, n, m, q):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = rank * n // world, (rank + 1) * n // world
        xs = gen.uniform(5, n, -20, 20, np.int64)
        p = Pred.ge(0)
        k_total = int((xs >= 0).sum())
        shape = gen.segment_shape(9, m, k_total)
        loc = NpC2Local(xs[lo:hi], p, shape)
        K, k, kt = D.c2_sharded(loc)
        assert kt == k_total
        zs_all = [None] * world
        dist.all_gather_object(zs_all, (K, loc.ys.tolist(), loc.zs.tolist()))
        p2 = NpPart2Local(xs[lo:hi], Pred.lt(3))
        nt, runs, mine = D.partition2_sharded(p2, exchange=True)
        slices = [None] * world
        dist.all_gather_object(slices, mine.tolist())
        parts = [None] * world
        dist.all_gather_object(parts, (runs.starts, runs.lengths, p2.ys.tolist()))
        if rank == 0:
            ys_g = np.zeros(k_total, np.int64)
            zs_g = np.zeros(k_total, np.int64)
            for K_r, ys_r, zs_r in zs_all:
                ys_g[K_r:K_r + len(ys_r)] = ys_r
                zs_g[K_r:K_r + len(zs_r)] = zs_r
            want_ys, want_zs = O.c2(p, xs, shape)
            p_out = np.zeros(n, np.int64)
            for starts, lengths, ys_r in parts:
                off = 0
                for s, ln in zip(starts, lengths):
                    p_out[s:s + ln] = ys_r[off:off + ln]
                    off += ln
            want_nt, want_p = O.partition2(Pred.lt(3), xs)
            exchanged = np.concatenate([np.array(x, np.int64) for x in slices])
            q.put((np.array_equal(ys_g, want_ys), np.array_equal(zs_g, want_zs), nt == want_nt,
                   np.array_equal(p_out, want_p) and np.array_equal(exchanged, want_p)
                   and all(len(slices[r]) == (r + 1) * n // world - r * n // world for r in range(world))))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("world,n,m", [(2, 1000, 23), (3, 2001, 40), (2, 7, 3)])
def test_sharded_c2_and_partition2_gloo(world, n, m):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    assert q.get() == (True, True, True, True)


# ------------------------------------------------------------------ scan / filter / partition3 / hist
class NpScanLocal:
    def __init__(self, xs):
        self.xs = xs

    def total(self):
        return int(self.xs.sum())

    def scan(self, seed, exclusive):
        inc = seed + np.cumsum(self.xs, dtype=np.int64)
        self.out = inc - self.xs if exclusive else inc


class NpFilterLocal:
    def __init__(self, xs, pred):
        self.xs, self.pred = xs, pred

    def filter(self):
        self.ys = O.filter_(self.pred, self.xs)
        return len(self.ys)


class NpPart3Local:
    def __init__(self, xs, p, q):
        self.xs, self.p, self.q = xs, p, q

    def partition3(self):
        m1, m2, self.ys = O.partition3(self.p, self.q, self.xs)
        return m1, m2, len(self.xs)


class NpHistLocal:
    def __init__(self, op, dlen, is_, vs):
        self.op, self.dlen, self.is_, self.vs = op, dlen, is_, vs

    def hist(self, ne):
        import torch

        return torch.from_numpy(O.hist(self.op, ne, self.dlen, self.is_, self.vs).astype(np.int64))


def _worker2(rank, world, port, n, q):
    import torch.distributed as dist

    from paper_2506_23058_b200 import _lib as L

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = rank * n // world, (rank + 1) * n // world
        xs = gen.uniform(11, n, -50, 50, np.int64)
        res = {}
        for exclusive in (False, True):
            sc = NpScanLocal(xs[lo:hi])
            tot = D.scan_sharded(sc, ne=7, exclusive=exclusive)
            parts = [None] * world
            dist.all_gather_object(parts, sc.out.tolist())
            want = O.scan_add(xs, 7)
            if exclusive:
                want = want - xs
            res[f"scan{int(exclusive)}"] = (tot == 7 + int(xs.sum())
                                            and np.array_equal(np.concatenate([np.array(p, np.int64) for p in parts]),
                                                               want))
        fl = NpFilterLocal(xs[lo:hi], Pred.ge(3))
        kt, runs = D.filter_sharded(fl)
        parts = [None] * world
        dist.all_gather_object(parts, (runs.starts, fl.ys.tolist()))
        out = np.zeros(kt, np.int64)
        for (s,), ys_r in parts:
            out[s:s + len(ys_r)] = ys_r
        res["filter"] = np.array_equal(out, O.filter_(Pred.ge(3), xs))
        p3 = NpPart3Local(xs[lo:hi], Pred.lt(-10), Pred.hash(5))
        (M1, M2), runs = D.partition3_sharded(p3)
        parts = [None] * world
        dist.all_gather_object(parts, (runs.starts, runs.lengths, p3.ys.tolist()))
        out = np.zeros(n, np.int64)
        for starts, lengths, ys_r in parts:
            off = 0
            for s, ln in zip(starts, lengths):
                out[s:s + ln] = ys_r[off:off + ln]
                off += ln
        wm1, wm2, wys = O.partition3(Pred.lt(-10), Pred.hash(5), xs)
        res["partition3"] = (M1, M2) == (wm1, wm2) and np.array_equal(out, wys)
        is_ = gen.uniform(12, n, -3, 40, np.int64)
        for op_name, op in (("min", L.HIST_MIN), ("max", L.HIST_MAX), ("add", L.HIST_ADD)):
            ne = {"min": 1 << 40, "max": -(1 << 40), "add": 5}[op_name]
            table = D.hist_sharded(NpHistLocal(op, 37, is_[lo:hi], xs[lo:hi]), op_name, ne)
            res[f"hist_{op_name}"] = np.array_equal(table.numpy(), O.hist(op, ne, 37, is_, xs))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 1001), (3, 2500)])
def test_sharded_scan_filter_partition3_hist_gloo(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker2, args=(r, world, port, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(180)
        assert pr.exitcode == 0
    res = q.get()
    assert all(res.values()), res
