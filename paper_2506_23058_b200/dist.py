"""Multi-GPU sharding of the hot path.

One process per GPU (torch.distributed, NCCL on the GPU box; gloo for the
CPU tests).  Inputs are sharded contiguously; the only exchanges are tiny
all-gathers of per-rank totals -- the data never moves:

* partition2 (C5): all-gather of each rank's true-count; rank r's local
  result [its trues | its falses] is exactly two runs of the global result,
  at [T_<r, T_<r + T_r) and [NT + F_<r, NT + F_<r + F_r).
* partition3 / filter: the same with per-class counts (partition_runs).
* scan (+): each rank's total (ixg_reduce_add) is all-gathered first; the
  rank then runs ONE seeded scan with ne + the totals of the ranks before it.
* hist: each rank builds the table of its shard; an all-reduce with the
  hist operator (min / max / sum) combines them (ne seeds rank 0 only for sum).
* CSR gather / map: shards by nnz range with `x` replicated; no exchange.
* C2 (filter + mkFlags + sgmSum): all-gather of each rank's filter count k_r
  gives its output offset K_r; the mkFlags bitmap is built from the global
  segment shape on every rank; each rank's segmented sum starts with carry
  (0, false) and reports its aggregate; an all-gather of the aggregates
  gives each rank the carry of the ranks before it, added to its outputs
  before its first segment start (the same fix-up the tiles use inside a GPU).

The orchestration is written against a small `Local` interface so that the
exact same code runs with the CUDA kernels (GpuLocal) and with a numpy
stand-in in the CPU multi-process tests (tests/test_dist.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Sequence, Tuple


# ----------------------------------------------------------------- arithmetic
def exclusive_offsets(counts: Sequence[int]) -> List[int]:
    out, acc = [], 0
    for c in counts:
        out.append(acc)
        acc += int(c)
    return out


def seg_combine(a: Tuple[int, bool], b: Tuple[int, bool]) -> Tuple[int, bool]:
    """(v1, f1) (+) (v2, f2) = (f2 ? v2 : v1 + v2, f1 || f2) -- PAPER.md:399-402."""
    (v1, f1), (v2, f2) = a, b
    return (v2 if f2 else v1 + v2, bool(f1 or f2))


def seg_carries(aggs: Sequence[Tuple[int, bool]]) -> List[Tuple[int, bool]]:
    """carry INTO each rank = segmented combine of the aggregates before it."""
    out, acc = [], (0, False)
    for a in aggs:
        out.append(acc)
        acc = seg_combine(acc, a)
    return out


@dataclass
class Runs:
    """Where a rank's local output lives in the global result."""
    starts: List[int]   # global start of each local run
    lengths: List[int]  # length of each run (local runs are stored back to back)


def partition2_runs(true_counts: Sequence[int], sizes: Sequence[int], rank: int) -> Tuple[int, Runs]:
    nt = sum(true_counts)
    t_before = exclusive_offsets(true_counts)[rank]
    falses = [s - t for s, t in zip(sizes, true_counts)]
    f_before = exclusive_offsets(falses)[rank]
    return nt, Runs([t_before, nt + f_before], [true_counts[rank], falses[rank]])


def partition_runs(counts: Sequence[Sequence[int]], rank: int) -> Tuple[List[int], Runs]:
    """counts[r][c] = rank r's class-c count, classes in output order.  Class c
    of the global result starts at G_c (the totals of the classes before it);
    rank r's class-c run at G_c + the class-c counts of the ranks before r.
    Returns (class totals, Runs of rank r's local [class 0 | class 1 | ...])."""
    k = len(counts[0])
    totals = [sum(int(row[c]) for row in counts) for c in range(k)]
    G = exclusive_offsets(totals)
    starts = [G[c] + sum(int(counts[q][c]) for q in range(rank)) for c in range(k)]
    return totals, Runs(starts, [int(counts[rank][c]) for c in range(k)])


# ----------------------------------------------------------------- collectives
def all_gather_ints(values: Sequence[int], group=None) -> List[List[int]]:
    """All-gather a few int64 per rank (NCCL needs device tensors)."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor(list(values), dtype=torch.int64, device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return [o.cpu().tolist() for o in out]


def all_gather_dev(t, out, group=None):
    """Device-resident all-gather of a few int64 per rank: rank r's `t` lands
    in out[r * len(t) : (r + 1) * len(t)].  Written as a SUM all-reduce of a
    zero-padded buffer, which NCCL runs stream-ordered (no host round trip)
    and gloo also supports on CUDA tensors (the 1-GPU functional tests)."""
    import torch.distributed as dist

    rank, k = dist.get_rank(group), t.numel()
    if out.is_cuda and dist.get_backend(group) != "nccl":  # gloo: through the host (functional runs only)
        host = out.new_zeros(out.shape, device="cpu")
        host[rank * k:(rank + 1) * k].copy_(t.reshape(-1))
        dist.all_reduce(host, op=dist.ReduceOp.SUM, group=group)
        out.copy_(host)
        return out
    out.zero_()
    out[rank * k:(rank + 1) * k].copy_(t.reshape(-1))
    dist.all_reduce(out, op=dist.ReduceOp.SUM, group=group)
    return out


def device_barrier(flag, group=None):
    """Stream-ordered barrier: when this completes on the stream, every
    rank's earlier work on its own stream has completed (each rank's
    contribution is issued after that work)."""
    import torch
    import torch.distributed as dist

    if flag.is_cuda and dist.get_backend(group) != "nccl":  # gloo: host barrier (functional runs only)
        torch.cuda.synchronize()
        dist.barrier(group=group)
        return
    dist.all_reduce(flag, op=dist.ReduceOp.SUM, group=group)


# ----------------------------------------------------------------- drivers
def c2_sharded(local, group=None):
    """Sharded C2.  `local` provides: filter() -> k; flag_bitmap(K_total);
    segsum(flag_base) -> (v, f); seg_carry(flag_base, carry_v).  Returns
    (K_r, k_r, K_total): this rank's outputs are positions [K_r, K_r + k_r)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    k = local.filter()
    ks = [row[0] for row in all_gather_ints([k], group)]
    K = exclusive_offsets(ks)
    k_total = sum(ks)
    local.flag_bitmap(k_total)
    v, f = local.segsum(K[rank])
    aggs = [(row[0], bool(row[1])) for row in all_gather_ints([v, int(f)], group)]
    carry = seg_carries(aggs)[rank]
    if carry[0] != 0:
        local.seg_carry(K[rank], carry[0])
    return K[rank], k, k_total


def partition2_sharded(local, group=None, exchange: bool = False):
    """Sharded partition2 (C5).  `local.partition2()` -> (true count, size);
    returns (num_true_global, Runs of this rank's local [trues | falses]).
    With `exchange`, the runs are then moved to the shards owning their
    global positions and the third result is this rank's contiguous slice
    of the global output (exchange_runs; NCCL all-to-all on the GPU box)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    t, size = local.partition2()
    rows = all_gather_ints([t, size], group)
    nt, runs = partition2_runs([r[0] for r in rows], [r[1] for r in rows], rank)
    if not exchange:
        return nt, runs
    return nt, runs, exchange_runs(local.ys_tensor(), [[r[0], r[1] - r[0]] for r in rows], rank, group)


def shard_bounds(n_total: int, world: int, rank: int) -> Tuple[int, int]:
    """contiguous destination shard [lo, hi) of rank r (the input split rule)."""
    return rank * n_total // world, (rank + 1) * n_total // world


def _overlap(a0: int, a1: int, b0: int, b1: int) -> int:
    return max(0, min(a1, b1) - max(a0, b0))


def exchange_runs(ys, all_counts: Sequence[Sequence[int]], rank: int, group=None):
    """Move each rank's class runs to the shards that own their global
    positions ('scatter destinations remapped per shard').
    `ys` holds this rank's local [class 0 | class 1 | ...]; all_counts[r][c]
    are every rank's class counts (already all-gathered).  One all-to-all per
    class: a class run's positions increase with the source rank, so the
    received pieces arrive in global order and the result is this rank's
    contiguous slice [lo, hi) of the global output (same tensor type/device)."""
    import torch
    import torch.distributed as dist

    world = len(all_counts)
    k = len(all_counts[0])
    n_total = sum(sum(int(x) for x in row) for row in all_counts)
    runs = [partition_runs(all_counts, q)[1] for q in range(world)]
    lo, hi = shard_bounds(n_total, world, rank)
    outs, off = [], 0
    for c in range(k):
        s0, ln = runs[rank].starts[c], runs[rank].lengths[c]
        send = [_overlap(s0, s0 + ln, *shard_bounds(n_total, world, r)) for r in range(world)]
        recv = [_overlap(runs[q].starts[c], runs[q].starts[c] + runs[q].lengths[c], lo, hi) for q in range(world)]
        out = torch.empty(sum(recv), dtype=ys.dtype, device=ys.device)
        dist.all_to_all_single(out, ys[off:off + ln].contiguous(), output_split_sizes=recv, input_split_sizes=send,
                               group=group)
        outs.append(out)
        off += ln
    return torch.cat(outs)


def partition3_sharded(local, group=None):
    """Sharded partition3.  `local.partition3()` -> (m1, m2, size) of the shard;
    returns ((M1, M2) global, Runs of this rank's local [c0 | c1 | c2])."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    m1, m2, size = local.partition3()
    rows = all_gather_ints([m1, m2, size], group)
    totals, runs = partition_runs([[r[0], r[1], r[2] - r[0] - r[1]] for r in rows], rank)
    return (totals[0], totals[1]), runs


def filter_sharded(local, group=None):
    """Sharded filter / filter_by.  `local.filter()` -> k of the shard; returns
    (k_total, Runs): the shard's outputs are global [K_r, K_r + k_r)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    k = local.filter()
    ks = [row[0] for row in all_gather_ints([k], group)]
    return sum(ks), Runs([exclusive_offsets(ks)[rank]], [k])


def scan_sharded(local, ne: int = 0, exclusive: bool = False, group=None) -> int:
    """Sharded scan (+) ne xs.  `local.total()` -> the shard's sum;
    `local.scan(seed, exclusive)` runs the seeded local scan.  Returns the
    global total (ne + sum of all shards)."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    ts = [row[0] for row in all_gather_ints([local.total()], group)]
    local.scan(ne + exclusive_offsets(ts)[rank], exclusive)
    return ne + sum(ts)


HIST_OPS = {"min": "MIN", "max": "MAX", "add": "SUM"}


def hist_sharded(local, op: str, ne: int, group=None):
    """Sharded hist op ne dlen is vs (oracle.py:306-316) over a contiguous
    shard of (is, vs): local tables, then one all-reduce with the operator.
    For `add` only rank 0 folds ne in."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    table = local.hist(ne if (op != "add" or rank == 0) else 0)
    dist.all_reduce(table, op=getattr(dist.ReduceOp, HIST_OPS[op]), group=group)
    return table


# ----------------------------------------------------------------- GPU backend
class GpuScanLocal:
    """scan (+) on one GPU's shard: ixg_reduce_add for the total, then one
    seeded ixg_scan_add."""

    def __init__(self, xs):
        from . import ops

        self.ops, self.xs = ops, xs
        self.out = None

    def total(self) -> int:
        return int(self.ops.reduce_add(self.xs).item())

    def scan(self, seed: int, exclusive: bool) -> None:
        self.out = self.ops.scan_add(self.xs, seed, exclusive=exclusive)


class GpuFilterLocal:
    def __init__(self, xs, pred):
        from . import _lib as L
        from . import ops

        self.ops, self.L, self.xs, self.pred = ops, L, xs, pred
        self.st = ops.Status(xs.device)
        self.ys = None

    def filter(self) -> int:
        self.ys, dk = self.ops.filter(self.xs, self.pred, self.L.VARIANT_ELIDED, self.st)
        return int(dk.item())


class GpuPart3Local:
    def __init__(self, xs, p, q):
        from . import _lib as L
        from . import ops

        self.ops, self.L, self.xs, self.p, self.q = ops, L, xs, p, q
        self.st = ops.Status(xs.device)
        self.ys = None

    def partition3(self):
        self.ys, dm = self.ops.partition3(self.xs, self.p, self.q, self.L.VARIANT_ELIDED, self.st)
        m1, m2 = dm.cpu().tolist()
        return m1, m2, self.xs.numel()


class GpuHistLocal:
    def __init__(self, op: int, dlen: int, is_, vs):
        from . import ops

        self.ops, self.op, self.dlen, self.is_, self.vs = ops, op, dlen, is_, vs

    def hist(self, ne: int):
        return self.ops.hist(self.op, ne, self.dlen, self.is_, self.vs)


# ----------------------------------------------------------------- GPU backend (C5 / C2)
class GpuPart2Local:
    """partition2 on one GPU's contiguous shard (the single-pass ixg_partition2
    kernel); partition2_sharded turns its true count into the shard's two
    output runs of the global result."""

    def __init__(self, xs, pred):
        import torch

        from . import _lib as L
        from . import ops

        self.ops, self.L = ops, L
        self.xs, self.pred = xs, pred
        self.ys = torch.empty_like(xs)
        self.dnt = torch.empty(1, dtype=torch.int64, device=xs.device)
        self.st = ops.Status(xs.device)

    def partition2(self):
        self.ops.partition2(self.xs, self.pred, self.L.VARIANT_ELIDED, self.st, ys=self.ys, d_nt=self.dnt)
        return int(self.dnt.item()), self.xs.numel()

    def ys_tensor(self):
        return self.ys


class GpuPart2PeerLocal:
    """Sharded partition2 (C5) with the exchange fused into the kernel: the
    global output is sharded contiguously (`shard` elements per rank, in a
    cudaMalloc'd buffer whose IPC handle every rank maps); a count pass and an
    all-gather of the counts give this rank's class bases, then ONE
    partition kernel stores each run straight to the owning shards (local or
    peer stores over NVLink) -- no separate all-to-all pass."""

    def __init__(self, xs, pred, group=None):
        import torch
        import torch.distributed as dist

        from . import ops

        self.ops, self.xs, self.pred, self.group = ops, xs, pred, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        sizes = [r[0] for r in all_gather_ints([xs.numel()], group)]
        if len(set(sizes)) != 1:
            raise ValueError("GpuPart2PeerLocal needs equal shards")
        self.sizes = sizes
        self.shard = sizes[0]
        self.buf = ops.DeviceBuffer(self.shard, xs.dtype, xs.device)
        handles = [None] * self.world
        dist.all_gather_object(handles, self.buf.ipc_handle(), group=group)
        self.opened = []
        self.ptrs = []
        for r, h in enumerate(handles):
            if r == self.rank:
                self.ptrs.append(self.buf.ptr)
            else:
                ptr = ops.ipc_open(h)
                self.opened.append(ptr)
                self.ptrs.append(ptr)
        self.d_tot = torch.empty(1, dtype=torch.int64, device=xs.device)
        self.d_counts = torch.empty(self.world, dtype=torch.int64, device=xs.device)
        self.d_off = torch.empty(2, dtype=torch.int64, device=xs.device)
        self.flag = torch.zeros(1, dtype=torch.int64, device=xs.device)

    @property
    def out(self):
        """this rank's contiguous slice of the global result"""
        return self.buf.tensor

    def step(self):
        """One sharded partition2, entirely stream-ordered: count pass ->
        device all-gather of the counts -> the peer-storing partition kernel
        (bases derived on the device) -> device barrier (every rank's peer
        stores into this rank's shard have landed).  Returns the device pair
        [T_<rank, NT] (read it only when needed)."""
        self.ops.partition_counts(self.xs, self.pred, d_tot=self.d_tot)
        all_gather_dev(self.d_tot, self.d_counts, self.group)
        self.ops.partition2_peer(self.xs, self.pred, self.ptrs, self.shard, self.d_counts, self.rank)
        self.ops.rank_offsets(self.d_counts, self.world, self.rank, out=self.d_off)
        device_barrier(self.flag, self.group)
        return self.d_off

    def close(self):
        for ptr in self.opened:
            self.ops.ipc_close(ptr)
        self.opened = []
        self.buf.free()


class GpuC2Local:
    """C2 on one GPU's shard with the CUDA kernels (ixg_filter, ixg_flag_bitmap,
    ixg_segsum, ixg_seg_carry).  `shape` is the GLOBAL segment shape."""

    def __init__(self, xs, pred, shape, z_dtype=None):
        import torch

        from . import ops

        self.ops = ops
        self.xs, self.pred, self.shape = xs, pred, shape.to(torch.int64).contiguous()
        self.dev = xs.device
        n = xs.numel()
        self.ys = torch.empty(n, dtype=xs.dtype, device=self.dev)
        self.zs = torch.empty(n, dtype=z_dtype or xs.dtype, device=self.dev)
        self.dk = torch.empty(1, dtype=torch.int64, device=self.dev)
        self.tot = torch.empty(2, dtype=torch.int64, device=self.dev)
        self.scratch = torch.empty(1, dtype=torch.int64, device=self.dev)
        self.st = ops.Status(self.dev)
        self.k = 0
        self.bits = None
        self.d_ks = self.d_off = self.d_aggs = None

    def step_device(self, group=None):
        """The whole sharded C2 step with every count, offset and carry kept
        on the device (no host round trip): filter -> all-gather of the
        counts -> [K_r, K_total] -> the mkFlags bits of this rank's window
        [K_r, K_r + k_r) of the global outputs -> sgmSum of this rank's
        outputs -> all-gather of the segmented aggregates -> the carry of the
        ranks before, added before the first flag.  Outputs: ys / zs [0, *dk), global offset
        d_off[0]."""
        import torch
        import torch.distributed as dist

        from . import _lib as L

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        n = self.xs.numel()
        if self.d_ks is None:
            self.d_ks = torch.empty(world, dtype=torch.int64, device=self.dev)
            self.d_off = torch.empty(2, dtype=torch.int64, device=self.dev)
            self.d_aggs = torch.empty(2 * world, dtype=torch.int64, device=self.dev)
        self.ops.filter(self.xs, self.pred, L.VARIANT_ELIDED, self.st, ys=self.ys, d_count=self.dk)
        all_gather_dev(self.dk, self.d_ks, group)
        self.ops.rank_offsets(self.d_ks, world, rank, out=self.d_off)
        # the mkFlags bits of this rank's own outputs only: global positions
        # [K_r, K_r + k_r) (d_off[0], dk), k_r bits instead of all K_total
        self.bits = self.ops.flag_bitmap(self.shape, n, d_nbits=self.dk, bits=self.bits, d_lo=self.d_off)
        self.ops.segsum(self.ys, n, self.bits, 0, self.zs, 0, False, self.tot, self.st, d_n=self.dk)
        all_gather_dev(self.tot, self.d_aggs, group)
        self.ops.seg_carry(self.bits, 0, self.zs, n, 0, self.scratch, self.st, d_n=self.dk, d_aggs=self.d_aggs,
                           rank=rank)

    def filter(self) -> int:
        from . import _lib as L

        self.ops.filter(self.xs, self.pred, L.VARIANT_ELIDED, self.st, ys=self.ys, d_count=self.dk)
        self.k = int(self.dk.item())
        return self.k

    def flag_bitmap(self, k_total: int) -> None:
        self.bits = self.ops.flag_bitmap(self.shape, k_total)

    def segsum(self, flag_base: int):
        self.ops.segsum(self.ys, self.k, self.bits, flag_base, self.zs, 0, False, self.tot, self.st)
        v, f = self.tot.cpu().tolist()
        return v, bool(f)

    def seg_carry(self, flag_base: int, carry_v: int) -> None:
        self.ops.seg_carry(self.bits, flag_base, self.zs, self.k, carry_v, self.scratch, self.st)
