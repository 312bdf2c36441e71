"""Multi-GPU sharding of the hot path.

One process per GPU (torch.distributed, NCCL on the GPU box; gloo for the
CPU tests).  Inputs are sharded contiguously; the only exchanges are tiny
all-gathers of per-rank totals -- the data never moves:

* partition2 (C5): all-gather of each rank's true-count; rank r's local
  result [its trues | its falses] is exactly two runs of the global result,
  at [T_<r, T_<r + T_r) and [NT + F_<r, NT + F_<r + F_r).
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


def partition2_sharded(local, group=None):
    """Sharded partition2 (C5).  `local.partition2()` -> (true count, size);
    returns (num_true_global, Runs of this rank's local [trues | falses])."""
    import torch.distributed as dist

    rank = dist.get_rank(group)
    t, size = local.partition2()
    rows = all_gather_ints([t, size], group)
    return partition2_runs([r[0] for r in rows], [r[1] for r in rows], rank)


# ----------------------------------------------------------------- GPU backend
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
