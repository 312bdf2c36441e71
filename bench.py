#!/usr/bin/env python
"""bench.py -- the driver's benchmark contract for the B200 index-array path.

Headline workload (BASELINE.json configs[1], the metric's single-GPU config):
  c2 = filter (x >= 0) + mkFlags (flag array from a segment shape) + sgmSum
  (segmented inclusive sum) over N = 2^28 int32 per GPU, m = 2^20 segments.
A "step" is one pass of the pipeline over one batch (the whole N).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2|c1|c3|c4|c5] [--quick]

Prints ONE JSON line on rank 0.  `value` is whole-job Gelem/s with inputs
resident in HBM (device-timed with CUDA events, max over ranks); `e2e` is
the same metric through the public C-ABI call with pinned host buffers and
the H2D/D2H copies inside the timed region; `roofline` is the dominant
kernel's algorithmic bytes / its event-timed duration against the measured
HBM copy peak; `cpu_baseline` is the oracle port (oracle/, OpenMP, all host
threads) on the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gelem/s and HBM GB/s (% of roofline), checked vs elided speedup, at 1/2/4/8 B200"
FALLBACK_HBM = 6650.0


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                s, m = float(parts[0]), float(parts[1])
            except ValueError:
                continue
            sm.append(s)
            mx.append(m)
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        load = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- dist
def dist_init():
    import torch

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        # IXG_DIST_BACKEND=gloo: a functional check of the multi-rank path
        # with fewer GPUs than ranks (ranks share devices round-robin; no
        # kernel waits on another rank, only host collectives)
        backend = os.environ.get("IXG_DIST_BACKEND", "nccl")
        dev = local % torch.cuda.device_count()
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    return rank, ws, local


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


# ----------------------------------------------------------------- workloads
class C2:
    """filter + mkFlags + sgmSum (corpus/c2_filter_sgmsum.ixl)."""

    name = "c2"

    scaling = "weak"  # N per GPU

    def describe(self, quick, ws):
        self.N = (1 << 22) if quick else (1 << 28)
        self.m = (1 << 14) if quick else (1 << 20)
        self.workload = (f"c2 = filter (x >= 0) + mkFlags + sgmSum: N=2^{self.N.bit_length() - 1} int32 uniform "
                         f"[-128,127] per GPU, m=2^{self.m.bit_length() - 1} segments per GPU (i64 shape, sum = k, "
                         ">=1% empty), zs int32" + (f"; {ws} contiguous shards, device all-gathers of counts and "
                                                     "segmented aggregates" if ws > 1 else ""))

    def __init__(self, quick, rank, ws):
        from paper_2506_23058_b200 import gen
        from paper_2506_23058_b200.pred import Pred

        self.describe(quick, ws)
        self.p = Pred.ge(0)
        self.rank, self.ws = rank, ws
        # each rank owns one contiguous shard of the global xs
        self.xs_h = gen.uniform(0, self.N, -128, 127, np.int32, offset=rank * self.N)
        self.k = int(np.count_nonzero(self.xs_h >= 0))
        if ws > 1:
            # weak scaling: the global problem is ws shards of N; the segment
            # shape covers ALL shards' outputs (m per GPU, sum = global k)
            from paper_2506_23058_b200 import dist as D

            ks = [r[0] for r in D.all_gather_ints([self.k])]
            self.k_total = sum(ks)
            self.shape_h = gen.segment_shape(1, self.m * ws, self.k_total)
        else:
            self.k_total = self.k
            self.shape_h = gen.segment_shape(1 + rank, self.m, self.k)

    def setup_device(self):
        import torch

        from paper_2506_23058_b200 import ops

        dev = torch.device("cuda")
        self.xs = torch.from_numpy(self.xs_h).to(dev)
        self.shape = torch.from_numpy(self.shape_h).to(dev)
        self.ys = torch.empty(self.N, dtype=torch.int32, device=dev)
        self.zs = torch.empty(self.N, dtype=torch.int32, device=dev)
        self.dk = torch.empty(1, dtype=torch.int64, device=dev)
        self.st = ops.Status(dev)
        if self.ws > 1:
            from paper_2506_23058_b200 import dist as D

            self.local = D.GpuC2Local(self.xs, self.p, self.shape)
            self.local.ys, self.local.zs, self.local.dk, self.local.st = self.ys, self.zs, self.dk, self.st

    def step(self, variant):
        from paper_2506_23058_b200 import ops

        if self.ws > 1:
            self.local.step_device()  # counts, offsets and carries stay on the device
            return
        ops.c2(self.xs, self.p, self.shape, variant, self.st, ys=self.ys, zs=self.zs, d_k=self.dk)

    def check(self, want):
        k = int(self.dk.item())
        s = self.st.read()
        ok = (s.ok and not s.narrow and k == self.k)
        if want is not None:
            ok = ok and np.array_equal(self.ys[:k].cpu().numpy(), want[0]) and np.array_equal(
                self.zs[:k].cpu().numpy(), want[1])
        return ok

    def units(self):
        return self.N

    def algo_bytes_step(self):
        return 4 * self.N + 8 * self.m + 8 * self.k

    def kernel(self):
        from paper_2506_23058_b200 import _lib as L

        if self.ws == 1:
            # one pass: xs read once, ys and zs written once; the mkFlags
            # bitmap it also reads (k/8 B) is an intermediate, which
            # SURVEY.md §8(d) counts as zero
            return (L.K_FILTER_FUSED, 4 * self.N + 8 * self.k,
                    "k_filter_b<int32,kSeg> (filter + sgmSum in one pass: 48 KB TMA tiles, runs leave as phase-shifted bulk stores, two look-back chains)")
        # sharded: the filter pass; the sgmSum pass is reported alongside
        return L.K_FILTER_FUSED, 4 * self.N + 4 * self.k, "k_filter_b<int32> (single-pass filter, 48 KB TMA tiles)"

    def kernels_extra(self):
        from paper_2506_23058_b200 import _lib as L

        if self.ws == 1:
            return []
        return [(L.K_SEGSUM, 8 * self.k, "k_segsum_b<int32,int32> (sgmSum over ys, flags from the mkFlags bitmap)")]

    def checked_families(self):
        """CHECKED C2: the scans (filter offsets -> inds i64, mkFlags starts,
        sgmSum over the i64 flag array) and the checked scatters (ys, flags);
        bytes = what each launch must read and write."""
        from paper_2506_23058_b200 import _lib as L

        n, m, k = self.N, self.m, self.k
        return [(L.K_SEGSUM, 12 * n + 16 * k, "k_segsum_b x2 (pred -> offs -> inds i64; sgmSum over the i64 "
                                              "flag array + ys -> zs), big-tile scans"),
                (L.K_SCAN, 16 * m, "k_scan (mkFlags segment starts)"),
                (L.K_SCATTER, 12 * n + 4 * k + 24 * m, "k_scatter_sa x2 (ys, flags; claims in set-associative shared windows)")]

    def checked_launches(self, kid):
        from paper_2506_23058_b200 import _lib as L

        return {L.K_SEGSUM: 2, L.K_SCATTER: 2}.get(kid, 1)

    def e2e_step(self, bufs):
        """pinned host -> device, pipeline, k -> host, ys/zs -> host."""
        from paper_2506_23058_b200 import ops

        xs_p, shape_p, ys_p, zs_p, variant = bufs
        self.xs.copy_(xs_p, non_blocking=True)
        self.shape.copy_(shape_p, non_blocking=True)
        if self.ws > 1:
            self.local.step_device()
            k = int(self.dk.item())
        else:
            ops.c2(self.xs, self.p, self.shape, variant, self.st, ys=self.ys, zs=self.zs, d_k=self.dk)
            k = int(self.dk.item())
        ys_p[:k].copy_(self.ys[:k], non_blocking=True)
        zs_p[:k].copy_(self.zs[:k], non_blocking=True)
        return 4 * self.N + 8 * self.m, 8 + 8 * k

    def e2e_bufs(self, variant):
        import torch

        return (torch.from_numpy(self.xs_h).pin_memory(), torch.from_numpy(self.shape_h).pin_memory(),
                torch.empty(self.N, dtype=torch.int32).pin_memory(),
                torch.empty(self.N, dtype=torch.int32).pin_memory(), variant)

    def e2e_pipeline(self, variant, steps):
        """pipelined e2e (see pipeline_e2e): xs / shape in, ys[:k] / zs[:k] out"""
        import torch

        from paper_2506_23058_b200 import ops

        if self.ws > 1:
            return None
        dev = torch.device("cuda")
        host = dict(xs=torch.from_numpy(self.xs_h).pin_memory(), sh=torch.from_numpy(self.shape_h).pin_memory())

        def make_set():
            return dict(xs=torch.empty(self.N, dtype=torch.int32, device=dev),
                        sh=torch.empty(len(self.shape_h), dtype=torch.int64, device=dev),
                        ys=torch.empty(self.N, dtype=torch.int32, device=dev),
                        zs=torch.empty(self.N, dtype=torch.int32, device=dev),
                        dk=torch.empty(1, dtype=torch.int64, device=dev), st=ops.Status(dev),
                        ys_p=torch.empty(self.N, dtype=torch.int32).pin_memory(),
                        zs_p=torch.empty(self.N, dtype=torch.int32).pin_memory(),
                        k_p=torch.empty(1, dtype=torch.int64).pin_memory())

        def h2d(b):
            b["xs"].copy_(host["xs"], non_blocking=True)
            b["sh"].copy_(host["sh"], non_blocking=True)

        def compute(b):
            ops.c2(b["xs"], self.p, b["sh"], variant, b["st"], ys=b["ys"], zs=b["zs"], d_k=b["dk"])
            b["k_p"].copy_(b["dk"], non_blocking=True)

        def d2h(b):  # runs after the compute event completed: k is on the host
            k = int(b["k_p"].item())
            b["ys_p"][:k].copy_(b["ys"][:k], non_blocking=True)
            b["zs_p"][:k].copy_(b["zs"][:k], non_blocking=True)
            return 8 + 8 * k

        ms, d2h_bytes = pipeline_e2e(make_set, h2d, compute, d2h, steps)
        return ms, 4 * self.N + 8 * len(self.shape_h), d2h_bytes

    def cpu_run(self, xs, shape, threads=0):
        from oracle import ixoracle as O

        return O.par_c2_i32(self.p, xs, shape, threads)

    def cpu_sample(self, budget_s):
        """the full per-GPU workload when it fits the budget, else a prefix."""
        return self.xs_h, self.shape_h, self.N


class C1:
    """partition2 (corpus partition2.ixl), 2^20 int32 (BASELINE configs[0]);
    with --config c5 the same program at 2^32 (configs[4])."""

    name = "c1"

    def describe(self, quick, ws, big=False):
        self.name = "c5" if big else "c1"
        self.big = big
        # C5: 2^32 in total over the GPUs (strong scaling); C1: 2^20 per GPU
        self.scaling = "strong" if big else "weak"
        self.N = ((1 << 24) if quick else (1 << 32) // ws) if big else (1 << 20)
        self.workload = (f"partition2 (x < 0), N=2^{self.N.bit_length() - 1} int32 uniform over int32"
                         + (f" per GPU (2^{(self.N * ws).bit_length() - 1} total)" if big else "")
                         + (f"; {ws} contiguous shards: device all-gather of per-shard true counts -> each shard's "
                            "two output runs of the global result, moved to the shards owning their positions"
                            if ws > 1 else ""))

    def __init__(self, quick, rank, ws, big=False):
        from paper_2506_23058_b200 import gen
        from paper_2506_23058_b200.pred import Pred

        self.describe(quick, ws, big)
        self.p = Pred.lt(0)
        self.xs_h = None if big else gen.uniform(0, self.N, -(1 << 31), (1 << 31) - 1, np.int32, offset=rank * self.N)
        self.rank, self.ws = rank, ws

    def setup_device(self):
        import torch

        from paper_2506_23058_b200 import ops

        dev = torch.device("cuda")
        if self.big:
            self.xs = ops.gen_uniform(self.N, -(1 << 31), (1 << 31) - 1, 0, torch.int32, offset=self.rank * self.N)
        else:
            self.xs = torch.from_numpy(self.xs_h).to(dev)
        self.ys = torch.empty(self.N, dtype=torch.int32, device=dev)
        self.dnt = torch.empty(1, dtype=torch.int64, device=dev)
        self.st = ops.Status(dev)
        self.sets = None
        if not self.big:
            # C1's 8 MB working set would stay in the 126 MB L2: the steps
            # rotate over 32 copies of (xs, ys) -- 256 MB, twice the L2 -- so
            # every step starts cold, with no flush kernel between the steps
            # (whose shared-memory reconfiguration would sit inside the next
            # step's start event)
            self.sets = [(self.xs.clone(), torch.empty_like(self.ys), torch.empty_like(self.dnt)) for _ in range(32)]
            self.turn = 0
        if self.ws > 1:
            from paper_2506_23058_b200 import dist as D

            self.local = D.GpuPart2Local(self.xs, self.p)
            self.local.ys, self.local.dnt, self.local.st = self.ys, self.dnt, self.st
            # default: the exchange fused into the partition kernel (peer
            # stores into IPC-mapped shards); IXG_C5_EXCHANGE=nccl selects the
            # NCCL all-to-all after the local partition
            self.peer = None
            self.exchange = os.environ.get("IXG_C5_EXCHANGE", "fused")
            if self.exchange == "fused":
                try:
                    self.peer = D.GpuPart2PeerLocal(self.xs, self.p)
                except Exception as e:  # no CUDA IPC between the ranks' GPUs
                    self.exchange = f"nccl (fused setup failed: {type(e).__name__})"
            self.workload += ("; exchange: peer stores over NVLink fused into the partition kernel (CUDA IPC)"
                              if self.exchange == "fused" else f"; exchange: one NCCL all-to-all per class "
                              f"({self.exchange})")

    def step(self, variant):
        from paper_2506_23058_b200 import ops

        if self.ws > 1:
            from paper_2506_23058_b200 import dist as D

            if self.peer is not None:
                self.d_off = self.peer.step()  # [T_<rank, NT] on the device; no host round trip
            else:
                self.nt_global, self.runs, self.mine = D.partition2_sharded(self.local, exchange=True)
            return
        if self.sets is not None:
            self.xs, self.ys, self.dnt = self.sets[self.turn]
            self.turn = (self.turn + 1) % len(self.sets)
        ops.partition2(self.xs, self.p, variant, self.st, ys=self.ys, d_nt=self.dnt)

    def check(self, want):
        s = self.st.read()
        ok = s.ok
        if want is not None:
            ok = ok and int(self.dnt.item()) == want[0] and np.array_equal(self.ys.cpu().numpy(), want[1])
        return ok

    def units(self):
        return self.N

    def algo_bytes_step(self):
        return 8 * self.N + 8

    def kernel(self):
        from paper_2506_23058_b200 import _lib as L

        # algorithmic bytes: xs read once, ys written once (the kernel reads xs
        # once per class segment; `traffic` shows the measured DRAM bytes)
        return L.K_PLACE, 8 * self.N, "k_filter_b<int32,NS=2> (stable partition: 2 class segments on one look-back chain)"

    def checked_families(self):
        """CHECKED partition2: the index scan (pred -> inds i64) and the
        checked scatter (claims privatised per tile)."""
        from paper_2506_23058_b200 import _lib as L

        n = self.N
        return [(L.K_CLASS_COUNT, 4 * n, "k_class_count (num_true)"),
                (L.K_SEGSUM, 12 * n, "k_segsum_b<ScanPart2Inds> (pred -> indices i64, big-tile scan)"),
                (L.K_SCATTER, 16 * n, "k_scatter_sa (indices + xs -> ys; claims in set-associative shared windows)")]

    def e2e_bufs(self, variant):
        import torch

        xs_h = self.xs_h if self.xs_h is not None else self.xs.cpu().numpy()
        return (torch.from_numpy(xs_h).pin_memory(), torch.empty(self.N, dtype=torch.int32).pin_memory(), variant)

    @property
    def e2e_steps(self):
        """C1's pipelined e2e step is ~0.1 ms: time 100 of them (C5: the default)"""
        return 0 if (self.big or self.ws > 1) else 100

    def e2e_pipeline(self, variant, steps):
        """pipelined e2e for C1 (see pipeline_e2e); C5 at 2^32 keeps the
        sequential e2e (two pinned 16 GiB output sets would be needed)"""
        import torch

        from paper_2506_23058_b200 import ops

        if self.ws > 1 or self.big:
            return None
        host = torch.from_numpy(self.xs_h).pin_memory()

        def make_set():
            return dict(xs=torch.empty_like(self.xs), ys=torch.empty_like(self.ys), dnt=torch.empty_like(self.dnt),
                        ys_p=torch.empty(self.N, dtype=torch.int32).pin_memory(),
                        nt_p=torch.empty(1, dtype=torch.int64).pin_memory())

        def h2d(b):
            b["xs"].copy_(host, non_blocking=True)

        def compute(b):
            ops.partition2(b["xs"], self.p, variant, self.st, ys=b["ys"], d_nt=b["dnt"])

        def d2h(b):
            b["ys_p"].copy_(b["ys"], non_blocking=True)
            b["nt_p"].copy_(b["dnt"], non_blocking=True)
            return 4 * self.N + 8

        # partition2's result has a fixed size (n): no host wait per step
        ms, d2h_bytes = pipeline_e2e(make_set, h2d, compute, d2h, steps, host_sync=False)
        return ms, 4 * self.N, d2h_bytes

    def e2e_step(self, bufs):
        import torch

        from paper_2506_23058_b200 import ops

        xs_p, ys_p, variant = bufs
        self.xs.copy_(xs_p, non_blocking=True)
        if self.ws > 1:
            from paper_2506_23058_b200 import dist as D

            if self.peer is not None:
                self.peer.step()
                ys_p.copy_(self.peer.out, non_blocking=True)
            else:
                _, _, mine = D.partition2_sharded(self.local, exchange=True)
                ys_p[:mine.numel()].copy_(mine, non_blocking=True)
            torch.cuda.synchronize()
            return 4 * self.N, 4 * self.N
        ops.partition2(self.xs, self.p, variant, self.st, ys=self.ys, d_nt=self.dnt)
        ys_p.copy_(self.ys, non_blocking=True)
        int(self.dnt.item())
        return 4 * self.N, 4 * self.N + 8

    def dropin(self):
        """C1 as BASELINE configs[0] states it: the program run through the
        drop-in eval_program (oracle.py:332-333 signature) with a Python list
        argument, verifier-selected variants, a Python list result -- and
        where the time of such a call goes."""
        import json as _json

        import torch

        from paper_2506_23058_b200 import executor, ir

        with open(os.path.join(ROOT, "paper_2506_23058_b200", "data", "programs.json")) as f:
            prog = ir.from_json(_json.load(f)["ref:partition2.ixl"]["program"])
        xs_list = self.xs_h.astype(np.int64).tolist()
        dev = torch.device("cuda")

        def med(fn, reps=7):
            ts = []
            for _ in range(reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = fn()
                torch.cuda.synchronize()
                ts.append(time.perf_counter() - t0)
            return statistics.median(ts) * 1e3, r

        t_call, (nt, ys) = med(lambda: executor.eval_program(prog, "partition2", [self.p, xs_list]))
        ok = nt == int((self.xs_h < 0).sum()) and len(ys) == len(xs_list)
        t_marshal, xd = med(lambda: executor._dev_i64(xs_list, dev))
        t_dev, _ = med(lambda: executor.eval_program(prog, "partition2", [self.p, xd], as_tensors=True))
        yd = executor.eval_program(prog, "partition2", [self.p, xd], as_tensors=True)[1]
        t_ret, _ = med(lambda: yd.cpu().numpy().tolist())
        return {"value": round(self.N / (t_call * 1e-3) / 1e9, 4), "unit": "Gelem/s",
                "ms_per_call": round(t_call, 3), "result_ok": bool(ok),
                "call": "paper_2506_23058_b200.eval_program(partition2.ixl, 'partition2', [Pred(x < 0), list of 2^20 "
                        "ints]) -> (int, list): selection, marshalling, kernels, status read, list result",
                "shares_ms": {"marshal_list_to_device": round(t_marshal, 3),
                              "device_call_incl_dispatch_and_status_read": round(t_dev, 3),
                              "result_to_list": round(t_ret, 3)}}

    def cpu_run(self, xs, threads=0):
        from oracle import ixoracle as O

        return O.par_partition2_i32(self.p, xs, threads)

    def cpu_sample(self, budget_s):
        if self.xs_h is None:
            from paper_2506_23058_b200 import gen

            n = min(self.N, 1 << 28)
            return gen.uniform(0, n, -(1 << 31), (1 << 31) - 1, np.int32), n
        return self.xs_h, self.N


class C3:
    """scatter dst is vs, n = m = 2^29 (BASELINE configs[2]): `is` = the
    partition2 destination index of random xs (two monotone streams, a true
    permutation); ELIDED = Sc1 (sc_bij: no init, no checks), CHECKED =
    sc_any (dst init + OOB test + idempotence check)."""

    name = "c3"
    cpu_desc = ("oracle/ixoracle_par.c ixo_par_scatter_i32 (OpenMP restatement of oracle.py:294-305 with its "
                "idempotence check: claim bitmap + value re-check)")

    scaling = "weak"  # an independent scatter per GPU (replicas)

    def describe(self, quick, ws, perm="streams"):
        self.N = (1 << 22) if quick else (1 << 29)
        self.perm = perm
        self.name = "c3r" if perm == "random" else "c3"
        if perm == "random":
            pat = "a uniformly random permutation (torch.randperm, Philox)"
        else:
            pat = "partition2 indices of random xs (i64 permutation, two monotone streams)"
        self.workload = (f"scatter dst is vs: n = m = 2^{self.N.bit_length() - 1}, is = {pat}, vs int32, "
                         "dst int32 zeros" + (f"; {ws} independent replicas" if ws > 1 else ""))

    def __init__(self, quick, rank, ws, perm="streams"):
        self.describe(quick, ws, perm)
        self.rank, self.ws = rank, ws

    def setup_device(self):
        import torch

        from paper_2506_23058_b200 import ops

        dev = torch.device("cuda")
        if self.perm == "random":
            g = torch.Generator(device=dev)
            g.manual_seed(11 + self.rank)
            self.is_ = torch.randperm(self.N, generator=g, device=dev, dtype=torch.int64)
        else:
            xs = ops.gen_uniform(self.N, -(1 << 31), (1 << 31) - 1, 11, torch.int32, offset=self.rank * self.N)
            c = xs < 0
            t = torch.cumsum(c, 0, dtype=torch.int64)
            nt = t[-1]
            i1 = torch.arange(1, self.N + 1, device=dev, dtype=torch.int64)
            self.is_ = torch.where(c, t - 1, nt + (i1 - t) - 1)
            del xs, c, t, i1
        self.vs = ops.gen_uniform(self.N, -(1 << 31), (1 << 31) - 1, 12, torch.int32, offset=self.rank * self.N)
        self.dst = torch.zeros(self.N, dtype=torch.int32, device=dev)
        self.out = torch.empty_like(self.dst)
        self.st = ops.Status(dev)

    def step(self, variant):
        from paper_2506_23058_b200 import _lib as L
        from paper_2506_23058_b200 import ops

        if variant == L.VARIANT_ELIDED:
            ops.scatter(self.out, self.is_, self.vs, 0, self.st)
        else:
            self.out.copy_(self.dst)  # dst init (the reference copies dst, oracle.py:295)
            ops.scatter(self.out, self.is_, self.vs, L.V_CONFLICT | L.V_INIT, self.st)

    def checked_families(self):
        from paper_2506_23058_b200 import _lib as L

        fams = [(L.K_SCATTER, 16 * self.N, "k_scatter_sa (claims in 2-way set-associative shared-memory windows)"
                 if self.perm != "random" else "k_scatter_pc<u32> over the binned pairs (8 + 4 + 4 B)")]
        if self.perm == "random":
            fams.append((L.K_BIN, 20 * self.N, "k_bin_partition (12 B in, 8 B binned pairs out)"))
        return fams

    def check(self, want):
        import torch

        ok = self.st.read().ok
        # a permutation scatter: out[is] == vs everywhere
        ok = ok and bool(torch.equal(self.out[self.is_], self.vs))
        return ok

    def units(self):
        return self.N

    def algo_bytes_step(self):
        return 16 * self.N

    def kernel(self):
        from paper_2506_23058_b200 import _lib as L

        if self.perm == "random":  # binned: the second pass over the (u32 index, value) pairs dominates
            return (L.K_SCATTER, 12 * self.N,
                    "k_scatter_ti<u32,int32> over the window-binned pairs (8 MB destination windows; u32 index + "
                    "i32 value read, i32 dst written); k_bin_partition before it")
        return (L.K_SCATTER, 16 * self.N,
                "k_scatter_t<int32> (TMA-staged 4096-element tiles, striped stores; is i64 + vs i32 read, dst i32 written)")

    def kernels_extra(self):
        from paper_2506_23058_b200 import _lib as L

        if self.perm != "random":
            return []
        return [(L.K_BIN, 20 * self.N, "k_bin_partition (is i64 + vs i32 read, u32 + i32 binned pairs written)")]

    def e2e_bufs(self, variant):
        import torch

        return (self.is_.cpu().pin_memory(), self.vs.cpu().pin_memory(), torch.empty(self.N, dtype=torch.int32).pin_memory(),
                variant)

    def e2e_pipeline(self, variant, steps):
        """pipelined e2e (see pipeline_e2e): is / vs in, the scattered dst out"""
        import torch

        from paper_2506_23058_b200 import ops

        if self.ws > 1:
            return None
        host = dict(is_=self.is_.cpu().pin_memory(), vs=self.vs.cpu().pin_memory())

        def make_set():
            return dict(is_=torch.empty_like(self.is_), vs=torch.empty_like(self.vs), out=torch.empty_like(self.out),
                        out_p=torch.empty(self.N, dtype=torch.int32).pin_memory())

        def h2d(b):
            b["is_"].copy_(host["is_"], non_blocking=True)
            b["vs"].copy_(host["vs"], non_blocking=True)

        def compute(b):
            ops.scatter(b["out"], b["is_"], b["vs"], 0, self.st)

        def d2h(b):
            b["out_p"].copy_(b["out"], non_blocking=True)
            return 4 * self.N

        ms, d2h_bytes = pipeline_e2e(make_set, h2d, compute, d2h, steps)
        return ms, 12 * self.N, d2h_bytes

    def e2e_step(self, bufs):
        from paper_2506_23058_b200 import ops

        is_p, vs_p, out_p, variant = bufs
        self.is_.copy_(is_p, non_blocking=True)
        self.vs.copy_(vs_p, non_blocking=True)
        ops.scatter(self.out, self.is_, self.vs, 0, self.st)
        out_p.copy_(self.out, non_blocking=True)
        return 12 * self.N, 4 * self.N

    def cpu_run(self, dst, is_, vs, out, threads=0):
        from oracle import ixoracle as O

        return O.par_scatter_i32(dst, is_, vs, threads, out=out)

    def cpu_sample(self, budget_s):
        """the full per-GPU workload (same is / vs / dst as the device arm)"""
        if not hasattr(self, "is_"):
            self.setup_device()
        out = np.empty(self.N, np.int32)
        return np.zeros(self.N, np.int32), self.is_.cpu().numpy(), self.vs.cpu().numpy(), out, self.N


class C4:
    """CSR flat gather map2 (\\v c -> v * x[c]) values indices (BASELINE
    configs[3]): nnz = 2^28, num_cols = 2^20, indices sorted within rows of
    64; ELIDED = csrg (Range proved), CHECKED = csrg_any (bounds checks)."""

    name = "c4"
    cpu_desc = "oracle/ixoracle_par.c ixo_par_csrg_i32 (OpenMP restatement with the bounds check of oracle.py:177-184)"

    scaling = "weak"  # an nnz shard per GPU, x replicated

    def describe(self, quick, ws):
        self.N = (1 << 22) if quick else (1 << 28)
        self.ncols = 1 << 20
        self.workload = (f"CSR gather v * x[c]: nnz = 2^{self.N.bit_length() - 1} per GPU, num_cols = 2^20, values/x "
                         "int32 in [-2^15, 2^15), indices i64 sorted within rows of 64")

    def __init__(self, quick, rank, ws):
        self.describe(quick, ws)
        self.rank, self.ws = rank, ws

    def setup_device(self):
        import torch

        from paper_2506_23058_b200 import ops

        dev = torch.device("cuda")
        self.x = ops.gen_uniform(self.ncols, -(1 << 15), (1 << 15) - 1, 21, torch.int32)
        self.vals = ops.gen_uniform(self.N, -(1 << 15), (1 << 15) - 1, 22, torch.int32, offset=self.rank * self.N)
        idx = ops.gen_uniform(self.N, 0, self.ncols - 1, 23, torch.int64, offset=self.rank * self.N)
        self.idx = idx.view(-1, 64).sort(dim=1).values.reshape(-1).contiguous()
        self.out = torch.empty(self.N, dtype=torch.int32, device=dev)
        self.st = ops.Status(dev)

    def step(self, variant):
        from paper_2506_23058_b200 import ops

        ops.csr_gather(self.x, self.vals, self.idx, variant, self.st, out=self.out)

    def check(self, want):
        import torch

        s = self.st.read()
        ref = (self.vals[:4096].long() * self.x[self.idx[:4096]].long()).int()
        return s.ok and bool(torch.equal(self.out[:4096], ref))

    def units(self):
        return self.N

    def algo_bytes_step(self):
        return 16 * self.N + 4 * self.ncols

    def kernel(self):
        from paper_2506_23058_b200 import _lib as L

        return L.K_CSR_GATHER, 16 * self.N + 4 * self.ncols, "k_csr_gather<int32>"

    def checked_families(self):
        from paper_2506_23058_b200 import _lib as L

        return [(L.K_CSR_GATHER, 16 * self.N + 4 * self.ncols, "k_csr_gather (every x[c] bounds-checked)")]

    def l2_ceiling(self, kms):
        """C4's binding roof is L2's random-sector rate, not HBM: measured
        here (outside the timed region) with hashed 4-byte reads of an
        L2-resident x of the same size and nothing else."""
        import ctypes

        import torch
        from cuda.bindings import driver

        from paper_2506_23058_b200 import jit

        src = ("typedef unsigned long long u64;\n"
               "__device__ __forceinline__ u64 mix(u64 z){z=(z^(z>>30))*0xBF58476D1CE4E5B9ULL;"
               "z=(z^(z>>27))*0x94D049BB133111EBULL;return z^(z>>31);}\n"
               'extern "C" __global__ void __launch_bounds__(256) rand_gather(const int* __restrict__ x, int mask, '
               "long long n, int* __restrict__ out){const long long st=(long long)gridDim.x*blockDim.x;int a=0;"
               "for(long long i=(long long)blockIdx.x*blockDim.x+threadIdx.x;i<n;i+=st*8){\n#pragma unroll\n"
               "for(int u=0;u<8;++u)a+=__ldg(&x[(int)(mix((u64)(i+u*st))&(u64)mask)]);}if(a==0x7fffffff)out[0]=a;}")
        kern = jit._Kernel(src, ("rand_gather",))
        x = self.x if self.x.numel() & (self.x.numel() - 1) == 0 else self.x[: 1 << (self.x.numel().bit_length() - 1)]
        out = torch.zeros(1, dtype=torch.int32, device=x.device)
        n = self.N
        vals = [ctypes.c_void_p(x.data_ptr()), ctypes.c_int(x.numel() - 1), ctypes.c_longlong(n),
                ctypes.c_void_p(out.data_ptr())]
        argv = (ctypes.c_void_p * len(vals))(*[ctypes.addressof(v) for v in vals])
        grid = torch.cuda.get_device_properties(x.device).multi_processor_count * 8

        def launch():
            (err,) = driver.cuLaunchKernel(kern.fns["rand_gather"], grid, 1, 1, 256, 1, 1, 0,
                                           torch.cuda.current_stream().cuda_stream, ctypes.addressof(argv), 0)
            assert int(err) == 0

        for _ in range(3):
            launch()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            launch()
        b.record()
        torch.cuda.synchronize()
        peak = n / (a.elapsed_time(b) / 5) / 1e6
        got = self.N / kms / 1e6
        return {"bound": "l2 (one 32-B sector per random 4-B read of x)", "unit": "G gathers/s",
                "achieved": round(got, 1), "peak": round(peak, 1), "frac": round(got / peak, 4),
                "peak_kind": "measured live: hashed 4-B reads of an L2-resident x of the same size, no streams",
                "note": "C4 also streams 16 B/nnz through L2 while gathering"}

    def e2e_bufs(self, variant):
        import torch

        return (self.vals.cpu().pin_memory(), self.idx.cpu().pin_memory(), torch.empty(self.N, dtype=torch.int32).pin_memory(),
                variant)

    def e2e_pipeline(self, variant, steps):
        """pipelined e2e (see pipeline_e2e): values / indices in, products out"""
        import torch

        from paper_2506_23058_b200 import ops

        if self.ws > 1:
            return None
        host = dict(vals=self.vals.cpu().pin_memory(), idx=self.idx.cpu().pin_memory())

        def make_set():
            return dict(vals=torch.empty_like(self.vals), idx=torch.empty_like(self.idx), out=torch.empty_like(self.out),
                        out_p=torch.empty(self.N, dtype=torch.int32).pin_memory())

        def h2d(b):
            b["vals"].copy_(host["vals"], non_blocking=True)
            b["idx"].copy_(host["idx"], non_blocking=True)

        def compute(b):
            ops.csr_gather(self.x, b["vals"], b["idx"], variant, self.st, out=b["out"])

        def d2h(b):
            b["out_p"].copy_(b["out"], non_blocking=True)
            return 4 * self.N

        ms, d2h_bytes = pipeline_e2e(make_set, h2d, compute, d2h, steps)
        return ms, 12 * self.N, d2h_bytes

    def e2e_step(self, bufs):
        from paper_2506_23058_b200 import ops

        v_p, i_p, o_p, variant = bufs
        self.vals.copy_(v_p, non_blocking=True)
        self.idx.copy_(i_p, non_blocking=True)
        ops.csr_gather(self.x, self.vals, self.idx, variant, self.st, out=self.out)
        o_p.copy_(self.out, non_blocking=True)
        return 12 * self.N, 4 * self.N

    def cpu_run(self, x, vals, idx, out, threads=0):
        from oracle import ixoracle as O

        return O.par_csrg_i32(x, vals, idx, threads, out=out)

    def cpu_sample(self, budget_s):
        """the full per-GPU workload (same x / values / indices as the device arm)"""
        if not hasattr(self, "vals"):
            self.setup_device()
        return (self.x.cpu().numpy(), self.vals.cpu().numpy(), self.idx.cpu().numpy(), np.empty(self.N, np.int32),
                self.N)


# ----------------------------------------------------------------- timing
def link_probe(h2d_bytes, d2h_bytes, reps=3):
    """The box's pinned-copy ceiling for an e2e step: the step's H2D bytes
    alone, its D2H bytes alone, and both at once on two streams (PCIe is
    full duplex on most boxes, not all).  e2e.link_frac = duplex_ms / the
    e2e step: 1.0 means the step runs at the link."""
    import torch

    h2d_bytes, d2h_bytes = max(int(h2d_bytes), 1), max(int(d2h_bytes), 1)
    # at most 1 GiB each way (C5 moves 16 GiB): times scale with the bytes
    scale = max(h2d_bytes, d2h_bytes) / min(max(h2d_bytes, d2h_bytes), 1 << 30)
    nb_in, nb_out = max(1, int(h2d_bytes / scale)), max(1, int(d2h_bytes / scale))
    h_in = torch.empty(nb_in, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(nb_out, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(nb_in, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(nb_out, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        for _ in range(reps):
            fn()
        b.record(cur)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    def duplex():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    t_in = timed(lambda: d_in.copy_(h_in, non_blocking=True)) * scale
    t_out = timed(lambda: h_out.copy_(d_out, non_blocking=True)) * scale
    t_dup = timed(duplex) * scale
    del h_in, h_out, d_in, d_out
    return {"h2d_GBs": round(h2d_bytes / (t_in * 1e-3) / 1e9, 2), "d2h_GBs": round(d2h_bytes / (t_out * 1e-3) / 1e9, 2),
            "serial_ms": round(t_in + t_out, 3), "duplex_ms": round(t_dup, 3)}


def pipeline_e2e(make_set, h2d, compute, d2h, steps, warm=2, host_sync=True):
    """The e2e step as a server runs it: two device/host buffer sets and three
    streams, so step i's host->device copy overlaps step i-1's device->host
    read-back (PCIe is full duplex) and the kernels run between them.  Every
    step still copies its whole input in and its whole result out.  d2h(b) is
    called on the host once step b's compute has finished (so it may read a
    result size from a pinned scalar); host_sync=False when the result's size
    is fixed (the read-back then follows the compute on the device only, and
    the host never waits inside the loop).  Returns (ms per step, d2h bytes)."""
    import torch

    sets = [make_set() for _ in range(2)]
    for b in sets:
        b.update(e_h2d=torch.cuda.Event(), e_cmp=torch.cuda.Event(), e_d2h=torch.cuda.Event(), used=False)
    s_h2d, s_cmp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    out_bytes = []

    def issue(i):
        b = sets[i % 2]
        if b["used"]:
            s_h2d.wait_event(b["e_cmp"])  # compute(i-2) has read this set's inputs
        with torch.cuda.stream(s_h2d):
            h2d(b)
            b["e_h2d"].record(s_h2d)
        s_cmp.wait_event(b["e_h2d"])
        if b["used"]:
            s_cmp.wait_event(b["e_d2h"])  # D2H(i-2) has read this set's outputs
        with torch.cuda.stream(s_cmp):
            compute(b)
            b["e_cmp"].record(s_cmp)
        b["used"] = True

    def read_back(i):
        b = sets[i % 2]
        if host_sync:
            b["e_cmp"].synchronize()
        s_d2h.wait_event(b["e_cmp"])
        with torch.cuda.stream(s_d2h):
            out_bytes.append(d2h(b))
            b["e_d2h"].record(s_d2h)

    def run(n):
        for i in range(n):
            issue(i)
            if i > 0:
                read_back(i - 1)
        read_back(n - 1)
        for b in sets:
            if b["used"]:
                cur.wait_event(b["e_d2h"])

    run(warm)
    torch.cuda.synchronize()
    for b in sets:
        b["used"] = False
    out_bytes.clear()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record(cur)
    s_h2d.wait_stream(cur)
    w0 = time.perf_counter()
    run(steps)
    w1 = time.perf_counter()
    t1.record(cur)
    torch.cuda.synchronize()
    if os.environ.get("IXG_E2E_HOSTTIME"):  # diagnostics: host enqueue time per step
        print(f"pipeline_e2e: host {1e3 * (w1 - w0) / steps:.4f} ms/step, device {t0.elapsed_time(t1) / steps:.4f}",
              file=sys.stderr)
    return t0.elapsed_time(t1) / steps, max(out_bytes)


def time_steps(wl, variant, steps, warmup, ws, kernel_id=None):
    import torch

    from paper_2506_23058_b200 import _lib as L
    from paper_2506_23058_b200 import ops

    lib = L.load(require_device=True)
    for _ in range(warmup):
        wl.step(variant)
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    launches0 = ops.launch_count()
    if kernel_id:
        lib.ixg_timer_start(kernel_id)
    pre = getattr(wl, "pre_step", None)
    if pre is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            wl.step(variant)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
    else:
        # per-step event pairs: the L2 flush between steps is not timed
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for a, b in evs:
            pre()
            a.record()
            wl.step(variant)
            b.record()
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for a, b in evs) / steps
    launches = ops.launch_count() - launches0
    kms = None
    if kernel_id:
        import ctypes

        tot, cnt = ctypes.c_double(0), ctypes.c_int64(0)
        L.check(lib.ixg_timer_stop(ctypes.byref(tot), ctypes.byref(cnt)), "timer")
        kms = tot.value / max(cnt.value, 1)
    barrier(ws)
    return max_over_ranks(ms, ws), launches, kms


def run_ours(args):
    import torch

    from paper_2506_23058_b200 import _lib as L

    rank, ws, local = dist_init()
    wl = make_workload(args, rank, ws)
    wl.setup_device()
    hbm, peak_kind = _peaks()
    selected = L.VARIANT_ELIDED  # the verifier's selection for every site of c2 / partition2
    # parity of the measured configuration against the CPU port
    want = None
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_baseline(wl, args)
        want = cpu.pop("_result", None)
    wl.step(selected)
    torch.cuda.synchronize()
    parity = wl.check(want)

    sampler = ClockSampler(local)
    sampler.start()
    # soak so the clock sampler sees the loaded state
    t_end = time.time() + (0.3 if args.quick else 1.5)
    while True:
        wl.step(selected)
        # every rank must run the same number of steps (each step holds
        # collectives): stop when any rank is past its deadline
        if (time.time() >= t_end) if ws == 1 else max_over_ranks(float(time.time() >= t_end), ws) > 0:
            break
    torch.cuda.synchronize()
    kid, kbytes, kname = wl.kernel()
    # the step on its own (nothing but the pipeline's launches in the stream),
    # then the dominant kernel's duration from a second pass with event
    # pairs around each of its launches (events between kernels would also
    # serialise programmatic dependent launch)
    ms, launches, _ = time_steps(wl, selected, args.steps, args.warmup, ws)
    _, _, kms = time_steps(wl, selected, args.steps, args.warmup, ws, kid)
    clocks = sampler.stop()
    others = []
    for okid, obytes, oname in (wl.kernels_extra() if hasattr(wl, "kernels_extra") else []):
        _, _, oms = time_steps(wl, selected, max(5, args.steps // 5), 2, ws, okid)
        if oms:
            others.append({"kernel": oname, "kernel_ms": round(oms, 5), "algo_bytes_per_launch": obytes,
                           "achieved": round(obytes / (oms * 1e-3) / 1e9, 1),
                           "frac": round(obytes / (oms * 1e-3) / 1e9 / hbm, 4)})
    ms_chk = parity_chk = None
    chk_fams = []
    if ws == 1:  # the CHECKED pipeline is single-GPU (the sharded path is the verified one)
        ms_chk, _, _ = time_steps(wl, L.VARIANT_CHECKED, max(3, args.steps // 4), 2, ws)
        parity_chk = wl.check(want)
        # the CHECKED step's kernel families: device time per step (events on
        # the launching stream around every launch of the family) against the
        # bytes those launches must move
        for fkid, fbytes, fname in (wl.checked_families() if hasattr(wl, "checked_families") else []):
            steps_f = max(3, args.steps // 4)
            _, _, fms_launch = time_steps(wl, L.VARIANT_CHECKED, steps_f, 2, ws, fkid)
            nl = wl.checked_launches(fkid) if hasattr(wl, "checked_launches") else 1
            if fms_launch:
                fms = fms_launch * nl
                chk_fams.append({"kernels": fname, "ms_per_step": round(fms, 4), "bytes_per_step": int(fbytes),
                                 "achieved": round(fbytes / (fms * 1e-3) / 1e9, 1),
                                 "frac": round(fbytes / (fms * 1e-3) / 1e9 / hbm, 4)})

    # e2e: pinned host buffers, copies inside the timed region
    e2e_steps = max(3, min(args.steps, 10))
    if getattr(wl, "e2e_steps", None):  # sub-millisecond steps: more of them
        e2e_steps = max(e2e_steps, wl.e2e_steps)
    pipelined = getattr(wl, "e2e_pipeline", None)
    res = pipelined(selected, e2e_steps) if pipelined is not None else None
    e2e_mode = "sequential: H2D, pipeline, D2H per step"
    if res is not None:
        e2e_ms, h2d, d2h = res
        e2e_ms = max_over_ranks(e2e_ms, ws)
        e2e_mode = ("two buffer sets: step i's H2D overlaps step i-1's D2H (full-duplex PCIe); every step copies "
                    "its whole input in and its result out")
    else:
        bufs = wl.e2e_bufs(selected)
        for _ in range(2):
            wl.e2e_step(bufs)
        torch.cuda.synchronize()
        barrier(ws)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(e2e_steps):
            h2d, d2h = wl.e2e_step(bufs)
        t1.record()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(t0.elapsed_time(t1) / e2e_steps, ws)
    try:  # this box's PCIe ceiling for the same bytes (box-dependent: e2e is copy-bound)
        link = link_probe(h2d, d2h)
    except Exception as ex:  # e.g. host memory: report, do not fail the line
        link = None
        print(f"bench.py: link probe skipped ({ex})", file=sys.stderr)
    units_total = wl.units() * ws
    value = units_total / (ms * 1e-3) / 1e9
    achieved = (kbytes / (kms * 1e-3) / 1e9) if kms else None
    traffic = _ncu_traffic(wl.name, wl.units())
    line = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "Gelem/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": wl.scaling,
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic",
        "config": config_of(wl, ws),
        "parity": {"vs_cpu_port": bool(parity) if want is not None else "checked in tests",
                   "checked_variant": bool(parity_chk) if want is not None else "checked in tests"},
        "hbm_gbs_step": round(wl.algo_bytes_step() / (ms * 1e-3) / 1e9, 1),
        "checked": {
            "ms_per_step": round(ms_chk, 4),
            "value": round(units_total / (ms_chk * 1e-3) / 1e9, 3),
            "elided_speedup": round(ms_chk / ms, 3),
            # the program's algorithmic bytes over the CHECKED step (what the
            # reference's behaviour costs on this GPU), and per kernel family
            "roofline": {"step_frac": round(wl.algo_bytes_step() / (ms_chk * 1e-3) / 1e9 / hbm, 4),
                         "families": chk_fams},
        } if ms_chk else None,
        "roofline": {
            "bound": "hbm",
            "kernel": kname,
            "achieved": round(achieved, 1) if achieved else None,
            "peak": hbm,
            "peak_kind": peak_kind,
            "peak_note": ("MEASURED_PEAKS hbm_gbs is a copy (50 % read / 50 % write); a read-heavy kernel can "
                          "exceed it -- ncu's dram__throughput pct_of_peak is the device-limit reference"),
            "unit": "GB/s",
            "frac": round(achieved / hbm, 4) if achieved else None,
            "traffic": traffic,
            "algo_bytes_per_launch": kbytes,
            "kernel_ms": round(kms, 5) if kms else None,
            "step": {"algo_bytes": wl.algo_bytes_step(), "ms": round(ms, 4),
                     "achieved": round(wl.algo_bytes_step() / (ms * 1e-3) / 1e9, 1),
                     "frac": round(wl.algo_bytes_step() / (ms * 1e-3) / 1e9 / hbm, 4)},
            "other_kernels": others,
        },
        "e2e": {
            "value": round(units_total / (e2e_ms * 1e-3) / 1e9, 4),
            "unit": "Gelem/s",
            "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(e2e_ms, 3),
            "mode": e2e_mode,
            "link": link,
            "link_frac": round(link["duplex_ms"] / e2e_ms, 4) if link else None,
        },
        "cpu_baseline": cpu,
        "clocks": clocks,
        "gpu_launches": int(launches),
    }
    dr = getattr(wl, "dropin", None)
    if dr is not None and ws == 1 and not wl.big:
        try:
            line["dropin"] = dr()
        except Exception as e:  # informational
            line["dropin"] = {"unavailable": f"{type(e).__name__}: {e}"}
    l2c = getattr(wl, "l2_ceiling", None)
    if l2c is not None and kms:
        try:
            line["roofline"]["l2"] = l2c(kms)
        except Exception as e:  # the extra roof is informational
            line["roofline"]["l2"] = {"unavailable": f"{type(e).__name__}: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def config_of(wl, ws) -> dict:
    """The `config` object of BOTH arms (identical keys and values)."""
    return {
        "workload": wl.workload,
        "variant": "verifier-selected (ELIDED: Sc1 scatters fused, mkFlags Ss2)",
        "parallelism": f"shards{ws}" if ws > 1 else "single",
        "l2": ("steps rotate over 32 copies of the 8 MB working set (256 MB > the 126 MB L2): cold inputs, no flush"
               if wl.name == "c1" else "inputs larger than the 126 MB L2, no flush"),
    }


def _ncu_traffic(name, units=None):
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full capture (profiles/ncu_<name>_full.json; scaled by the units of
    this run when the capture was taken at another size), else null."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_{name}_full.json")) as f:
            d = json.load(f)
    except Exception:
        return None
    if units and d.get("dram_bytes_per_unit") and d.get("units") != units:
        return round(d["dram_bytes_per_unit"] * units)
    return d.get("dram_bytes_per_launch")


def cpu_baseline(wl, args):
    """The oracle port (OpenMP, all host threads) on the same workload."""
    from oracle import ixoracle as O

    threads = O.threads()
    inputs = wl.cpu_sample(20.0)
    n = inputs[-1]
    res = wl.cpu_run(*inputs[:-1], threads)
    times = []
    t_budget = time.time() + (3.0 if args.quick else 10.0)
    while True:
        t0 = time.perf_counter()
        wl.cpu_run(*inputs[:-1], threads)
        times.append(time.perf_counter() - t0)
        if time.time() > t_budget or len(times) >= 20:
            break
    best = statistics.median(times)
    out = {
        "value": round(n / best / 1e9, 4),
        "unit": "Gelem/s",
        "cores": threads,
        "kind": "port",
        "sample": (f"{len(times)} runs of the {wl.name} workload at n={n} by "
                   f"{getattr(wl, 'cpu_desc', 'oracle/ixoracle_par.c (OpenMP)')}, median"),
        "ms_per_run": round(best * 1e3, 2),
    }
    if n == wl.units() and wl.name in ("c1", "c2", "c5"):
        out["_result"] = (res[0], res[1])  # (ys, zs) / (num_true, ys): the parity reference of the device arm
    return out


def run_reference(args):
    """--impl reference: the reference's CPU path on the host cores.  The
    reference is Python and cannot travel to the GPU box, so this is its
    restatement oracle/ (C, OpenMP, every host thread) on the same config."""
    rank = int(os.environ.get("RANK", "0"))
    ws = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    from oracle import ixoracle as O

    wl = make_workload(args, 0, 1)
    wl_cfg = make_workload(args, 0, ws, describe_only=True)
    threads = O.threads()
    inputs = wl.cpu_sample(20.0)
    n = inputs[-1]
    for _ in range(args.warmup):
        wl.cpu_run(*inputs[:-1], threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        wl.cpu_run(*inputs[:-1], threads)
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    value = n / (ms * 1e-3) / 1e9
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 4),
        "unit": "Gelem/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": wl_cfg.scaling,
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic",
        "config": config_of(wl_cfg, ws),
        "cpu_baseline": {"value": round(value, 4), "unit": "Gelem/s", "cores": threads, "kind": "port",
                         "sample": f"one full pass over n={n} per step (the single-GPU workload): "
                                   f"{getattr(wl, 'cpu_desc', 'oracle/ixoracle_par.c (OpenMP)')}"},
        "e2e": {"value": round(value, 4), "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def make_workload(args, rank, ws, describe_only=False):
    """describe_only: the workload's name / description / scaling for `ws`
    ranks without touching a device or a process group (the reference arm)."""
    if args.config == "c2":
        wl = C2.__new__(C2) if describe_only else C2(args.quick, rank, ws)
    elif args.config in ("c1", "c5"):
        wl = C1.__new__(C1) if describe_only else C1(args.quick, rank, ws, big=args.config == "c5")
    elif args.config == "c3":
        wl = C3.__new__(C3) if describe_only else C3(args.quick, rank, ws, perm=args.perm)
    elif args.config == "c4":
        wl = C4.__new__(C4) if describe_only else C4(args.quick, rank, ws)
    else:
        raise SystemExit(f"unknown config {args.config}")
    if describe_only:
        wl.describe(args.quick, ws, **({"big": args.config == "c5"} if args.config in ("c1", "c5") else {}),
                    **({"perm": args.perm} if args.config == "c3" else {}))
    return wl


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def main():
    if os.environ.get("IXG_HANG_DUMP"):  # diagnostics: every thread's stack to stderr after N s
        import faulthandler

        faulthandler.dump_traceback_later(float(os.environ["IXG_HANG_DUMP"]), exit=True)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2", "c1", "c3", "c4", "c5"])
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--perm", default="streams", choices=["streams", "random"],
                    help="c3: the index array (two monotone streams, SURVEY §8d C3, or a random permutation)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        # one process per GPU: re-launch this command under torchrun (NCCL, 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
        os.execv(sys.executable, cmd + sys.argv[1:])
    if ws_env is not None and int(ws_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
    run_ours(args)


if __name__ == "__main__":
    main()
