"""Run one pipeline a few times (target for ncu captures; development tool).

python tools/prof_run.py <c2|filter|partition2|scan|csr|peer|map_jit|scan_jit> [log2n] [reps]
(CHECKED=1 in the environment: the all-CHECKED variants)
"""

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import _lib as L  # noqa: E402
from paper_2506_23058_b200 import gen, ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402


def main():
    what = sys.argv[1]
    n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 28)
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    variant = L.VARIANT_CHECKED if os.environ.get("CHECKED") else L.VARIANT_ELIDED
    dev = torch.device("cuda")
    st = ops.Status(dev)
    if what in ("c2", "filter"):
        xs = ops.gen_uniform(n, -128, 127, 0, torch.int32, device=dev)
        k = int((xs >= 0).sum().item())
        shape = torch.from_numpy(gen.segment_shape(1, max(1, n >> 8), k)).to(dev)
        ys = torch.empty(n, dtype=torch.int32, device=dev)
        zs = torch.empty(n, dtype=torch.int32, device=dev)
        dk = torch.empty(1, dtype=torch.int64, device=dev)
        for _ in range(reps):
            if what == "c2":
                ops.c2(xs, Pred.ge(0), shape, variant, st, ys=ys, zs=zs, d_k=dk)
            else:
                ops.filter(xs, Pred.ge(0), variant, st, ys=ys, d_count=dk)
    elif what == "partition2":
        xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 1, torch.int32, device=dev)
        ys = torch.empty(n, dtype=torch.int32, device=dev)
        dnt = torch.empty(1, dtype=torch.int64, device=dev)
        for _ in range(reps):
            ops.partition2(xs, Pred.lt(0), variant, st, ys=ys, d_nt=dnt)
    elif what == "scan":
        xs = ops.gen_uniform(n, -128, 127, 0, torch.int64, device=dev)
        out = torch.empty(n, dtype=torch.int64, device=dev)
        for _ in range(reps):
            ops.scan_add(xs, 0, out=out)
    elif what == "csr":
        ncols = 1 << 20
        x = ops.gen_uniform(ncols, -(1 << 15), (1 << 15) - 1, 3, torch.int32, device=dev)
        vals = ops.gen_uniform(n, -(1 << 15), (1 << 15) - 1, 4, torch.int32, device=dev)
        idx = ops.gen_uniform(n, 0, ncols - 1, 5, torch.int64, device=dev)
        out = torch.empty(n, dtype=torch.int32, device=dev)
        for _ in range(reps):
            ops.csr_gather(x, vals, idx, variant, st, out=out)
    elif what == "peer":  # the sharded partition2 kernel, two simulated ranks' shards in one process
        per = n // 2
        xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 1, torch.int32, device=dev)
        bufs = [torch.empty(per, dtype=torch.int32, device=dev) for _ in range(2)]
        ptrs = [b.data_ptr() for b in bufs]
        shards = [xs[r * per:(r + 1) * per] for r in range(2)]
        counts = torch.stack([ops.partition_counts(x, Pred.lt(0))[0] for x in shards])
        for _ in range(reps):
            for r in range(2):
                ops.partition2_peer(shards[r], Pred.lt(0), ptrs, per, counts, r)
    elif what in ("map_jit", "scan_jit"):  # NVRTC kernels of the generic executor
        from paper_2506_23058_b200 import ir, jit, jit_fold

        xs = ops.gen_uniform(n, -1000, 1000, 2, torch.int64, device=dev)
        ys = ops.gen_uniform(n, -1000, 1000, 3, torch.int64, device=dev)
        if what == "map_jit":  # map2 (\a b -> if a < b then a * 3 + b else b - a) xs ys
            lam = ir.Lambda(("a", "b"), ir.If(ir.BinOp("<", ir.VarE("a"), ir.VarE("b")),
                                              ir.BinOp("+", ir.BinOp("*", ir.VarE("a"), ir.Const(3)), ir.VarE("b")),
                                              ir.BinOp("-", ir.VarE("b"), ir.VarE("a"))))
            for _ in range(reps):
                jit.map_jit(lam, [xs, ys], {}, lambda node: 0, n, st, device=dev)
        else:  # scan (\a b -> if b < a then b else a) 0 xs  (a min-scan: tiled, associative)
            lam = ir.Lambda(("a", "b"), ir.If(ir.BinOp("<", ir.VarE("b"), ir.VarE("a")), ir.VarE("b"), ir.VarE("a")))
            for _ in range(reps):
                jit_fold.scan(lam, [0], [xs], {}, lambda node: 0, st, device=dev)
    torch.cuda.synchronize()
    assert st.read().ok
    print("ok", what, n, reps)


if __name__ == "__main__":
    main()
