"""Run one pipeline a few times (target for ncu captures; development tool).

python tools/prof_run.py <c2|filter|partition2|scan|csr> [log2n] [reps]
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
    torch.cuda.synchronize()
    assert st.read().ok
    print("ok", what, n, reps)


if __name__ == "__main__":
    main()
