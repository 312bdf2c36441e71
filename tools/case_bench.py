"""Time the paper's other case studies on device
inputs, verifier-selected vs all-CHECKED (development tool):

* maxMatching's get_smallest_pairs (hist-min + H[es[i]] == is[i] + 2x
  filter_by; the H[i] bounds site and both filter_by scatters proved):
  through the drop-in eval_program on device tensors;
* kmeans_ker (CSR row loop, f64, five bounds sites proved): ixg_kmeans_ker
  over every row.

python tools/case_bench.py [log2 edges]
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import _lib as L  # noqa: E402
from paper_2506_23058_b200 import eval_program, ir, ops  # noqa: E402

DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_23058_b200", "data")


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    dev = torch.device("cuda")
    progs = json.load(open(os.path.join(DATA, "programs.json")))
    out = {}
    # maxMatching
    prog = ir.from_json(progs["ref:maxmatching.ixl"]["program"])
    n, nv = 1 << lg, 1 << 20
    es = ops.gen_uniform(n, 0, nv - 1, 21, torch.int64, device=dev)
    is_ = (torch.arange(n, device=dev, dtype=torch.int64) * 0x9E3779B97F4A7C15) & ((1 << 40) - 1)  # injective
    for variant in ("selected", "checked"):
        ms = timeit(lambda v=variant: eval_program(prog, "get_smallest_pairs", [nv, 1 << 62, es, is_],
                                                   as_tensors=True, variant=v))
        out[f"get_smallest_pairs_{variant}"] = {"ms": ms, "Gelem/s": n / ms / 1e6}
    out["get_smallest_pairs_speedup"] = out["get_smallest_pairs_checked"]["ms"] / out["get_smallest_pairs_selected"]["ms"]
    # kmeans_ker over all rows
    rows_n, ncols = 1 << 20, 1 << 12
    lens = ops.gen_uniform(rows_n, 0, 127, 22, torch.int64, device=dev)
    ptr = torch.zeros(rows_n + 1, dtype=torch.int64, device=dev)
    ptr[1:] = torch.cumsum(lens, 0)
    nnz = int(ptr[-1].item())
    vals = torch.rand(nnz, dtype=torch.float64, device=dev)
    idx = ops.gen_uniform(nnz, 0, ncols - 1, 23, torch.int64, device=dev)
    cl = torch.rand(ncols, dtype=torch.float64, device=dev)
    rows = torch.arange(rows_n, dtype=torch.int64, device=dev)
    st = ops.Status(dev)
    for name, variant in (("selected", L.VARIANT_ELIDED), ("checked", L.VARIANT_CHECKED)):
        ms = timeit(lambda v=variant: ops.kmeans_ker(rows, ptr, cl, vals, idx, v, st))
        out[f"kmeans_ker_{name}"] = {"ms": ms, "Gnnz/s": nnz / ms / 1e6, "nnz": nnz}
    out["kmeans_ker_speedup"] = out["kmeans_ker_checked"]["ms"] / out["kmeans_ker_selected"]["ms"]
    out["status_ok"] = st.read().ok
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
