"""The drop-in eval_program on device-resident int64 inputs (the element
type Python ints arrive as), verifier-selected vs all-CHECKED, for the
corpus programs of the benchmark configs (development tool).

python tools/dropin_bench.py [log2 n]
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import eval_program, gen, ir, ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402

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
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 27
    n = 1 << lg
    dev = torch.device("cuda")
    progs = json.load(open(os.path.join(DATA, "programs.json")))
    P = {k: ir.from_json(v["program"]) for k, v in progs.items()}
    xs = ops.gen_uniform(n, -128, 127, 7, torch.int64, device=dev)
    k = int((xs >= 0).sum().item())
    shape = torch.from_numpy(gen.segment_shape(8, n >> 8, k)).to(dev)
    cases = {
        "c2": (P["own:c2_filter_sgmsum.ixl"], "c2", [Pred.ge(0), xs, shape]),
        "partition2": (P["ref:partition2.ixl"], "partition2", [Pred.lt(0), xs]),
        "filter": (P["ref:filter.ixl"], "filter", [Pred.ge(0), xs]),
    }
    out = {"n": n, "dtype": "int64"}
    for name, (prog, fun, args) in cases.items():
        for variant in ("selected", "checked"):
            ms = timeit(lambda: eval_program(prog, fun, args, as_tensors=True, variant=variant))
            out[f"{name}_{variant}"] = {"ms": round(ms, 4), "Gelem/s": round(n / ms / 1e6, 2)}
        out[f"{name}_speedup"] = round(out[f"{name}_checked"]["ms"] / out[f"{name}_selected"]["ms"], 2)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
