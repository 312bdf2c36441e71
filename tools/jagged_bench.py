"""Time the jagged corpus programs (partition2L, filter_seg) through the
drop-in eval_program on device-resident inputs (development tool).

python tools/jagged_bench.py [log2n]
They run on the generic executor (one kernel per combinator) with the
verifier's selection: nothing of partition2L is proved in this reference
(mkSgmDescr is unanalyzable), filter_seg's compaction scatter is.
"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import eval_program, gen, ir  # noqa: E402

DATA = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2506_23058_b200", "data")


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    progs = json.load(open(os.path.join(DATA, "programs.json")))
    dev = torch.device("cuda")
    m = (1 << lg) // 64
    shp = gen.uniform(3, m, 0, 127, np.int64)
    n = int(shp.sum())
    cs = gen.uniform(4, n, 0, 1, np.int64).astype(bool)
    xs = gen.uniform(5, n, -1000, 1000, np.int64)
    args = [torch.from_numpy(shp).to(dev), torch.from_numpy(cs.astype(np.uint8)).to(dev), torch.from_numpy(xs).to(dev)]
    out = {"n": n, "m": m}
    for key, fun in (("own:partition2l.ixl", "partition2L"), ("own:filter_seg.ixl", "filter_seg")):
        prog = ir.from_json(progs[key]["program"])
        for variant in ("selected", "checked"):
            for _ in range(2):
                eval_program(prog, fun, args, as_tensors=True, variant=variant)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            reps = 5
            for _ in range(reps):
                eval_program(prog, fun, args, as_tensors=True, variant=variant)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / reps
            out[f"{fun}_{variant}"] = {"ms": ms, "Gelem/s": n / ms / 1e6}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
