"""partition2 at the paper's sizes (50 M / 100 M / 200 M 4-byte elements,
PAPER.md:3298-3300, A100 Futhark): verifier-selected (ELIDED + Sc1) vs
all-CHECKED on one B200 (development tool).

python tools/paper_sizes.py
"""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import _lib as L  # noqa: E402
from paper_2506_23058_b200 import ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402

PAPER = {50: (12.0, 4.4, 4.7), 100: (38.0, 7.0, 7.5), 200: (135.0, 12.2, 12.8)}  # checked ms, static x, +Opt x


def timeit(fn, reps=10, warm=3):
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
    dev = torch.device("cuda")
    out = {}
    for m in (50, 100, 200):
        n = m * 1000 * 1000
        xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 5, torch.int32, device=dev)
        ys = torch.empty(n, dtype=torch.int32, device=dev)
        d = torch.empty(1, dtype=torch.int64, device=dev)
        st = ops.Status(dev)
        el = timeit(lambda: ops.partition2(xs, Pred.lt(0), L.VARIANT_ELIDED, st, ys=ys, d_nt=d))
        ch = timeit(lambda: ops.partition2(xs, Pred.lt(0), L.VARIANT_CHECKED, st, ys=ys, d_nt=d))
        pc, ps, po = PAPER[m]
        out[f"{m}M"] = {"elided_ms": round(el, 4), "checked_ms": round(ch, 4), "speedup": round(ch / el, 2),
                        "elided_Gelem_s": round(n / el / 1e6, 1),
                        "paper_A100": {"checked_ms": pc, "static_x": ps, "opt_x": po,
                                       "opt_Gelem_s": round(n / (pc / po) / 1e6, 1)}}
        del xs, ys
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
