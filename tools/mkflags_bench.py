"""C2 step pieces at full size: bitmap clear, mkFlags (clear + scan), and
the whole ELIDED C2 call, CUDA-event timed over back-to-back repetitions
(development tool).

python tools/mkflags_bench.py [reps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import gen, ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402


def timed(fn, reps):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    n, m = 1 << 28, 1 << 20
    xs_h = gen.uniform(0, n, -128, 127, np.int32)
    k = int(np.count_nonzero(xs_h >= 0))
    shape = torch.from_numpy(gen.segment_shape(1, m, k)).cuda()
    xs = torch.from_numpy(xs_h).cuda()
    bits = torch.empty(int(ops._lib().ixg_bitmap_words(n)), dtype=torch.int32, device="cuda")
    ys = torch.empty(n, dtype=torch.int32, device="cuda")
    zs = torch.empty(n, dtype=torch.int32, device="cuda")
    dk = torch.empty(1, dtype=torch.int64, device="cuda")
    scn = torch.empty(m, dtype=torch.int64, device="cuda")
    st = ops.Status(xs.device)
    r = {
        "bitmap clear (torch zero_)": timed(lambda: bits.zero_(), reps),
        "mkFlags (clear + scan)": timed(lambda: ops.flag_bitmap(shape, n, bits=bits), reps),
        "mkFlags scan, no bits (nbits 0)": timed(lambda: ops.flag_bitmap(shape, 0, bits=bits), reps),
        "scan_add over the shape": timed(lambda: ops.scan_add(shape, out=scn), reps),
        "c2 ELIDED step": timed(lambda: ops.c2(xs, Pred.ge(0), shape, 0, st, ys=ys, zs=zs, d_k=dk), reps),
    }
    for key, v in r.items():
        print(f"{key:32s} {v:9.2f} us")


if __name__ == "__main__":
    main()
