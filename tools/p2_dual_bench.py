"""Single-GPU partition2 two ways at full size (development A/B): the
one-pass two-segment kernel (xs read per class, 12 B/elem) against a count
pass + the one-read dual placement of ixg_partition2_peer with one rank
(4 + 8 B/elem).  CUDA-event timed, back-to-back calls.

python tools/p2_dual_bench.py [log2n ...]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402


def timed(fn, reps):
    for _ in range(2):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    p = Pred.lt(0)
    for lg in [int(a) for a in sys.argv[1:]] or [28, 31]:
        n = 1 << lg
        xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 0, torch.int32)
        ys = torch.empty(n, dtype=torch.int32, device="cuda")
        ys2 = torch.empty(n, dtype=torch.int32, device="cuda")
        st = ops.Status(xs.device)
        dnt = torch.empty(1, dtype=torch.int64, device="cuda")
        reps = 20 if lg <= 28 else 5
        t_seg = timed(lambda: ops.partition2(xs, p, 0, st, ys=ys, d_nt=dnt), reps)

        def dual():
            ops.partition_counts(xs, p, d_tot=dnt)
            ops.partition2_peer(xs, p, [ys2.data_ptr()], n, dnt, 0)

        t_dual = timed(dual, reps)
        t_cnt = timed(lambda: ops.partition_counts(xs, p, d_tot=dnt), reps)
        same = bool(torch.equal(ys, ys2))
        gb = 8 * n / 1e9
        print(f"2^{lg}: two-segment {t_seg:.3f} ms ({gb / t_seg:.0f} GB/s algorithmic) | count + dual {t_dual:.3f} ms "
              f"({gb / t_dual:.0f} GB/s; count alone {t_cnt:.3f} ms) | identical {same}")
        del xs, ys, ys2
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
