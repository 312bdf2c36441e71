"""Per-CTA timeline of the big-tile compaction kernel (development tool).

Needs a library built with -DIXG_TRACE (IXGPU_LIB=...):
    IXG_TILE=12288 python tools/trace_filter.py <filter|c2> [log2n] [i32|i64]   (i64: IXG_TILE=8192)
Prints per-phase durations (ns) over CTAs and the number of CTAs in flight.
k_filter_b trace slots: 0 start, 1 counted, 2 CTA scan, 3 compacted, 4 base
known (bar 2), 5 look-back warp done, 6 stores done (filter), 7 look-back
rounds/spins; C2: 6 ys stored, 8 seg pass 1 + scan, 9 pass 2 done, 10 carry
known (bar 3), 11 zs stored, 12 look-back warp carry done, 13 seg look-back
rounds/spins.
"""

import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import _lib as L  # noqa: E402
from paper_2506_23058_b200 import gen, ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402

SLOTS = 20


def phase(a, nm, i, j):
    d = a[:, j] - a[:, i]
    print(f"  {nm:11s} median {np.median(d):8.0f} ns  p90 {np.percentile(d, 90):8.0f}  mean {d.mean():8.0f}")


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "filter"
    n = 1 << (int(sys.argv[2]) if len(sys.argv) > 2 else 28)
    dev = torch.device("cuda")
    st = ops.Status(dev)
    dt = torch.int64 if (len(sys.argv) > 3 and sys.argv[3] == "i64") else torch.int32
    xs = ops.gen_uniform(n, -128, 127, 0, dt, device=dev)
    ys = torch.empty(n, dtype=dt, device=dev)
    zs = torch.empty(n, dtype=dt, device=dev)
    dk = torch.empty(1, dtype=torch.int64, device=dev)
    k = int((xs >= 0).sum().item())
    shape = torch.from_numpy(gen.segment_shape(1, max(1, n >> 8), k)).to(dev)
    for _ in range(3):
        if what == "c2":
            ops.c2(xs, Pred.ge(0), shape, 0, st, ys=ys, zs=zs, d_k=dk)
        elif what == "part2":
            ops.partition2(xs, Pred.lt(0), 0, st, ys=ys, d_nt=dk)
        else:
            ops.filter(xs, Pred.ge(0), 0, st, ys=ys, d_count=dk)
    torch.cuda.synchronize()
    lib = L.load()
    cnt = (1 << 17) * SLOTS
    buf = (ctypes.c_ulonglong * cnt)()
    L.check(lib.ixg_trace_read(buf, cnt), "trace")
    a = np.frombuffer(buf, dtype=np.uint64).reshape(-1, SLOTS).astype(np.int64)
    tile = int(os.environ.get("IXG_TILE", "12288"))
    tiles = min((n + tile - 1) // tile, a.shape[0])
    a = a[:tiles]
    t0 = a[:, 0].min()
    for c in (0, 1, 2, 3, 4, 5, 6, 8, 9, 10, 11, 12):
        a[:, c] -= t0
    end = 11 if what == "c2" else 6
    print(f"tiles {tiles}, kernel span {a[:, end].max() / 1e3:.1f} us")
    phase(a, "load+count", 0, 1)
    phase(a, "cta_scan", 1, 2)
    phase(a, "compact", 2, 3)
    phase(a, "wait_base", 3, 4)
    phase(a, "lookback", 0, 5)
    if what == "c2":
        phase(a, "ys_store", 4, 6)
        if a[:, 14].any():
            a[:, 14] -= t0
            a[:, 15] -= t0
            phase(a, " shift", 4, 14)
            a[:, 16] -= t0
            a[:, 17] -= t0
            phase(a, "  pre-shift", 4, 16)
            phase(a, "  to last round bar", 16, 17)
            phase(a, " fence+bar", 14, 15)
            phase(a, " bulk issue", 15, 6)
        phase(a, "seg_p1+scan", 6, 8)
        phase(a, "seg_pass2", 8, 9)
        phase(a, "wait_carry", 9, 10)
        phase(a, "zs_store", 10, 11)
        phase(a, "lb_carry", 4, 12)
        r2 = a[:, 13] >> 32
        print(f"  seg look-back rounds mean {r2.mean():.2f}, spins mean {(a[:, 13] & 0xFFFFFFFF).mean():.1f}")
    else:
        phase(a, "store", 4, 6)
    cum = {c: int(np.median(a[:, c] - a[:, 0])) for c in range(1, 18) if a[:, c].any() and c not in (7, 13)}
    if a[:, 18].any():
        lb, last, first = a[:, 5] - a[:, 0], a[:, 18] - t0 - a[:, 0], a[:, 19] - t0 - a[:, 0]
        print(f"  bar 2: first worker warp arrives {np.median(first):.0f}, last {np.median(last):.0f}, "
              f"look-back warp {np.median(lb):.0f} (median); look-back warp last in "
              f"{100 * np.mean(lb > last):.0f} % of tiles, by median {np.median(np.maximum(lb - last, 0)):.0f}")
    print("  cumulative medians from start (slot: ns):", cum)
    for r in [x for x in (100, 5000, 15000) if x < tiles]:
        print(f"  tile {r}:", {c: int(a[r, c] - a[r, 0]) for c in (1, 2, 3, 4, 5, 6, 14, 15, 16, 17)})
    print("  frac slot5 > slot4:", float(np.mean(a[:, 5] > a[:, 4])))
    life = a[:, end] - a[:, 0]
    print(f"  life        median {np.median(life):8.0f} ns  p90 {np.percentile(life, 90):8.0f}")
    mid = a[:, end].max() / 2
    print("  in flight at mid:", int(((a[:, 0] <= mid) & (a[:, end] >= mid)).sum()))
    starts = np.sort(a[:, 0])
    print(f"  start interval (median over tiles) {np.median(np.diff(starts)):.1f} ns")
    rounds, spins = a[:, 7] >> 32, a[:, 7] & 0xFFFFFFFF
    print(f"  look-back rounds mean {rounds.mean():.2f} max {rounds.max()}, "
          f"first-slot spins mean {spins.mean():.1f} p90 {np.percentile(spins, 90):.0f}")


if __name__ == "__main__":
    main()
