"""Quick per-pipeline device timings (development tool, not the bench contract).

python tools/kbench.py [log2n]
Times the ELIDED and CHECKED variants of each pipeline on device-resident
inputs with CUDA events and reports Gelem/s and algorithmic GB/s.
"""

import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_23058_b200 import _lib as L  # noqa: E402
from paper_2506_23058_b200 import gen, ops  # noqa: E402
from paper_2506_23058_b200.pred import Pred  # noqa: E402


def timeit(fn, reps=20, warm=3):
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


def ktime(kid, fn, reps=10):
    lib = L.load()
    fn()
    torch.cuda.synchronize()
    lib.ixg_timer_start(kid)
    for _ in range(reps):
        fn()
    tot, cnt = ctypes.c_double(0), ctypes.c_int64(0)
    lib.ixg_timer_stop(ctypes.byref(tot), ctypes.byref(cnt))
    return tot.value / max(cnt.value, 1)


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 28
    n = 1 << lg
    dev = torch.device("cuda")
    out = {}
    src = torch.empty(n, dtype=torch.int32, device=dev)
    dst = torch.empty_like(src)
    ms = timeit(lambda: dst.copy_(src))
    out["copy_i32"] = {"ms": ms, "GBps": 8 * n / ms / 1e6}

    xs = ops.gen_uniform(n, -128, 127, 0, torch.int32, device=dev)
    k = int((xs >= 0).sum().item())
    m = max(1, n >> 8)
    shape = torch.from_numpy(gen.segment_shape(1, m, k)).to(dev)
    st = ops.Status(dev)
    ys = torch.empty(n, dtype=torch.int32, device=dev)
    zs = torch.empty(n, dtype=torch.int32, device=dev)
    dk = torch.empty(1, dtype=torch.int64, device=dev)
    p = Pred.ge(0)
    for name, var in (("elided", L.VARIANT_ELIDED), ("checked", L.VARIANT_CHECKED)):
        f = lambda var=var: ops.c2(xs, p, shape, var, st, ys=ys, zs=zs, d_k=dk)  # noqa: E731
        ms = timeit(f, reps=10)
        out[f"c2_{name}"] = {"ms": ms, "Gelem/s": n / ms / 1e6, "algoGBps": (4 * n + 8 * m + 8 * k) / ms / 1e6}
    kms = ktime(L.K_FILTER_FUSED, lambda: ops.c2(xs, p, shape, 0, st, ys=ys, zs=zs, d_k=dk))
    out["c2_fused_kernel"] = {"ms": kms, "algoGBps": (4 * n + 8 * k) / kms / 1e6}
    f = lambda: ops.filter(xs, p, 0, st, ys=ys, d_count=dk)  # noqa: E731
    kms = ktime(L.K_FILTER_FUSED, f)
    out["filter_kernel"] = {"ms": kms, "algoGBps": (4 * n + 4 * k) / kms / 1e6}
    # the sharded / split C2's sgmSum pass over the filtered ys (k elements)
    bits = ops.flag_bitmap(shape, k)
    tot = torch.empty(2, dtype=torch.int64, device=dev)
    kms = ktime(L.K_SEGSUM, lambda: ops.segsum(ys, k, bits, 0, zs, 0, False, tot, st))
    out["segsum_kernel"] = {"ms": kms, "algoGBps": 8 * k / kms / 1e6}

    xs2 = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 1, torch.int32, device=dev)
    dnt = torch.empty(1, dtype=torch.int64, device=dev)
    for name, var in (("elided", L.VARIANT_ELIDED), ("checked", L.VARIANT_CHECKED)):
        f = lambda var=var: ops.partition2(xs2, Pred.lt(0), var, st, ys=ys, d_nt=dnt)  # noqa: E731
        ms = timeit(f, reps=10)
        out[f"partition2_{name}"] = {"ms": ms, "Gelem/s": n / ms / 1e6, "algoGBps": 8 * n / ms / 1e6}
    f = lambda: ops.partition2(xs2, Pred.lt(0), 0, st, ys=ys, d_nt=dnt)  # noqa: E731
    out["place_kernel"] = {"ms": ktime(L.K_PLACE, f)}
    out["count_kernel"] = {"ms": ktime(L.K_CLASS_COUNT, f)}
    out["place_kernel"]["algoGBps"] = 8 * n / out["place_kernel"]["ms"] / 1e6
    out["count_kernel"]["GBps"] = 4 * n / max(out["count_kernel"]["ms"], 1e-9) / 1e6
    dm = torch.empty(2, dtype=torch.int64, device=dev)
    for name, var in (("elided", L.VARIANT_ELIDED), ("checked", L.VARIANT_CHECKED)):
        f = lambda var=var: ops.partition3(xs2, Pred.lt(-(1 << 30)), Pred.hash(7), var, st, ys=ys, d_m=dm)  # noqa: E731
        ms = timeit(f, reps=10)
        out[f"partition3_{name}"] = {"ms": ms, "Gelem/s": n / ms / 1e6, "algoGBps": 8 * n / ms / 1e6}

    # the drop-in path's element type: int64 (the language's i64), 2^27 elements = 1 GiB
    n64 = n // 2
    x64s = ops.gen_uniform(n64, -128, 127, 0, torch.int64, device=dev)
    y64 = torch.empty(n64, dtype=torch.int64, device=dev)
    kms = ktime(L.K_FILTER_FUSED, lambda: ops.filter(x64s, p, 0, st, ys=y64, d_count=dk))
    k64 = int(dk.item())
    out["filter_i64_kernel"] = {"ms": kms, "algoGBps": (8 * n64 + 8 * k64) / kms / 1e6}
    kms = ktime(L.K_PLACE, lambda: ops.partition2(x64s, Pred.lt(0), 0, st, ys=y64, d_nt=dnt))
    out["partition2_i64_kernel"] = {"ms": kms, "algoGBps": 16 * n64 / kms / 1e6}
    del x64s, y64

    # library reference points (CUB via torch): stream compaction and scan
    mask = xs >= 0
    out["torch_masked_select"] = {"ms": timeit(lambda: torch.masked_select(xs, mask), reps=5)}
    out["torch_cumsum_i32"] = {"ms": timeit(lambda: torch.cumsum(xs, 0, dtype=torch.int64), reps=5)}
    so32 = torch.empty(n, dtype=torch.int64, device=dev)
    ms = timeit(lambda: ops.scan_add(xs, 0, out=so32))
    out["scan_i32"] = {"ms": ms, "GBps": 12 * n / ms / 1e6}
    del so32
    x64 = xs.to(torch.int64)
    so = torch.empty(n, dtype=torch.int64, device=dev)
    ms = timeit(lambda: ops.scan_add(x64, 0, out=so))
    out["scan_i64"] = {"ms": ms, "GBps": 16 * n / ms / 1e6}
    ok = st.read().ok
    out["status_ok"] = ok
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
