"""Per-kernel timings of the sharded-C2 pieces on one GPU (development tool):
filter, sgmSum over k (exact and capacity grid), mkFlags, the fused C2, scan_add, CHECKED C2.

IXGPU_LIB=... python tools/segsum_bench.py [prof]"""
import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2506_23058_b200 import ops, gen, _lib as L
from paper_2506_23058_b200.pred import Pred
dev = torch.device('cuda')
N = 1 << 28
xs = ops.gen_uniform(N, -128, 127, 0, torch.int32, device=dev)
st = ops.Status(dev)
ys = torch.empty(N, dtype=torch.int32, device=dev); zs = torch.empty(N, dtype=torch.int32, device=dev)
dk = torch.empty(1, dtype=torch.int64, device=dev)
ops.filter(xs, Pred.ge(0), L.VARIANT_ELIDED, st, ys=ys, d_count=dk)
k = int(dk.item())
shape = torch.from_numpy(gen.segment_shape(1, 1 << 20, k)).to(dev)
bits = ops.flag_bitmap(shape, k)
tot = torch.empty(2, dtype=torch.int64, device=dev)
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
fb = torch.zeros(1, dtype=torch.int64, device=dev)
print("k", k)
print("filter 2^28", t(lambda: ops.filter(xs, Pred.ge(0), L.VARIANT_ELIDED, st, ys=ys, d_count=dk)))
print("segsum n=k", t(lambda: ops.segsum(ys, k, bits, 0, zs, 0, False, tot, st)))
print("segsum n=cap d_n", t(lambda: ops.segsum(ys, N, bits, 0, zs, 0, False, tot, st, d_n=dk, d_flag_base=fb)))
print("flag_bitmap m=2^20", t(lambda: ops.flag_bitmap(shape, k, bits=bits)))
print("fused c2", t(lambda: ops.c2(xs, Pred.ge(0), shape, 0, st, ys=ys, zs=zs, d_k=dk)))
if len(sys.argv) > 1:
    for _ in range(4): ops.segsum(ys, k, bits, 0, zs, 0, False, tot, st)
    torch.cuda.synchronize()
out64 = torch.empty(N, dtype=torch.int64, device=dev)
print("scan_add i32->i64 2^28", t(lambda: ops.scan_add(xs, out=out64, status=st)))
print("c2 CHECKED", t(lambda: ops.c2(xs, Pred.ge(0), shape, L.VARIANT_CHECKED, st, ys=ys, zs=zs, d_k=dk), reps=5))
