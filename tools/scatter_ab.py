"""A/B timing of the scatter paths on the C3 inputs (development tool):
IXGPU_LIB=... python tools/scatter_ab.py [random|streams] [reps]
Prints per-kernel (TimedLaunch) and whole-call ms, ELIDED and CHECKED."""
import os, sys, json, torch
sys.path.insert(0, '.')
from paper_2506_23058_b200 import ops, _lib as L
kind = sys.argv[1] if len(sys.argv) > 1 else 'random'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n = 1 << 29
dev = torch.device('cuda')
g = torch.Generator(device=dev); g.manual_seed(11)
if kind == 'random':
    is_ = torch.randperm(n, generator=g, device=dev, dtype=torch.int64)
else:
    xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 11, torch.int32)
    c = xs < 0; t = torch.cumsum(c, 0, dtype=torch.int64); i1 = torch.arange(1, n + 1, device=dev, dtype=torch.int64)
    is_ = torch.where(c, t - 1, t[-1] + (i1 - t) - 1); del xs, c, t, i1
vs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 12, torch.int32)
out = torch.zeros(n, dtype=torch.int32, device=dev)
st = ops.Status(dev)
res = {"lib": os.environ.get("IXGPU_LIB", "default"), "kind": kind}
want = torch.zeros(n, dtype=torch.int32, device=dev); want[is_] = vs
for name, bits in (("elided", 0), ("checked", L.V_CONFLICT | L.V_INIT)):
    for _ in range(3):
        ops.scatter(out, is_, vs, bits, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        ops.scatter(out, is_, vs, bits, st)
    e1.record(); torch.cuda.synchronize()
    res[name + "_ms"] = round(e0.elapsed_time(e1) / reps, 4)
    res[name + "_ok"] = bool(torch.equal(out, want))
print(json.dumps(res))
