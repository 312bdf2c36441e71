"""C3 scatter inputs for ncu captures (development tool): python tools/c3prof.py KIND...

KIND: streams | random (the C3 / C3-secondary index patterns at 2^29), with the
suffix _chk for the CHECKED scatter; two scatters each."""
import sys, torch
sys.path.insert(0, '.')
from paper_2506_23058_b200 import ops, _lib as L
n = 1 << 29
dev = torch.device('cuda')
g = torch.Generator(device=dev); g.manual_seed(11)
for kind in sys.argv[1:]:
    if kind.startswith('random'):
        is_ = torch.randperm(n, generator=g, device=dev, dtype=torch.int64)
    else:
        xs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 11, torch.int32)
        c = xs < 0; t = torch.cumsum(c, 0, dtype=torch.int64); i1 = torch.arange(1, n + 1, device=dev, dtype=torch.int64)
        is_ = torch.where(c, t - 1, t[-1] + (i1 - t) - 1); del xs, c, t, i1
    vs = ops.gen_uniform(n, -(1 << 31), (1 << 31) - 1, 12, torch.int32)
    out = torch.zeros(n, dtype=torch.int32, device=dev)
    st = ops.Status(dev)
    bits = L.V_CONFLICT | L.V_INIT if kind.endswith('chk') else 0
    for _ in range(2):
        ops.scatter(out, is_, vs, bits, st)
    torch.cuda.synchronize()
    del is_, vs, out
