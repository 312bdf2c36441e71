import sys, time, torch
sys.path.insert(0, '.')
from paper_2506_23058_b200 import ops, _lib as L
from paper_2506_23058_b200.pred import Pred
xs = torch.randint(-2**31, 2**31-1, (1<<20,), dtype=torch.int32, device='cuda')
ys = torch.empty_like(xs); d = torch.empty(1, dtype=torch.int64, device='cuda'); st = ops.Status(torch.device('cuda'))
p = Pred.lt(0)
for _ in range(10): ops.partition2(xs, p, 0, st, ys=ys, d_nt=d)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(1000): ops.partition2(xs, p, 0, st, ys=ys, d_nt=d)
t1 = time.perf_counter()
torch.cuda.synchronize()
print("host us per call", (t1 - t) * 1e3, "gpu us per call", (time.perf_counter() - t) * 1e3)
