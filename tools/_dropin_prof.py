import json, os, sys, time, torch
sys.path.insert(0, os.getcwd())
from paper_2506_23058_b200 import eval_program, gen, ir, ops
from paper_2506_23058_b200.pred import Pred
DATA = "paper_2506_23058_b200/data"
n = 1 << 27
dev = torch.device("cuda")
progs = json.load(open(os.path.join(DATA, "programs.json")))
P = ir.from_json(progs["own:c2_filter_sgmsum.ixl"]["program"])
xs = ops.gen_uniform(n, -128, 127, 7, torch.int64, device=dev)
k = int((xs >= 0).sum().item())
shape = torch.from_numpy(gen.segment_shape(8, n >> 8, k)).to(dev)
args = [Pred.ge(0), xs, shape]
for _ in range(3):
    eval_program(P, "c2", args, as_tensors=True)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    t0 = time.perf_counter(); eval_program(P, "c2", args, as_tensors=True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print("wall ms per call", sorted(ts)[5] * 1e3)
if len(sys.argv) > 1:
    torch.cuda.cudart().cudaProfilerStart()
    eval_program(P, "c2", args, as_tensors=True); torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
