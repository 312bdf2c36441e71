import cProfile, pstats, json, os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_2506_23058_b200 import eval_program, ir, ops
from paper_2506_23058_b200.pred import Pred
progs = json.load(open("paper_2506_23058_b200/data/programs.json"))
prog = ir.from_json(progs["ref:filter.ixl"]["program"])
xs = ops.gen_uniform(1 << 20, -128, 127, 7, torch.int64, device=torch.device("cuda"))
for _ in range(5): eval_program(prog, "filter", [Pred.ge(0), xs], as_tensors=True)
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
for _ in range(100): eval_program(prog, "filter", [Pred.ge(0), xs], as_tensors=True)
torch.cuda.synchronize()
print("us per call", (time.perf_counter() - t0) * 1e4)
cProfile.run('for _ in range(100): eval_program(prog, "filter", [Pred.ge(0), xs], as_tensors=True)', '/tmp/p.out')
pstats.Stats('/tmp/p.out').sort_stats('cumulative').print_stats(25)
