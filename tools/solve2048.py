import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1408_6497_b200 as arena
from paper_1408_6497_b200 import problems
n = 2048
src = problems.config(5, n)
f = torch.empty((n,)*3, dtype=torch.float64, device="cuda")
problems.fill_device(src, "f", f)
p = arena.Plan(n, 64)
p.solve_device(f, f)
torch.cuda.synchronize()
print("ok")
