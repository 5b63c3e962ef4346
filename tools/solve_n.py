"""One solve at --n (any n, any path) for ncu captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_6497_b200 as arena  # noqa: E402
from paper_1408_6497_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=768)
ap.add_argument("--precision", type=int, default=64)
a = ap.parse_args()
f = torch.empty((a.n,) * 3, dtype=torch.float64, device="cuda")
problems.fill_device(problems.config(4, a.n), "f", f)
if a.precision == 32:
    f = f.float()
u = torch.empty_like(f)
arena.Plan(a.n, a.precision).solve_device(f, u)
torch.cuda.synchronize()
print("ok", a.n)
