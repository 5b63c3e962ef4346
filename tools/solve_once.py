"""Minimal driver for ncu captures: build the config-4 source at --n, run --reps solves."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_6497_b200 as arena  # noqa: E402
from paper_1408_6497_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--precision", type=int, default=64)
a = ap.parse_args()
src = problems.config(4, a.n)
f = torch.empty((a.n,) * 3, dtype=torch.float64, device="cuda")
problems.fill_device(src, "f", f)
if a.precision == 32:
    f = f.float()
u = torch.empty_like(f)
p = arena.Plan(a.n, a.precision)
for _ in range(a.reps):
    p.solve_device(f, u)
torch.cuda.synchronize()
print("ok", a.n, a.reps)
