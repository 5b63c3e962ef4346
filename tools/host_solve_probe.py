"""Host-buffer solve at 1024^3: pageable (numpy) vs pinned buffers through arena_poisson_solve_host."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, numpy as np, torch
import paper_1408_6497_b200 as arena
n = 1024
f = np.empty((n, n, n)); f[:] = 1.0
f[0, 0, 0] = 2.0
u = np.empty_like(f)
p = arena.get_plan(n)
p.solve_host(f, u)
for _ in range(2):
    t0 = time.perf_counter(); p.solve_host(f, u); t1 = time.perf_counter()
    print("pageable host solve", round((t1 - t0) * 1e3, 1), "ms")
hf = torch.empty((n, n, n), dtype=torch.float64, pin_memory=True); hf.copy_(torch.from_numpy(f))
hu = torch.empty_like(hf, pin_memory=True)
for _ in range(2):
    t0 = time.perf_counter(); p.solve_host(hf, hu); t1 = time.perf_counter()
    print("pinned host solve", round((t1 - t0) * 1e3, 1), "ms")
import os; print("cpus", len(os.sched_getaffinity(0)))
