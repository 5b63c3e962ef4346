"""Per-phase times of the pencil decomposition on ONE GPU (loopback: the Pr x Pc virtual
ranks' kernels run one after another, exchanges are device copies), plain vs folded
distribution, config-5 / config-4 sources solved in place, checked against the analytic u.

    python tools/pencil_fold_timing.py [--n 2048] [--precision 32] [--grid 2x4]

Phase times / (Pr Pc) are the per-rank pass times (plus the copies, equal in volume for
both layouts); phases: 0 K1 (+ row exchange), 1 K2 (+ column), 2 K3 (+ column back),
3 K4 (+ row back), 4 K5."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_6497_b200 as arena  # noqa: E402
from paper_1408_6497_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=2048)
ap.add_argument("--precision", type=int, default=32)
ap.add_argument("--grid", default="2x4")
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
pr, pc = (int(x) for x in a.grid.split("x"))
n = a.n
dt = torch.float64 if a.precision == 64 else torch.float32
src = problems.config(a.config, n)
for folded in (False, True):
    f = torch.empty((n, n, n), dtype=dt, device="cuda")
    blk = 64
    for i0 in range(0, n, blk):  # f in fp64 blocks, rounded to the run's precision
        tmp = torch.empty((blk, n, n), dtype=torch.float64, device="cuda")
        problems.fill_device(src, "f", tmp, 64, 0, i0, blk)
        f[i0:i0 + blk].copy_(tmp)
        del tmp
    torch.cuda.synchronize()
    s = arena.Pencil(n, pr, pc, loopback=True, precision=a.precision, folded=folded)
    st = torch.cuda.current_stream().cuda_stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    tot = [0.0] * 5
    for rep in range(a.reps + 1):
        if rep > 0:  # timed solves re-solve the (overwritten) field: timing only
            pass
        ev[0].record()
        for p in range(5):
            s.solve_phase(p, f, f, st)
            ev[p + 1].record()
        torch.cuda.synchronize()
        if rep == 0:
            # parity of the first solve vs the analytic u (gauge-aligned rel L2, fp64 blocks)
            num = den = su = sa = 0.0
            for i0 in range(0, n, blk):
                ua = torch.empty((blk, n, n), dtype=torch.float64, device="cuda")
                problems.fill_device(src, "u", ua, 64, 0, i0, blk)
                su += f[i0:i0 + blk].double().sum().item()
                sa += ua.sum().item()
                del ua
            shift, mean_a = (sa - su) / n ** 3, sa / n ** 3
            for i0 in range(0, n, blk):
                ua = torch.empty((blk, n, n), dtype=torch.float64, device="cuda")
                problems.fill_device(src, "u", ua, 64, 0, i0, blk)
                d = f[i0:i0 + blk].double() + shift - ua
                num += (d * d).sum().item()
                den += ((ua - mean_a) ** 2).sum().item()
                del ua, d
            rel = (num / den) ** 0.5
            continue
        for p in range(5):
            tot[p] += ev[p].elapsed_time(ev[p + 1])
    ms = [t / a.reps for t in tot]
    print(json.dumps({"n": n, "precision": a.precision, "grid": a.grid, "folded": folded,
                      "phase_ms_all_ranks": ms, "phase_ms_per_rank": [m / (pr * pc) for m in ms],
                      "solve_ms_all_ranks": sum(ms), "rel_l2_vs_analytic_first_solve": rel}), flush=True)
    s.close()
    del f
    torch.cuda.empty_cache()
