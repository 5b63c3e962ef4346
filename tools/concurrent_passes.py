"""Experiment (DESIGN 7.1): do a DRAM-latency-bound pass pair (K1 + K2) and the fp64-bound x pass (K3)
fill each other's idle resources when they share the GPU?  Two one-rank peer slabs (own workspaces)
run phase 0 (K1 + K2) and phase 1 (K3) — sequentially on all SMs, then concurrently on two streams
with each slab's persistent kernels limited to half the SMs (ARENA_FFT_SMS at plan creation)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1408_6497_b200 as arena  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = 10


def make(sms):
    if sms:
        os.environ["ARENA_FFT_SMS"] = str(sms)
    else:
        os.environ.pop("ARENA_FFT_SMS", None)
    s = arena.Slab(n, 1, loopback=True)  # one virtual rank: the slab's kernels on the single-GPU geometry
    s.set_exchange(arena.XCHG_PEER)      # no exchange copies (the passes store in place)
    return s


f = torch.rand((n, n, n), dtype=torch.float64, device="cuda") - 0.5
u = torch.empty_like(f)
f2, u2 = f.clone(), torch.empty_like(f)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


out = {"n": n}
A, B = make(0), make(0)
out["zy_all_sms_ms"] = timed(lambda: A.solve_phase(0, f, u))
out["x_all_sms_ms"] = timed(lambda: B.solve_phase(1, f2, u2))
out["sequential_ms"] = out["zy_all_sms_ms"] + out["x_all_sms_ms"]
for sx in (74, 60, 88):
    A2, B2 = make(148 - sx), make(sx)

    def both():
        e = torch.cuda.Event()
        e.record()
        s1.wait_event(e)
        s2.wait_event(e)
        A2.solve_phase(0, f, u, stream=s1.cuda_stream)
        B2.solve_phase(1, f2, u2, stream=s2.cuda_stream)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    out[f"concurrent_x{sx}_zy{148 - sx}_ms"] = timed(both)
    out[f"zy_alone_{148 - sx}_sms_ms"] = timed(lambda: A2.solve_phase(0, f, u))
    out[f"x_alone_{sx}_sms_ms"] = timed(lambda: B2.solve_phase(1, f2, u2))
    del A2, B2
print(json.dumps(out))
