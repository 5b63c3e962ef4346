#!/usr/bin/env python3
"""Benchmark of the spectral Poisson solve (BASELINE.json metric: Poisson
unknowns solved/sec, fp64 FFT solve, % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 1024] [--impl ours|reference]

One step = one full solve (r2c 3D FFT, Poisson scale, c2r 3D FFT) of the
BASELINE config-4 source (1024^3 fp64, 64 random Fourier modes, seed 4),
inputs resident in HBM.  The field (8.6 GB) is far larger than L2 (126 MB),
so no L2 flush is needed between steps.  Prints ONE JSON line on rank 0.

--impl reference times the reference's own CPU solver (fft_solver.cpp:51-87
over the FFTW3-API shim, oracle/_ref; the C restatement oracle/lib when that
was not built) on the host cores, on a bounded 512^3 sample of the same source.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "Poisson unknowns solved/sec (fp64 FFT solve)"
UNIT = "unknowns/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--precision", type=int, default=64, choices=(64, 32))
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--inplace", action="store_true",
                    help="solve in place (u aliases f): f + workspace only, so 2048^3 fp64 fits one GPU "
                         "(default for n >= 2048); parity then from one solve of a fresh f, checked in plane blocks")
    ap.add_argument("--cpu-n", type=int, default=512, help="grid of the bounded CPU sample")
    ap.add_argument("--slab", action="store_true", help="use the slab (NCCL) path even with one rank")
    ap.add_argument("--decomp", default="slab", choices=("slab", "pencil"), help="multi-GPU decomposition")
    ap.add_argument("--pgrid", default=None, help="pencil process grid RxC (default: near-square, R <= C)")
    ap.add_argument("--xchg", default="peer", choices=("peer", "nccl"),
                    help="exchange: peer = fused into the passes as NVLink stores (CUDA IPC), nccl = send/recv")
    return ap.parse_args()


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(n: int, elem: int):
    """Per-kernel algorithmic HBM bytes: R = real field, C = half spectrum."""
    R = n ** 3 * elem
    C = n * n * (n // 2 + 1) * 2 * elem
    per = {"zfwd_r2c": R + C, "yfwd": 2 * C, "xmid_fwd_scale_inv": 2 * C, "yinv": 2 * C, "zinv_c2r": C + R,
           # L2-fused pairs: HBM sees f read + spectrum write (and the reverse) once
           "zy_fused_fwd": R + C, "yz_fused_inv": C + R,
           # generic (any n) path: five sweeps (x forward * symbol * x backward fused)
           "gen_z_r2c": R + C, "gen_y_fwd": 2 * C, "gen_xmid_fwd_scale_inv": 2 * C,
           "gen_y_inv": 2 * C, "gen_z_c2r": C + R,
           # radix-3 split path (n = 3M): two extra spectrum sweeps (split, merge)
           "split3_fwd": 2 * C, "split3_inv": 2 * C, "zsplit_r2c": R + C, "zsplit_c2r": C + R}
    return per, 2 * R + 8 * C


def cpu_sample(n: int, config: int, kind=None, min_seconds: float = 10.0, max_runs: int = 3):
    """Time the oracle on a bounded sample: solve the config source at n^3 until
    min_seconds elapsed or max_runs done; returns (unknowns/s, kind, threads, runs)."""
    import numpy as np

    import oracle
    from paper_1408_6497_b200 import problems

    kind = kind or oracle.best_kind()
    threads = len(os.sched_getaffinity(0))
    oracle.set_threads(threads, kind)
    src = problems.config(config, n)
    f = _host_source(src)
    oracle.poisson_solve(f[:8, :8, :8].copy(), kind)  # warm the library
    runs, t0 = 0, time.perf_counter()
    while True:
        oracle.poisson_solve(f, kind)
        runs += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or runs >= max_runs:
            break
    return n ** 3 * runs / el, kind, threads, runs


def _host_source(src):
    """Config source on the host without the GPU: separable per-mode evaluation."""
    import numpy as np

    from paper_1408_6497_b200 import problems

    n = src.n
    if isinstance(src, problems.ModeSource):
        # Re sum a e^{2 pi i k.x} = inverse DFT of a sparse Hermitian spectrum (scipy pocketfft).
        import scipy.fft as sf

        F = np.zeros((n, n, n), dtype=np.complex128)
        for (kx, ky, kz), c in zip(src.k, src.f_coef()):
            F[kx % n, ky % n, kz % n] += 0.5 * c
            F[-kx % n, -ky % n, -kz % n] += 0.5 * np.conj(c)
        out = sf.ifftn(F, workers=len(os.sched_getaffinity(0)), overwrite_x=True).real * float(n) ** 3
        del F
        return np.ascontiguousarray(out)
    return problems.eval_host(src, "f")


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU solver on the host cores, rank 0 only."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_1408_6497_b200 import problems

    kind = oracle.best_kind()
    threads = len(os.sched_getaffinity(0))
    oracle.set_threads(threads, kind)
    n = args.cpu_n
    src = problems.config(args.config, n)
    f = _host_source(src)
    for _ in range(args.warmup):
        oracle.poisson_solve(f, kind)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.poisson_solve(f, kind)
    el = time.perf_counter() - t0
    v = n ** 3 * args.steps / el
    sample = (f"{n}^3 sample of config {args.config}'s source (same 64 modes), full solve per step; "
              f"engine: {'reference fft_solver.cpp over FFTW3-API shim (oracle/_ref)' if kind == 'ref' else 'C restatement (oracle/lib)'}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C{args.config}: {problems.CONFIG_TEXT[args.config]}", "n": args.n,
                   "sample_n": n},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference" if kind == "ref" else "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _inplace_parity(plan, src, f, sh, prec, block=64):
    """In-place mode: solve a fresh f once (u overwrites f) and compare with the analytic u
    generated block by block of planes — the gauge-aligned errors of arena_field_compare
    (problems.cpp:88-106) accumulated over the blocks in two passes, fp64 sums."""
    import torch

    from paper_1408_6497_b200 import problems

    n = src.n
    f64 = torch.empty((n, n, n), dtype=torch.float64, device="cuda") if prec != 64 else f
    problems.fill_device(src, "f", f64, 64, sh)
    f64 -= f64.mean()
    if prec != 64:
        f.copy_(f64)
        del f64
    plan.solve_device(f, f, sh)
    torch.cuda.synchronize()
    buf = torch.empty((block, n, n), dtype=torch.float64, device="cuda")
    su = sa = 0.0
    amax = 0.0
    for i0 in range(0, n, block):
        problems.fill_device(src, "u", buf, 64, sh, i0, block)
        su += f[i0:i0 + block].double().sum().item()
        sa += buf.sum().item()
        amax = max(amax, buf.abs().max().item())
    N = float(n) ** 3
    shift, mean_e = (sa - su) / N, sa / N
    d2 = e2 = dmax = 0.0
    for i0 in range(0, n, block):
        problems.fill_device(src, "u", buf, 64, sh, i0, block)
        d = f[i0:i0 + block].double() + shift - buf
        d2 += (d * d).sum().item()
        dmax = max(dmax, d.abs().max().item())
        e2 += ((buf - mean_e) ** 2).sum().item()
    del buf
    return math.sqrt(d2 / e2), dmax / amax


def run_ours(args, rank, world, local):
    import numpy as np
    import torch

    import paper_1408_6497_b200 as arena
    from paper_1408_6497_b200 import problems

    torch.cuda.set_device(local)
    dist = None  # single GPU (N > 1 runs the slab decomposition, run_slab)
    n, prec = args.n, args.precision
    elem = 8 if prec == 64 else 4
    dt = torch.float64 if prec == 64 else torch.float32
    src = problems.config(args.config, n)
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    # ---- inputs resident in HBM (f as fp64, rounded to fp32 for fp32 runs)
    f64 = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
    problems.fill_device(src, "f", f64, 64, sh)
    f64 -= f64.mean()
    f = f64 if prec == 64 else f64.float()
    inplace = args.inplace or n >= 2048
    if inplace and prec != 64:
        del f64
    u = f if inplace else torch.empty_like(f)
    plan = arena.Plan(n, prec, local)
    launches = plan.launches_per_solve

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        plan.solve_device(f, u, sh)
    torch.cuda.synchronize()

    # ---- timed region: K solves, CUDA events on the launching stream, per-kernel events inside.
    # n <= 256 replays a CUDA graph per solve, which per-kernel events would defeat: there
    # the K solves are timed as replayed and the per-kernel split comes from a second K.
    graphs = n <= 256 and os.environ.get("ARENA_FFT_GRAPHS", "1") != "0"
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(stage_events):
        plan.set_stage_timing(stage_events)
        barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            plan.solve_device(f, u, sh)
        end.record(stream)
        torch.cuda.synchronize()
        barrier()
        r = start.elapsed_time(end), plan.stage_times()
        plan.set_stage_timing(False)
        return r

    with ClockSampler(local) as clk:
        ms_total, (stage_ms, nsol) = timed(not graphs)
    if graphs:
        _, (stage_ms, nsol) = timed(True)
    if dist is not None:
        t = torch.tensor([ms_total], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = t.item()
    ms_step = ms_total / args.steps
    value = world * n ** 3 / (ms_step / 1e3)  # replicas: every rank solves its own n^3

    # ---- parity of the timed output vs the analytic solution (band-limited source: exact)
    # (device reductions, arena_field_compare: gauge-aligned as problems.cpp:88-106)
    if inplace:
        rel_an, linf_an = _inplace_parity(plan, src, f, sh, prec)
    else:
        ua = torch.empty((n, n, n), dtype=torch.float64, device="cuda")
        problems.fill_device(src, "u", ua, 64, sh)
        cmp = arena.field_compare(u if prec == 64 else u.double(), ua)
        rel_an, linf_an = cmp["rel_l2"], cmp["linf_rel"]
        del ua

    # ---- roofline of the dominant kernel
    peak, peak_kind = _peaks()
    per_kernel, b_solve = algorithmic_bytes(n, elem)
    dom = max(stage_ms, key=lambda k: stage_ms[k])
    dom_ms = stage_ms[dom] / nsol
    achieved = per_kernel[dom] / (dom_ms / 1e3) / 1e9
    traffic = None
    tf = os.path.join(REPO, "profiles", "traffic_latest.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"{n}_{prec}", {}).get(dom)
        except Exception:
            traffic = None
    kernels = {k: {"ms": stage_ms[k] / nsol, "alg_bytes": per_kernel[k],
                   "gbs": per_kernel[k] / (stage_ms[k] / nsol / 1e3) / 1e9,
                   "share": stage_ms[k] / sum(stage_ms.values())} for k in stage_ms}
    solve_gbs = b_solve / (ms_step / 1e3) / 1e9

    # ---- e2e through the public host API: pinned host f -> device -> solve -> host u, every step.
    # arena_poisson_solve_host_batch overlaps the copy-in of step s+1 and the copy-out of step s-1
    # with the solve of step s (PCIe is full duplex), the way a user streams many fields.
    e2e = None
    if inplace and not args.no_e2e:  # 4 pinned n^3 host buffers would not fit the host
        e2e = {"value": None, "unit": UNIT, "h2d_bytes_per_step": n ** 3 * elem, "d2h_bytes_per_step": n ** 3 * elem,
               "skipped": "in-place large-n run: the e2e host stream needs 4 pinned n^3 buffers"}
    elif not args.no_e2e:
        hf = [torch.empty((n, n, n), dtype=dt, pin_memory=True) for _ in range(2)]
        hu = [torch.empty((n, n, n), dtype=dt, pin_memory=True) for _ in range(2)]
        for h in hf:
            h.copy_(f)
        plan.solve_host(hf[0], hu[0])  # warm (allocates the plan's host-path buffers)
        ksteps = max(2, min(args.steps, 16))  # a stream of fields: pipeline fill/drain amortised
        plan.solve_host_batch([hf[s % 2] for s in range(2)], [hu[s % 2] for s in range(2)])  # warm batch buffers
        t0 = time.perf_counter()
        plan.solve_host_batch([hf[s % 2] for s in range(ksteps)], [hu[s % 2] for s in range(ksteps)])
        el = time.perf_counter() - t0
        t0 = time.perf_counter()
        plan.solve_host(hf[0], hu[0])
        el_single = time.perf_counter() - t0
        e2e = {"value": n ** 3 * ksteps / el, "unit": UNIT, "h2d_bytes_per_step": n ** 3 * elem,
               "d2h_bytes_per_step": n ** 3 * elem, "steps": ksteps, "ms_per_step": el / ksteps * 1e3,
               "api": "arena_poisson_solve_host_batch (pinned host buffers; copy-in/solve/copy-out overlapped)",
               "single_call_ms": el_single * 1e3,
               "single_call_value": n ** 3 / el_single}
        e2e["matches_device_path"] = bool(torch.allclose(hu[0], u.cpu()))
        del hf, hu

    # ---- CPU baseline (rank 0, N=1 only), bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            v, kind, threads, runs = cpu_sample(args.cpu_n, args.config)
            cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference" if kind == "ref" else "port",
                   "sample": f"{args.cpu_n}^3 solve(s) of config {args.config}'s source ({runs} run(s)), "
                             f"{'reference fft_solver.cpp over FFTW3-API shim' if kind == 'ref' else 'C restatement'}"
                             f", OpenMP over lines"}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": None, "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
            "dtype": "f64" if prec == 64 else "f32", "data": "synthetic",
            "config": {"workload": f"C{args.config}: {problems.CONFIG_TEXT[args.config]}", "n": n,
                       "precision": prec, "decomposition": "single-GPU" if world == 1 else f"{world} replicas",
                       "l2": f"inputs larger than L2 ({n ** 3 * elem / 1e9:.1f} GB field), no flush",
                       "in_place": inplace,
                       "path": "pow2" if plan.path == arena.PATH_POW2 else "generic"},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "solve_alg_bytes": b_solve, "solve_achieved_gbs": solve_gbs, "solve_frac": solve_gbs / peak,
                         "kernels": kernels},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,
            "clocks": clk.summary(),
            "parity": {"rel_l2_vs_analytic": rel_an, "linf_rel_vs_analytic": linf_an},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_slab(args, rank, world, local):
    """N > 1: slab decomposition over the ranks' GPUs, NCCL all-to-alls (strong scaling:
    the n^3 problem is fixed, each rank owns n/N planes)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1408_6497_b200 as arena
    from paper_1408_6497_b200 import problems

    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, prec = args.n, args.precision
    elem = 8 if prec == 64 else 4
    dt = torch.float64 if prec == 64 else torch.float32
    src = problems.config(args.config, n)
    pencil = args.decomp == "pencil"
    if pencil:
        if args.pgrid:
            pr, pc = (int(x) for x in args.pgrid.lower().split("x"))
        else:
            pr = 1
            while pr * pr * 4 <= world:
                pr *= 2
            pc = world // pr
        assert pr * pc == world, "pencil grid must cover all ranks"
    else:
        pr, pc = world, 1
    ni, nj = n // pr, n // pc
    i0, j0 = (rank // pc) * ni, (rank % pc) * nj
    stream = torch.cuda.current_stream()
    sh = stream.cuda_stream

    # this rank's block of f, global mean removed
    f64 = torch.empty((ni, nj, n), dtype=torch.float64, device="cuda")
    problems.fill_device(src, "f", f64, 64, sh, i0, ni, j0, nj)
    tot = f64.sum().reshape(1)
    dist.all_reduce(tot)
    f64 -= tot.item() / float(n) ** 3
    f = f64 if prec == 64 else f64.float()
    u = torch.empty_like(f)

    ua = torch.empty((ni, nj, n), dtype=torch.float64, device="cuda")
    problems.fill_device(src, "u", ua, 64, sh, i0, ni, j0, nj)

    def rel_vs_analytic():
        sums = torch.stack([ua.sum()])
        dist.all_reduce(sums)
        mean_u = sums[0].item() / float(n) ** 3
        d2 = torch.stack([((u.double() - (ua - mean_u)) ** 2).sum(), ((ua - mean_u) ** 2).sum()])
        dist.all_reduce(d2)
        return (d2[0] / d2[1]).sqrt().item()

    def make_nccl():
        nb = arena.lib.arena_nccl_unique_id_bytes()
        idt = torch.zeros(nb, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(arena.nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nid = bytes(idt.cpu().numpy().tobytes())
        if pencil:
            return arena.Pencil(n, pr, pc, rank=rank, nccl_id=nid, precision=prec, device=local)
        return arena.Slab(n, world, rank=rank, nccl_id=nid, precision=prec, device=local)

    def vote(ok):  # every rank takes the same branch
        t = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        return t.item() == 1

    def try_peer():
        nb = arena.lib.arena_pencil_peer_handle_bytes() if pencil else arena.lib.arena_slab_peer_handle_bytes()
        s, err = None, None
        try:
            if pencil:
                s = arena.Pencil(n, pr, pc, rank=rank, peer=True, precision=prec, device=local)
            else:
                s = arena.Slab(n, world, rank=rank, peer=True, precision=prec, device=local)
            hb = s.peer_handles()
        except Exception as exc:
            err, hb = exc, bytes(nb)
        h = torch.frombuffer(bytearray(hb), dtype=torch.uint8).cuda()
        hs = [torch.empty_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        if not vote(err is None):
            return None, err or "another rank failed to export"
        try:
            s.peer_attach(b"".join(bytes(x.cpu().numpy().tobytes()) for x in hs))
        except Exception as exc:
            err = exc
        if not vote(err is None):
            return None, err or "another rank failed to attach"
        try:
            for _ in range(max(1, args.warmup)):
                s.solve_device(f, u, sh)
            torch.cuda.synchronize()
            s.barrier_status()
        except Exception as exc:
            err = exc
        if not vote(err is None):
            return None, err or "another rank failed"
        r = rel_vs_analytic()
        if not r <= (1e-12 if prec == 64 else 1e-5):
            return None, f"parity {r:.2e}"
        return s, None

    xchg = args.xchg
    note = None
    slab = None
    if xchg == "peer":
        slab, err = try_peer()
        if slab is None:  # fall back to the NCCL exchange, and say so
            note = f"peer exchange unavailable ({err}); NCCL used"
            xchg = "nccl"
    if slab is None:
        slab = make_nccl()

    for _ in range(args.warmup):
        slab.solve_device(f, u, sh)
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            slab.solve_device(f, u, sh)
        end.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    t = torch.tensor([start.elapsed_time(end)], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = t.item() / args.steps
    value = n ** 3 / (ms_step / 1e3)

    if xchg == "peer":
        slab.barrier_status()
    rel_an = rel_vs_analytic()

    peak, peak_kind = _peaks()
    _, b_solve = algorithmic_bytes(n, elem)
    C = n * n * (n // 2 + 1) * 2 * elem
    hbm_per_gpu = b_solve / world
    if pencil:
        nvl_per_gpu = 2 * (C / world) * ((pr - 1) / pr + (pc - 1) / pc)
    else:
        nvl_per_gpu = 2 * (C / world) * (world - 1) / world
    nvl_peak = 770.0  # GB/s per direction, measured peer copy (B200_PROFILING.md)
    t_roof = max(hbm_per_gpu / (peak * 1e9), nvl_per_gpu / (nvl_peak * 1e9))

    e2e = None
    if not args.no_e2e:
        hf = torch.empty((ni, nj, n), dtype=dt, pin_memory=True)
        hf.copy_(f)
        hu = torch.empty_like(hf, pin_memory=True)
        ksteps = max(1, min(args.steps, 3))
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(ksteps):
            f.copy_(hf, non_blocking=True)
            slab.solve_device(f, u, sh)
            hu.copy_(u, non_blocking=True)
            torch.cuda.synchronize()
        el = time.perf_counter() - t0
        te = torch.tensor([el], device="cuda", dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        el = te.item()
        e2e = {"value": n ** 3 * ksteps / el, "unit": UNIT, "h2d_bytes_per_step": n ** 3 * elem,
               "d2h_bytes_per_step": n ** 3 * elem, "steps": ksteps, "ms_per_step": el / ksteps * 1e3,
               "api": "arena_slab/pencil_solve_device with per-rank pinned H2D/D2H of the rank's block"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64" if prec == 64 else "f32", "data": "synthetic",
            "config": {"workload": f"C{args.config}: {problems.CONFIG_TEXT[args.config]}", "n": n, "precision": prec,
                       "decomposition": ((f"pencil {pr}x{pc}, " + (
                                             "4 row/column all-to-alls fused into K1-K4 as stores into the peers' "
                                             "buffers (CUDA IPC over NVLink) + device flag barriers"
                                             if xchg == "peer" else "NCCL row/column all-to-alls (4 per solve)"))
                                         if pencil else f"slab x{world} over i, " + (
                                             "all-to-alls fused into K2/K3 as stores into the peers' "
                                             "workspaces (CUDA IPC over NVLink) + device flag barriers"
                                             if xchg == "peer" else "NCCL grouped send/recv all-to-all")),
                       "exchange": xchg, "exchange_note": note,
                       "l2": "inputs larger than L2, no flush"},
            "roofline": {"bound": "hbm+nvlink", "achieved": hbm_per_gpu / (ms_step / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": t_roof / (ms_step / 1e3), "traffic": None, "peak_kind": peak_kind,
                         "nvlink_bytes_per_gpu": nvl_per_gpu, "nvlink_peak_gbs": nvl_peak,
                         "t_roof_ms": t_roof * 1e3},
            "cpu_baseline": None,
            "e2e": e2e,
            "gpu_launches": slab.launches_per_solve * args.steps,
            "clocks": clk.summary(),
            "parity": {"rel_l2_vs_analytic": rel_an},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def main():
    args = _args()
    rank, world, local = _dist()
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif world > 1 or args.slab or args.pgrid:
        run_slab(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
