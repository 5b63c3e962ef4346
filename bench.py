#!/usr/bin/env python3
"""Benchmark of the spectral Poisson solve (BASELINE.json metric: Poisson
unknowns solved/sec, fp64 FFT solve, % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 1024] [--impl ours|reference]

One step = one full solve (r2c 3D FFT, Poisson scale, c2r 3D FFT) of the
BASELINE config-4 source (1024^3 fp64, 64 random Fourier modes, seed 4),
inputs resident in HBM.  The field (8.6 GB) is far larger than L2 (126 MB),
so no L2 flush is needed between steps.  Prints ONE JSON line on rank 0.

--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one rank per GPU, 127.0.0.1) and runs the slab decomposition (strong scaling).

--impl reference times the reference's own CPU solver (fft_solver.cpp:51-87,
compiled unmodified over the FFTW3-API shim: oracle/_ref) on all host cores,
each step one full solve of the SAME n^3 config source (same_config), plus one
1-core solve (the reference's FFTW is single-threaded) and a scipy pocketfft
all-core restatement ("B-all").  That arm never loads this
repo's CUDA library (checked against /proc/self/maps).
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
    ap.add_argument("--cpu-runs", type=int, default=3, help="CPU baseline: median of this many full solves")
    ap.add_argument("--no-one-core", action="store_true", help="reference arm: skip the 1-core solve")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: gloo ranks, no solve, one JSON line")
    ap.add_argument("--slab", action="store_true", help="use the slab (NCCL) path even with one rank")
    ap.add_argument("--decomp", default="slab", choices=("slab", "pencil"), help="multi-GPU decomposition")
    ap.add_argument("--pgrid", default=None, help="pencil process grid RxC (default: near-square, R <= C)")
    ap.add_argument("--fold", action="store_true",
                    help="pencil: folded distribution (quadrant z passes, n/2-point strided passes; default at n >= 2048)")
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


def _workload(config: int, n: int, prec: int) -> str:
    """config.workload text; fp32 runs solve the fp64 source rounded to fp32."""
    from paper_1408_6497_b200 import problems

    txt = problems.CONFIG_TEXT[config]
    base_n = {1: 64, 2: 256, 3: 512, 4: 1024, 5: 2048}[config]
    if n != base_n:
        txt = txt.replace(f"N={base_n}^3", f"N={n}^3")
    if prec == 32:
        txt = txt.replace("fp64", "fp32 (f rounded from the fp64 source)")
    return f"C{config}: {txt}"


def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _median(xs):
    xs = sorted(xs)
    m = len(xs) // 2
    return xs[m] if len(xs) % 2 else 0.5 * (xs[m - 1] + xs[m])


def _repo_libs_mapped():
    """This repo's shared objects mapped into the process (the reference arm must map
    none of paper_1408_6497_b200/lib; oracle/ libraries are the reference's own code)."""
    out = set()
    try:
        with open("/proc/self/maps") as fh:
            for ln in fh:
                path = ln.split()[-1] if len(ln.split()) >= 6 else ""
                if path.startswith(REPO) and ".so" in path:
                    out.add(os.path.relpath(path, REPO))
    except OSError:
        pass
    return sorted(out)


def cpu_reference_solves(f, runs: int, threads: int):
    """Time `runs` full solves of the host field f by the reference's own solver
    (fft_solver.cpp:51-87 over the FFTW3-API shim; the C restatement where the
    reference was not built).  Returns (per-run seconds, kind, the last u)."""
    import oracle

    kind = oracle.best_kind()
    oracle.set_threads(threads, kind)
    ts, u = [], None
    for _ in range(runs):
        u = None
        t0 = time.perf_counter()
        u = oracle.poisson_solve(f, kind)
        ts.append(time.perf_counter() - t0)
    return ts, kind, u


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU solver on the host cores, rank 0 only,
    each step one full solve of the same n^3 source the GPU arm solves."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_1408_6497_b200 import problems  # pure Python: the package maps no CUDA library on import

    n = args.n
    threads = len(os.sched_getaffinity(0))
    src = problems.config(args.config, n)
    t0 = time.perf_counter()
    f = problems.host_field(src, "f")
    f -= f.mean()
    t_src = time.perf_counter() - t0
    kind = oracle.best_kind()
    oracle.set_threads(threads, kind)
    for _ in range(args.warmup):
        oracle.poisson_solve(f, kind)
    ts, kind, u = cpu_reference_solves(f, args.steps, threads)
    el = sum(ts)
    v = n ** 3 * args.steps / el
    engine = ("reference fft_solver.cpp (unmodified) over the FFTW3-API shim, oracle/_ref" if kind == "ref"
              else "C restatement of fft_solver.cpp, oracle/lib")
    parity = {}
    if isinstance(src, problems.ModeSource) and 2 * int(abs(src.k).max()) < n:  # resolved and band-limited:
        # the analytic u is exact on the grid (coarser grids alias the modes)
        ua = problems.host_field(src, "u")
        ua -= ua.mean()
        parity["rel_l2_vs_analytic"] = float(np.linalg.norm(u - ua) / np.linalg.norm(ua))
        del ua
    extras = {}
    # the reference's FFTW is single-threaded (no fftw_init_threads, proj/src/CMakeLists.txt:3,17)
    if not args.no_one_core:
        t1, _, _ = cpu_reference_solves(f, 1, 1)
        extras["one_core"] = {"value": n ** 3 / t1[0], "unit": UNIT, "cores": 1, "s_per_solve": t1[0],
                              "kind": "reference" if kind == "ref" else "port",
                              "note": "reference-faithful: FFTW single-threaded, one full solve"}
    # B-all: the strongest CPU engine here (scipy pocketfft, all cores), median of 3
    tb, ub = [], None
    for _ in range(3):
        t0 = time.perf_counter()
        ub = oracle.pocketfft_poisson(f, threads)
        tb.append(time.perf_counter() - t0)
    extras["b_all"] = {"value": n ** 3 / _median(tb), "unit": UNIT, "cores": threads, "s_per_solve": _median(tb),
                       "runs": len(tb), "kind": "port",
                       "engine": "scipy.fft pocketfft restatement of fft_solver.cpp:51-87 (oracle.pocketfft_poisson)",
                       "rel_l2_vs_reference": float(np.linalg.norm(ub - u) / np.linalg.norm(u))}
    del ub
    mapped = _repo_libs_mapped()
    sample = (f"full {n}^3 solves of config {args.config}'s source (the GPU arm's workload), one per step; "
              f"engine: {engine}; {threads} OpenMP threads on the FFT lines (the reference's own copies, "
              f"zero-fills and scale loop run single-threaded as written)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": _workload(args.config, n, 64), "n": n, "sample_n": n, "same_config": True,
                   "source_seconds": t_src},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "reference" if kind == "ref" else "port",
                         "sample": sample, "cpu_model": _cpu_model(), "s_per_solve_median": _median(ts), **extras},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": parity,
        "repo_libs_mapped": mapped,
    }
    if any(m.startswith("paper_1408_6497_b200") for m in mapped):
        line["invalid"] = "the reference arm mapped this repo's CUDA library"
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

    # ---- CPU baseline (rank 0, N=1 only) on the IDENTICAL fp64 buffer the GPU solved, before any
    # pinned allocation: the reference's own solver, median of --cpu-runs full solves; its output
    # is also the oracle the timed GPU output is compared with (north_star: rel L2 <= 1e-12 fp64,
    # <= 1e-5 fp32 against the fp64 oracle).
    cpu, rel_or = None, None
    if rank == 0 and world == 1 and not args.no_cpu and not inplace:
        try:
            fh = f64.cpu().numpy()
            threads = len(os.sched_getaffinity(0))
            ts, kind, uo = cpu_reference_solves(fh, max(1, args.cpu_runs), threads)
            del fh
            uo_d = torch.from_numpy(uo).to("cuda")
            del uo
            ud = u.double() if prec != 64 else u
            rel_or = ((ud - uo_d).norm() / uo_d.norm()).item()
            del uo_d, ud
            cpu = {"value": n ** 3 / _median(ts), "unit": UNIT, "cores": threads,
                   "kind": "reference" if kind == "ref" else "port",
                   "sample": f"the same {n}^3 fp64 field the GPU solved, {len(ts)} full solve(s), median; "
                             + ("reference fft_solver.cpp (unmodified) over the FFTW3-API shim (oracle/_ref)"
                                if kind == "ref" else "C restatement (oracle/lib)")
                             + f", {threads} OpenMP threads on the FFT lines",
                   "s_per_solve": ts, "cpu_model": _cpu_model()}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": None, "sample": f"failed: {exc}"}

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

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak" if world > 1 else "strong", "vs_baseline": None,
            "dtype": "f64" if prec == 64 else "f32", "data": "synthetic",
            "config": {"workload": _workload(args.config, n, prec), "n": n,
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
            "parity": {"rel_l2_vs_analytic": rel_an, "linf_rel_vs_analytic": linf_an, "rel_l2_vs_oracle": rel_or,
                       "tolerance_vs_oracle": 1e-12 if prec == 64 else 1e-5},
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def _nccl_init_lines():
    """This rank's NCCL communicator-creation lines (NCCL_DEBUG=INFO into the file _relaunch set)."""
    import socket

    path = os.path.join("/tmp", f"arena_bench_nccl.{socket.gethostname()}.{os.getpid()}.log")
    try:
        with open(path) as fh:
            return [ln.strip() for ln in fh if "Init COMPLETE" in ln or "nranks" in ln.lower()][-4:]
    except OSError:
        return None


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
    # folded pencil (quadrant z passes, n/2-point strided tiles): default at n >= 2048, where the
    # plain pencil's n-point y / x tiles no longer fit 128-byte rows
    fold = pencil and (args.fold or n >= 2048)

    def fill_block(which, out):
        if not fold:
            problems.fill_device(src, which, out, 64, sh, i0, ni, j0, nj)
            return
        for gi, gj, li, lj, bi, bj in arena.fold_blocks(n, pr, pc, rank // pc, rank % pc):
            tmp = torch.empty((bi, bj, n), dtype=torch.float64, device="cuda")
            problems.fill_device(src, which, tmp, 64, sh, gi, bi, gj, bj)
            out[li:li + bi, lj:lj + bj].copy_(tmp)
            del tmp

    fill_block("f", f64)
    tot = f64.sum().reshape(1)
    dist.all_reduce(tot)
    f64 -= tot.item() / float(n) ** 3
    f = f64 if prec == 64 else f64.float()
    u = torch.empty_like(f)

    ua = torch.empty((ni, nj, n), dtype=torch.float64, device="cuda")
    fill_block("u", ua)

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
            return arena.Pencil(n, pr, pc, rank=rank, nccl_id=nid, precision=prec, device=local, folded=fold)
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
                s = arena.Pencil(n, pr, pc, rank=rank, peer=True, precision=prec, device=local, folded=fold)
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

    # ---- per-stage times (a second, separately timed run with events between the stages;
    # the headline region above has no extra events), max over ranks per stage
    stages = None
    if not pencil:
        slab.set_stage_timing(True)
        kst = max(1, min(args.steps, 5))
        dist.barrier()
        for _ in range(kst):
            slab.solve_device(f, u, sh)
        torch.cuda.synchronize()
        st_ms, nst = slab.stage_times()
        slab.set_stage_timing(False)
        tt = torch.tensor([st_ms[k] / nst for k in arena.Slab.STAGES], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        stages = {k: tt[i].item() for i, k in enumerate(arena.Slab.STAGES)}

    peak, peak_kind = _peaks()
    _, b_solve = algorithmic_bytes(n, elem)
    C = n * n * (n // 2 + 1) * 2 * elem
    hbm_per_gpu = b_solve / world
    if pencil:
        nvl_per_gpu = 2 * (C / world) * ((pr - 1) / pr + (pc - 1) / pc)
    else:
        nvl_per_gpu = 2 * (C / world) * (world - 1) / world
    nvl_peak = 770.0  # GB/s per direction, measured peer copy (B200_PROFILING.md)
    nvl_spec = 900.0  # NVLink 5, 18 links, per direction
    t_roof = max(hbm_per_gpu / (peak * 1e9), nvl_per_gpu / (nvl_peak * 1e9))
    nvlink = {"bytes_per_gpu_per_solve": nvl_per_gpu, "peak_gbs_measured_copy": nvl_peak, "spec_gbs": nvl_spec,
              "achieved_gbs_whole_solve": nvl_per_gpu / (ms_step / 1e3) / 1e9}
    if stages is not None:
        # exchange #1 leaves in K2 (peer stores) or in the NCCL send/recv after it; #2 in K3 / after it
        sent = slab.chunk_bytes * (world - 1)
        ph1 = stages["xchg1"] + (stages["k1k2"] if xchg == "peer" else 0.0)
        ph2 = stages["xchg2"] + (stages["k3"] if xchg == "peer" else 0.0)
        nvlink.update({"bytes_sent_per_exchange": sent, "stage_ms": stages,
                       "exchange_gbs": [sent / (ph1 / 1e3) / 1e9 if ph1 > 0 else None,
                                        sent / (ph2 / 1e3) / 1e9 if ph2 > 0 else None],
                       "exchange_gbs_note": ("peer: bytes over the time of the pass that stores them (K2 / K3) "
                                             "plus its barrier" if xchg == "peer" else
                                             "nccl: bytes over the grouped send/recv stage")})

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
            "config": {"workload": _workload(args.config, n, prec), "n": n, "precision": prec,
                       "decomposition": ((f"pencil {pr}x{pc}, " + (
                                             "4 row/column all-to-alls fused into K1-K4 as stores into the peers' "
                                             "buffers (CUDA IPC over NVLink) + device flag barriers"
                                             if xchg == "peer" else "NCCL row/column all-to-alls (4 per solve)"))
                                         if pencil else f"slab x{world} over i, " + (
                                             "all-to-alls fused into K2/K3 as stores into the peers' "
                                             "workspaces (CUDA IPC over NVLink) + device flag barriers"
                                             if xchg == "peer" else "NCCL grouped send/recv all-to-all")),
                       "exchange": xchg, "exchange_note": note, "folded": fold,
                       "l2": "inputs larger than L2, no flush"},
            "roofline": {"bound": "hbm+nvlink", "achieved": hbm_per_gpu / (ms_step / 1e3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": t_roof / (ms_step / 1e3), "traffic": None, "peak_kind": peak_kind,
                         "nvlink_bytes_per_gpu": nvl_per_gpu, "nvlink_peak_gbs": nvl_peak,
                         "t_roof_ms": t_roof * 1e3},
            "nvlink": nvlink,
            "nccl_init": _nccl_init_lines(),
            "cpu_baseline": None,
            "cpu_baseline_note": "measured on rank 0 at N=1 only (bench.py --gpus 1)",
            "e2e": e2e,
            "gpu_launches": slab.launches_per_solve * args.steps,
            "clocks": clk.summary(),
            "parity": {"rel_l2_vs_analytic": rel_an},
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def _free_port() -> int:
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _relaunch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: one rank per GPU under
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    env = dict(os.environ)
    if "NCCL_DEBUG" not in env:  # NCCL communicator creation stays checkable, off stdout
        env["NCCL_DEBUG"] = "INFO"
        env["NCCL_DEBUG_SUBSYS"] = "INIT"
        env["NCCL_DEBUG_FILE"] = os.path.join("/tmp", "arena_bench_nccl.%h.%p.log")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd, env=env).returncode


def run_dry(args, rank, world):
    """Launcher check (no GPU, gloo): every rank joins, the max over ranks of a per-rank
    number is reduced as the real timing is, rank 0 prints one line."""
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "dry_run": True, "max_over_ranks": t.item(),
                          "world_size": dist.get_world_size()}), flush=True)
    dist.destroy_process_group()


def main():
    args = _args()
    launched = "WORLD_SIZE" in os.environ
    if not launched and args.gpus > 1 and args.impl == "ours":
        sys.exit(_relaunch(args))
    rank, world, local = _dist()
    if launched and args.gpus != world and args.impl == "ours":
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}\n")
        sys.exit(2)
    if args.dry_run:
        run_dry(args, rank, world)
    elif args.impl == "reference":
        run_reference(args, rank, world if launched else args.gpus)
    elif world > 1 or args.slab or args.pgrid:
        run_slab(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
