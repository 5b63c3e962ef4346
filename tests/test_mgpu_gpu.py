"""One process, several GPUs (arena_mgpu_*, the drop-in's ARENA_FFT_NGPU path).

The GPU pool gives one B200 per call, so the ranks are placed on device 0 by
passing devices=[0]*P: every code path runs — per-rank workspaces, peer-store
K2 / K3 into the other ranks' workspaces, cross-device-event phase ordering,
parallel per-rank host copies — except the physical NVLink transfer, which
a multi-GPU box adds (cudaDeviceEnablePeerAccess between distinct devices)."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import paper_1408_6497_b200 as arena

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("n,P", [(16, 2), (32, 4), (64, 8), (128, 2), (256, 4)])
def test_mgpu_host_vs_oracle(cuda, n, P):
    f = np.random.default_rng(n * P).uniform(-1, 1, (n, n, n))
    m = arena.MultiGPU(n, P, devices=[0] * P)
    u = np.empty_like(f)
    m.solve_host(f, u)
    assert _rel(u, oracle.poisson_solve(f)) <= 1e-12
    u2 = np.empty_like(f)
    m.solve_host(f, u2)  # repeated: same streams, events, staging
    assert np.array_equal(u, u2)
    m.close()


@pytest.mark.parametrize("n,P", [(64, 2), (256, 8)])
def test_mgpu_device_shards_vs_oracle(cuda, n, P):
    torch = cuda
    f = np.random.default_rng(n + P).uniform(-1, 1, (n, n, n))
    m = arena.MultiGPU(n, P, devices=[0] * P)
    ni = n // P
    fs = [torch.from_numpy(f[v * ni:(v + 1) * ni].copy()).cuda() for v in range(P)]
    us = [torch.empty_like(x) for x in fs]
    m.solve_device(fs, us)
    torch.cuda.synchronize()
    u = np.concatenate([x.cpu().numpy() for x in us])
    assert _rel(u, oracle.poisson_solve(f)) <= 1e-12
    m.solve_device(fs, fs)  # in place
    torch.cuda.synchronize()
    assert _rel(np.concatenate([x.cpu().numpy() for x in fs]), oracle.poisson_solve(f)) <= 1e-12
    m.close()


def test_mgpu_fp32(cuda):
    n, P = 128, 4
    f = np.random.default_rng(3).uniform(-1, 1, (n, n, n))
    m = arena.MultiGPU(n, P, devices=[0] * P, precision=32)
    u = np.empty((n, n, n), dtype=np.float32)
    m.solve_host(f.astype(np.float32), u)
    assert _rel(u.astype(np.float64), oracle.poisson_solve(f.astype(np.float32).astype(np.float64))) <= 1e-5


def test_mgpu_rejects_bad_sizes(cuda):
    with pytest.raises(Exception):
        arena.MultiGPU(12, 2)  # not a power of two
    with pytest.raises(Exception):
        arena.MultiGPU(16, 16)  # more than 8 ranks


@pytest.mark.parametrize("ngpu", ["2", "4"])
def test_reference_test_fft_dropin_multi_gpu(cuda, tmp_path, ngpu):
    """The reference's unmodified tests/test_fft.cpp against the drop-in with
    ARENA_FFT_NGPU set: poisson_spectral_solve of the power-of-two grids runs on
    the multi-GPU path (ranks on device 0 here), the rest on one GPU."""
    if not os.path.exists(oracle.TEST_FFT_DROPIN):
        pytest.fail("oracle/_ref/test_fft_dropin not built")
    env = dict(os.environ, ARENA_FFT_NGPU=ngpu, ARENA_FFT_DEVICES=",".join(["0"] * int(ngpu)))
    r = subprocess.run([oracle.TEST_FFT_DROPIN], cwd=tmp_path, capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
