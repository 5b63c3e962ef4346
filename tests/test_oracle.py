"""CPU tests: the oracle is pinned to the reference before anything is compared to it."""
import os
import subprocess

import numpy as np
import pytest

import oracle
from paper_1408_6497_b200 import problems

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _rel(a, b):
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d > 0 else 1.0)


@pytest.mark.parametrize("exe", [oracle.TEST_FFT_REF, oracle.TEST_PROBLEMS_REF])
def test_reference_own_tests_pass_on_oracle(exe, tmp_path):
    """The reference's unmodified test_fft.cpp / test_problems.cpp (T1-T12)
    against the reference's fft_solver.cpp over the FFTW3-API shim."""
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref not built here (needs /root/reference): make -C oracle ref")
    r = subprocess.run([exe], cwd=tmp_path, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert " 0 failed" in r.stdout


@pytest.mark.parametrize("kind", ["port", "ref"])
def test_oracle_matches_golden_poisson(kind):
    if not oracle.available(kind):
        pytest.skip(f"oracle {kind} not built")
    z = np.load(os.path.join(GOLDEN, "poisson_golden.npz"))
    names = sorted({k[:-2] for k in z.files})
    assert len(names) >= 14
    for name in names:
        u = oracle.poisson_solve(z[name + "_f"], kind)
        assert _rel(u, z[name + "_u"]) <= 1e-14 or np.abs(u - z[name + "_u"]).max() < 1e-15, name


@pytest.mark.parametrize("kind", ["port", "ref"])
def test_oracle_matches_golden_dft3(kind):
    if not oracle.available(kind):
        pytest.skip(f"oracle {kind} not built")
    z = np.load(os.path.join(GOLDEN, "dft3_golden.npz"))
    for n in (2, 4, 6, 8, 10):
        g, s = z[f"dft_n{n}_g"], z[f"dft_n{n}_spec"]
        assert _rel(oracle.dft3_forward(g, kind), s) <= 1e-14
        assert _rel(oracle.dft3_inverse(s, n, kind), g) <= 1e-14


def test_port_vs_direct_dft():
    """oracle::direct_dft3 semantics (oracles.cpp:13-29) at n = 3, 4 (T3 uses n = 4)."""
    for n in (3, 4):
        g = np.random.default_rng(99).uniform(-1, 1, (n, n, n))
        fast = oracle.dft3_forward(g, "port")
        slow = oracle.direct_dft3(g)
        assert np.abs(fast - slow).max() <= 1e-12 * np.abs(slow).max()


def test_port_single_mode_exact():
    """T5 (test_fft.cpp:82-92): f = 4 pi^2 sin(2 pi x1) -> u = sin(2 pi x1), abs 1e-12."""
    for n in (4, 8, 16):
        x = np.arange(n) / n
        f = np.broadcast_to(4 * np.pi ** 2 * np.sin(2 * np.pi * x)[:, None, None], (n, n, n)).copy()
        u = oracle.poisson_solve(f, "port")
        assert np.abs(u - np.sin(2 * np.pi * x)[:, None, None]).max() < 1e-12


def test_port_analytic_modes_and_gaussian():
    """Config sources at small n: oracle solve vs analytic u (spectral accuracy)."""
    src = problems.random_modes(32, 16, 5, seed=11)
    u = oracle.poisson_solve(problems.eval_host(src, "f"), "port")
    assert _rel(u, problems.eval_host(src, "u")) < 1e-13
    g = problems.gaussian(64, 300.0, seed=3)
    f = problems.eval_host(g, "f")
    u = oracle.poisson_solve(f - f.mean(), "port")
    ua = problems.eval_host(g, "u")
    assert _rel(u, ua - ua.mean()) < 1e-9


def test_mt19937_64_matches_std():
    """C++ [rand.predef]: the 10000th draw of default-seeded std::mt19937_64 is 9981545732273789042."""
    r = problems.MT19937_64()
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042


def test_config_sources_deterministic():
    a, b = problems.config(4), problems.config(4)
    assert a.k.shape == (64, 3) and np.array_equal(a.k, b.k) and np.array_equal(a.a, b.a)
    assert np.all(np.abs(a.k) <= 32) and not np.any(np.all(a.k == 0, axis=1))
    c = problems.config(2)
    assert c.k.shape == (32, 3) and np.all(np.abs(c.k) <= 8)
    g = problems.config(3)
    assert all(0.0 <= x < 1.0 for x in g.center) and g.alpha == 1e4


@pytest.mark.parametrize("n", [2, 3, 5, 6, 7, 9, 12, 16, 30, 64, 96])
def test_shim_engine_vs_independent_restatement(n):
    """The FFTW stand-in behind the shim (oracle/fftw_shim/vfft.c: Stockham, 8 lines per
    SIMD batch, two real rows per complex FFT) against the independent recursive
    restatement (oracle/offt.c) — odd n, odd row counts, generic radices."""
    if not oracle.available("ref"):
        pytest.skip("oracle/_ref not built")
    f = np.random.default_rng(n).standard_normal((n, n, n))
    a, b = oracle.poisson_solve(f, "ref"), oracle.poisson_solve(f, "port")
    assert _rel(a, b) <= 1e-14
    g = np.random.default_rng(n + 1).standard_normal((n, n, n))
    assert _rel(oracle.dft3_forward(g, "ref"), oracle.dft3_forward(g, "port")) <= 1e-14


def test_pocketfft_restatement_vs_reference():
    """B-all engine of the CPU baseline (scipy pocketfft) against the reference solver."""
    for n in (6, 7, 32):
        f = np.random.default_rng(n).standard_normal((n, n, n))
        assert _rel(oracle.pocketfft_poisson(f), oracle.poisson_solve(f)) <= 1e-14
