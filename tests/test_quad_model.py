"""CPU model of the quadrant formulation (csrc/poisson_quad.cuh), no GPU.

For n = 2H the z passes apply the first radix-2 step of the i and j transforms
to each row quad, Y_{ci,cj}[i',j',k] = W_n^{ci i' + cj j'} sum_{a,b} (-1)^{a ci + b cj}
X[i' + aH, j' + bH, k] (X = the rows' r2c spectra), after which the H x H 2-D DFT of
Y_{ci,cj} over (i', j') is the full spectrum at (2 i'' + ci, 2 j'' + cj).  The
inverse z pass undoes the step.  Checked here with numpy FFTs against the direct
3-D r2c / c2r of the reference's convention (fft_solver.cpp:60-80), and the Poisson
symbol with the quadrant frequencies against the oracle's solve.
"""
import numpy as np
import pytest

import oracle


def _hadamard(x):  # x[a, b] -> y[ci, cj] = sum (-1)^{a ci + b cj} x[a, b]
    s0, d0 = x[0, 0] + x[0, 1], x[0, 0] - x[0, 1]
    s1, d1 = x[1, 0] + x[1, 1], x[1, 0] - x[1, 1]
    return np.array([[s0 + s1, d0 + d1], [s0 - s1, d0 - d1]])


def _quad_forward(f):
    n = f.shape[0]
    H = n // 2
    X = np.fft.rfft(f, axis=2)  # rows' r2c (K1's row transform)
    x = X.reshape(2, H, 2, H, -1).transpose(0, 2, 1, 3, 4)  # [a, b, i', j', k]
    y = _hadamard(x)
    ip = np.arange(H)[:, None]
    jp = np.arange(H)[None, :]
    for ci in range(2):
        for cj in range(2):
            y[ci, cj] *= np.exp(-2j * np.pi * (ci * ip + cj * jp) / n)[..., None]
    return y  # [ci, cj, i', j', k]


@pytest.mark.parametrize("n", [4, 8, 16, 32])
def test_quadrant_split_reproduces_spectrum(n):
    f = np.random.default_rng(n).uniform(-1, 1, (n, n, n))
    y = _quad_forward(f)
    full = np.fft.rfftn(f)
    for ci in range(2):
        for cj in range(2):
            sub = np.fft.fft2(y[ci, cj], axes=(0, 1))
            assert np.allclose(sub, full[ci::2, cj::2], rtol=0, atol=1e-10 * np.abs(full).max())


@pytest.mark.parametrize("n", [8, 16, 32])
def test_quadrant_solve_matches_oracle(n):
    """Whole solve in the quadrant order: split, H-point 2-D DFTs, symbol at
    (2 i'' + ci, 2 j'' + cj, k), inverse 2-D DFTs, inverse step, rows' c2r."""
    f = np.random.default_rng(100 + n).uniform(-1, 1, (n, n, n))
    H = n // 2
    y = _quad_forward(f)
    sf = lambda m: np.where(m <= n // 2, m, m - n)  # signed_freq, fft_solver.hpp:19
    kk = np.arange(n // 2 + 1)
    out = np.empty_like(y)
    for ci in range(2):
        for cj in range(2):
            s = np.fft.fft2(y[ci, cj], axes=(0, 1))
            ki = sf(2 * np.arange(H) + ci)[:, None, None]
            kj = sf(2 * np.arange(H) + cj)[None, :, None]
            k2 = (ki * ki + kj * kj + kk[None, None, :] ** 2).astype(np.float64)
            with np.errstate(divide="ignore"):
                m = np.where(k2 == 0, 0.0, (1.0 / n ** 3) / (4 * np.pi ** 2 * k2))
            out[ci, cj] = np.fft.ifft2(s * m, axes=(0, 1)) * H * H  # unnormalised inverse
    ip = np.arange(H)[:, None]
    jp = np.arange(H)[None, :]
    for ci in range(2):
        for cj in range(2):
            out[ci, cj] *= np.exp(2j * np.pi * (ci * ip + cj * jp) / n)[..., None]
    x = _hadamard(out)  # [a, b, i', j', k]
    X = x.transpose(0, 2, 1, 3, 4).reshape(n, n, -1)
    u = np.fft.irfft(X, n=n, axis=2) * n  # unnormalised c2r
    ref = oracle.poisson_solve(f)
    assert np.linalg.norm(u - ref) <= 1e-12 * np.linalg.norm(ref)


@pytest.mark.parametrize("R,M", [(3, 2), (3, 4), (3, 8), (5, 2), (5, 4)])
def test_radix3_split_reproduces_spectrum(R, M):
    """The radix-3 split of poisson_split3.cuh: Y_{ci,cj} = W_n^{ci i' + cj j'}
    sum_{a,b} W_3^{a ci + b cj} X[i' + aM, j' + bM]; its M x M DFT is the spectrum
    at (3 i'' + ci, 3 j'' + cj)."""
    n = R * M
    f = np.random.default_rng(M + R).uniform(-1, 1, (n, n, n))
    X = np.fft.rfft(f, axis=2).reshape(R, M, R, M, -1).transpose(0, 2, 1, 3, 4)  # [a, b, i', j', k]
    WR = np.exp(-2j * np.pi / R)
    full = np.fft.rfftn(f)
    ip = np.arange(M)[:, None]
    jp = np.arange(M)[None, :]
    for ci in range(R):
        for cj in range(R):
            Y = sum(WR ** (a * ci + b * cj) * X[a, b] for a in range(R) for b in range(R))
            Y = Y * np.exp(-2j * np.pi * (ci * ip + cj * jp) / n)[..., None]
            sub = np.fft.fft2(Y, axes=(0, 1))
            assert np.allclose(sub, full[ci::R, cj::R], rtol=0, atol=1e-10 * np.abs(full).max())
