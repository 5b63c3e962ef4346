"""CPU index model of the sm_100a kernels (tests/sim/engine_sim.py) driven by the
tile geometry compiled into libarena_fft.so (arena_pow2_kernel_geometry): every
Stockham plan / swizzled exchange used by the power-of-two path is replayed on
random data and checked against numpy, and the shared-memory exchange is
checked collision-free.  No GPU needed."""
import ctypes
import os
import sys

import numpy as np
import pytest

import paper_1408_6497_b200 as arena

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "sim"))
import engine_sim as sim  # noqa: E402

POW2 = [2, 4, 8, 16, 32, 64, 128, 256, 512, 1024, 2048]


def geometry(n, prec, with_x=False):
    out = (ctypes.c_int * 15)()
    arena.lib.arena_pow2_kernel_geometry.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    assert arena.lib.arena_pow2_kernel_geometry(n, prec, out) == 0
    keys = ("line", "E", "L", "threads", "smem")
    z, s, x = (dict(zip(keys, out[5 * i:5 * i + 5])) for i in range(3))
    return (z, s, x) if with_x else (z, s)


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("n", POW2)
def test_tile_geometry_is_launchable(n, prec):
    z, s, x = geometry(n, prec, with_x=True)
    vb = 2 * (prec // 8)
    assert x["line"] == n and x["smem"] >= x["line"] * x["L"] * vb
    for g in (z, s, x):
        assert g["L"] & (g["L"] - 1) == 0, g
        assert g["threads"] == g["L"] * (g["line"] // g["E"]) <= 1024, g
        assert g["smem"] <= 227 * 1024, g
    assert z["line"] == n // 2 and s["line"] == n
    assert (n * n) % z["L"] == 0  # z grid covers every row exactly
    assert z["smem"] >= (z["line"] * z["L"] + z["L"]) * vb
    assert s["smem"] >= s["line"] * s["L"] * vb


@pytest.mark.parametrize("prec", [64, 32])
@pytest.mark.parametrize("n", POW2)
def test_stockham_plan_replay(n, prec):
    z, s, x = geometry(n, prec, with_x=True)
    vb = 2 * (prec // 8)
    for g in (z, s, x):
        N, E, L = g["line"], g["E"], g["L"]
        if N < 2:
            continue
        Lm = min(L, 2)  # lines are independent; two suffice to exercise the interleaved layout
        for S in (-1, +1):
            err = sim.check_line(N, E, L, S, vbytes=vb, lines_checked=Lm)
            assert err < 1e-13, (N, E, L, S, err)


@pytest.mark.parametrize("n", [4, 8, 16])
def test_full_solve_model_vs_oracle(n):
    import oracle

    z, s = geometry(n, 64)
    f = np.random.default_rng(n).uniform(-1, 1, (n, n, n))
    u = sim.solve_model(f, z, s)
    assert np.linalg.norm(u - oracle.poisson_solve(f)) <= 1e-13 * np.linalg.norm(u)


@pytest.mark.parametrize("n", POW2)
def test_blocked_row_layout_is_a_bijection(n):
    """row_off (poisson_pow2.cuh): S rows grouped in j-blocks of JB; every (i, j)
    gets its own ncp-element row inside the n*n*ncp workspace."""
    jb = min(64, n)  # ARENA_JBLOCK
    ncp = (n // 2 + 1 + 7) // 8 * 8
    i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    rows = ((j // jb) * n + i) * jb + (j % jb)
    assert np.array_equal(np.sort(rows.ravel()), np.arange(n * n))
    assert rows.max() * ncp + ncp <= n * n * ncp


def _fused_decode(w, planes, c1, c2, lag):
    """Mirror of poisson_fused.cuh fused_decode."""
    A = lag * c1
    if w < A:
        return 1, w // c1, w % c1
    w -= A
    mid = (planes - lag) * (c1 + c2)
    if w < mid:
        r, s = lag + w // (c1 + c2), w % (c1 + c2)
        return (1, r, s) if s < c1 else (0, r - lag, s - c1)
    w -= mid
    return 0, planes - lag + w // c2, w % c2


@pytest.mark.parametrize("planes,c1,c2,lag", [(1024, 128, 129, 2), (1024, 129, 128, 2), (128, 128, 129, 4),
                                               (4, 3, 5, 4), (16, 7, 2, 1)])
def test_fused_schedule_is_a_deadlock_free_permutation(planes, c1, c2, lag):
    """Every (pass, plane, item) is dispatched exactly once, and every second-pass
    item of plane p comes after all first-pass items of plane p, so in-order
    dispatch never waits on an item that has not been handed out."""
    total = planes * (c1 + c2)
    seen = set()
    last_first = {}
    for w in range(total):
        first, p, s = _fused_decode(w, planes, c1, c2, lag)
        assert 0 <= p < planes and 0 <= s < (c1 if first else c2)
        key = (first, p, s)
        assert key not in seen
        seen.add(key)
        if first:
            last_first[p] = w
        else:
            assert last_first.get(p, -1) >= 0 and p in last_first
    assert len(seen) == total


# ---- FMA form of the twiddled radix-4 step (fft_engine.cuh: CTw / tw_rot / bfly4_tw) -------------
def _ctw(R, ex, S):
    """Restates CTw<R, EX, S>: exp(S 2 pi i ex / R) = rho * C * (1 + i T), rho in {1, S i}, |T| <= 1."""
    m = (ex * (64 // R)) % 64
    qt = (m + 7) // 16
    rm = m - 16 * qt
    assert -7 <= rm <= 8
    ang = 2 * np.pi * rm / 64
    return bool(qt & 1), (-1.0 if qt & 2 else 1.0) * np.cos(ang), S * np.tan(ang)


def _tw_rot(a, R, ex, S):
    rot, _, T = _ctw(R, ex, S)
    r = (a.real - T * a.imag) + 1j * (a.imag + T * a.real)
    return r * (S * 1j) if rot else r


def _dft_fma(x, S):
    """Restates Dft<R, S, FMA = true>::run on the last axis (R = 2, 4 direct, else one radix-4 DIT step)."""
    R = x.shape[-1]
    if R == 1:
        return x
    if R == 2:
        return np.stack([x[..., 0] + x[..., 1], x[..., 0] - x[..., 1]], -1)
    if R == 4:
        s02, d02 = x[..., 0] + x[..., 2], x[..., 0] - x[..., 2]
        s13, d13 = x[..., 1] + x[..., 3], (S * 1j) * (x[..., 1] - x[..., 3])
        return np.stack([s02 + s13, d02 + d13, s02 - s13, d02 - d13], -1)
    Q = R // 4
    a = [_dft_fma(x[..., n1::4], S) for n1 in range(4)]
    out = np.empty_like(x)
    for k1 in range(Q):
        c = [_ctw(R, n * k1, S)[1] for n in range(4)]
        p = [a[0][..., k1]] + [_tw_rot(a[n][..., k1], R, n * k1, S) for n in (1, 2, 3)]
        s02, d02 = p[0] + c[2] * p[2], p[0] - c[2] * p[2]
        r31 = c[3] / c[1]
        u, v = p[1] + r31 * p[3], p[1] - r31 * p[3]
        out[..., k1] = s02 + c[1] * u
        out[..., k1 + 2 * Q] = s02 - c[1] * u
        out[..., k1 + Q] = d02 + c[1] * (S * 1j) * v
        out[..., k1 + 3 * Q] = d02 - c[1] * (S * 1j) * v
    return out


@pytest.mark.parametrize("S", [-1, +1])
@pytest.mark.parametrize("R", [8, 16, 32, 64])
def test_fma_twiddle_form_is_the_twiddle(R, S):
    rng = np.random.default_rng(R + S)
    a = rng.standard_normal(16) + 1j * rng.standard_normal(16)
    for ex in range(0, 3 * (R // 4)):
        rot, C, T = _ctw(R, ex, S)
        assert abs(T) <= 1.0 + 1e-15 and abs(C) >= np.cos(np.pi / 4) - 1e-15
        w = np.exp(S * 2j * np.pi * ex / R)
        np.testing.assert_allclose(C * _tw_rot(a, R, ex, S), w * a, rtol=0, atol=2e-15 * np.abs(a).max())


@pytest.mark.parametrize("S", [-1, +1])
@pytest.mark.parametrize("R", [8, 16, 32, 64])
def test_fma_form_dft_matches_numpy(R, S):
    rng = np.random.default_rng(7 * R + S)
    x = rng.standard_normal((5, R)) + 1j * rng.standard_normal((5, R))
    ref = np.fft.fft(x, axis=-1) if S < 0 else np.fft.ifft(x, axis=-1) * R
    got = _dft_fma(x, S)
    assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 5e-16


# ---- Hermitian pairs in the z passes (poisson_pow2.cuh zfwd_rows / zinv_rows, ARENA_Z_PAIRS) ---------
@pytest.mark.parametrize("n", [4, 8, 32, 64, 1024])
def test_r2c_split_in_hermitian_pairs(n):
    """X[k] = S - U, X[M-k] = conj(S + U) with A = Z[k], B = conj(Z[M-k]), S = (A + B)/2,
    U = (i/2) W_n^k (A - B): one pair per k in [0, M/2) (k = 0 pairs with the Nyquist output),
    X[M/2] = conj(Z[M/2]) — against numpy's rfft."""
    rng = np.random.default_rng(n)
    f = rng.standard_normal(n)
    M = n // 2
    Z = np.fft.fft(f[0::2] + 1j * f[1::2])
    X = np.zeros(M + 1, dtype=complex)
    for k in range(M // 2):
        A, B = Z[k], np.conj(Z[(M - k) % M])
        S, U = 0.5 * (A + B), 0.5j * np.exp(-2j * np.pi * k / n) * (A - B)
        X[k] = S - U
        X[M - k] = np.conj(S + U)
    X[M // 2] = np.conj(Z[M // 2])
    ref = np.fft.rfft(f)
    assert np.linalg.norm(X - ref) <= 1e-14 * np.linalg.norm(ref)
    assert X[0].imag == 0 or abs(X[0].imag) < 1e-15 * abs(X[0])


@pytest.mark.parametrize("n", [4, 8, 32, 64, 1024])
def test_c2r_preprocessing_in_hermitian_pairs(n):
    """Z[k] = Ep + Op, Z[M-k] = conj(Ep - Op) with A = X[k], B = conj(X[M-k]), Ep = A + B,
    Op = i conj(W_n^k) (A - B); Z[M/2] = 2 conj(X[M/2]); the imaginary parts of X[0] and X[M]
    ignored (FFTW c2r) — the M-point backward FFT of Z is then n * irfft(X), interleaved."""
    rng = np.random.default_rng(n + 1)
    M = n // 2
    X = rng.standard_normal(M + 1) + 1j * rng.standard_normal(M + 1)  # junk imaginary parts at 0 and M too
    Z = np.zeros(M, dtype=complex)
    for k in range(M // 2):
        A, C = X[k], X[M - k]
        if k == 0:
            A, C = A.real + 0j, C.real + 0j
        B = np.conj(C)
        Ep, Op = A + B, 1j * np.exp(2j * np.pi * k / n) * (A - B)
        Z[k] = Ep + Op
        if k:
            Z[M - k] = np.conj(Ep - Op)
    Z[M // 2] = 2 * np.conj(X[M // 2])
    z = np.fft.ifft(Z) * M
    u = np.empty(n)
    u[0::2], u[1::2] = z.real, z.imag
    Xc = X.copy()
    Xc[0], Xc[M] = X[0].real, X[M].real
    ref = np.fft.irfft(Xc, n) * n
    assert np.linalg.norm(u - ref) <= 1e-13 * np.linalg.norm(ref)
