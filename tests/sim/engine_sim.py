"""Index model of csrc/fft_engine.cuh + csrc/poisson_pow2.cuh on the CPU.

Replays the CUDA kernels' thread / element / shared-memory index arithmetic
with numpy — one Python iteration per (thread, element) — so the Stockham
plan, the swizzled exchange and the r2c/c2r splits can be checked without a
GPU.  Mirrors: num_stages / stage_log2 / stage_ns / smem_idx /
stage_compute / stage_exchange (fft_engine.cuh), k_zfwd / k_ypass / k_xmid /
k_zinv (poisson_pow2.cuh).
"""
import numpy as np


def ilog2(x):
    return 0 if x <= 1 else 1 + ilog2(x // 2)


def num_stages(N, E):
    return 0 if N <= 1 else -(-ilog2(N) // ilog2(E))


def stage_log2(N, E, s):
    ns, b = num_stages(N, E), ilog2(N)
    return b // ns + (1 if s < b % ns else 0)


def stage_ns(N, E, s):
    return 1 if s == 0 else stage_ns(N, E, s - 1) << stage_log2(N, E, s - 1)


def smem_idx(pos, l, L, SW, vbytes):
    G = (128 // vbytes) // L
    if G <= 1 or SW == 0:
        return pos * L + l
    return (pos ^ ((pos >> SW) & (G - 1))) * L + l


def dft(a, S):
    R = len(a)
    r = np.arange(R)
    return np.exp(S * 2j * np.pi * np.outer(r, r) / R) @ a


def line_fft(v, N, E, L, S, tw, twmul, vbytes=16, lines=None):
    """v: [L, P, E] complex, thread (l, t) holding elements t + P*e.  Only lines in
    `lines` are computed (the exchange is still checked for the whole tile)."""
    P = N // E
    lines = range(L) if lines is None else lines
    nst = num_stages(N, E)
    SW = stage_log2(N, E, 0) if N > 1 else 0
    v = v.copy()
    for st in range(nst):
        R = 1 << stage_log2(N, E, st)
        NS = stage_ns(N, E, st)
        NB = E // R
        for l in lines:
            for t in range(P):
                for q in range(NB):
                    a = np.array([v[l, t, q + NB * r] for r in range(R)])
                    if NS > 1:
                        base = ((t + P * q) & (NS - 1)) * (N // (NS * R)) * twmul
                        for r in range(1, R):
                            w = tw[base * r]
                            a[r] *= w if S < 0 else np.conj(w)
                    a = dft(a, S)
                    for r in range(R):
                        v[l, t, q + NB * r] = a[r]
        if st + 1 < nst:
            sm = np.full(N * L, np.nan + 0j)
            for l in range(L):
                for t in range(P):
                    for q in range(NB):
                        b = t + P * q
                        dst = (b & ~(NS - 1)) * R + (b & (NS - 1))
                        for r in range(R):
                            idx = smem_idx(dst + r * NS, l, L, SW, vbytes)
                            assert 0 <= idx < N * L and np.isnan(sm[idx]), "shared-memory write collision"
                            sm[idx] = v[l, t, q + NB * r] if l in lines else 0.0
            for l in lines:
                for t in range(P):
                    for e in range(E):
                        v[l, t, e] = sm[smem_idx(t + P * e, l, L, SW, vbytes)]
    return v


def _to_threads(x, P, E):
    L = x.shape[0]
    v = np.empty((L, P, E), complex)
    for t in range(P):
        for e in range(E):
            v[:, t, e] = x[:, t + P * e]
    return v


def _from_threads(v, P, E):
    L = v.shape[0]
    x = np.empty((L, P * E), complex)
    for t in range(P):
        for e in range(E):
            x[:, t + P * e] = v[:, t, e]
    return x


def check_line(N, E, L, S, vbytes=16, lines_checked=None):
    tw = np.exp(-2j * np.pi * np.arange(N) / N)
    P = N // E
    rng = np.random.default_rng(N * 7 + L)
    x = rng.standard_normal((L, N)) + 1j * rng.standard_normal((L, N))
    lines = list(range(lines_checked if lines_checked else L))
    y = _from_threads(line_fft(_to_threads(x, P, E), N, E, L, S, tw, 1, vbytes, lines), P, E)
    ref = np.fft.fft(x, axis=1) if S < 0 else np.fft.ifft(x, axis=1) * N
    return float(np.abs(y[lines] - ref[lines]).max() / np.abs(ref[lines]).max())


def _lines_fft(x, g, S, tw, twmul):
    """Apply the engine to a batch of lines x [B, N] in tiles of g['L']."""
    N, E, L = g["line"], g["E"], g["L"]
    P = N // E
    out = np.empty_like(x)
    for b0 in range(0, x.shape[0], L):
        tile = np.zeros((L, N), complex)
        m = min(L, x.shape[0] - b0)
        tile[:m] = x[b0:b0 + m]
        out[b0:b0 + m] = _from_threads(line_fft(_to_threads(tile, P, E), N, E, L, S, tw, twmul), P, E)[:m]
    return out


def solve_model(f, zg, sg):
    """Whole power-of-two solve as the five kernels compute it."""
    n = f.shape[0]
    M, nc = n // 2, n // 2 + 1
    tw = np.exp(-2j * np.pi * np.arange(n) / n)
    # K1 zfwd
    z = f.reshape(n * n, M, 2)
    Z = _lines_fft(z[:, :, 0] + 1j * z[:, :, 1], zg, -1, tw, 2) if M > 1 else z[:, :, 0] + 1j * z[:, :, 1]
    S = np.zeros((n * n, nc), complex)
    for k in range(M):
        A, B = Z[:, k], np.conj(Z[:, (M - k) & (M - 1)])
        WD = tw[k] * (A - B)
        S[:, k] = 0.5 * (A.real + B.real + WD.imag) + 0.5j * (A.imag + B.imag - WD.real)
        if k == 0:
            S[:, M] = A.real - A.imag
    S = S.reshape(n, n, nc)
    # K2 y forward, K3 x fwd / scale / inv, K4 y inverse
    yl = lambda A, s: _lines_fft(A.transpose(0, 2, 1).reshape(-1, n), sg, s, tw, 1).reshape(n, nc, n).transpose(0, 2, 1)
    xl = lambda A, s: _lines_fft(A.transpose(1, 2, 0).reshape(-1, n), sg, s, tw, 1).reshape(n, nc, n).transpose(2, 0, 1)
    S = yl(S, -1)
    S = xl(S, -1)
    ki = np.array([i if i <= n // 2 else i - n for i in range(n)], float)
    k2 = ki[:, None, None] ** 2 + ki[None, :, None] ** 2 + np.arange(nc, dtype=float)[None, None, :] ** 2
    with np.errstate(divide="ignore"):
        S = S * np.where(k2 == 0, 0.0, (1.0 / (float(n) * n * n)) / (4.0 * np.pi * np.pi * k2))
    S = xl(S, +1)
    S = yl(S, +1)
    # K5 zinv
    S = S.reshape(n * n, nc)
    Zp = np.zeros((n * n, M), complex)
    for k in range(M):
        A = S[:, k].copy()
        Bs = (S[:, M] if k == 0 else S[:, M - k]).copy()
        if k == 0:
            A, Bs = A.real + 0j, Bs.real + 0j
        Ep, Op = A + np.conj(Bs), (A - np.conj(Bs)) * np.conj(tw[k])
        Zp[:, k] = Ep + 1j * Op
    z = _lines_fft(Zp, zg, +1, tw, 2) if M > 1 else Zp
    u = np.empty((n * n, n))
    u[:, 0::2], u[:, 1::2] = z.real, z.imag
    return u.reshape(n, n, n)
