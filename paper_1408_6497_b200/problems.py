"""Synthetic sources of BASELINE.json's configs.

No dataset is involved: the paper uses manufactured solutions
(PAPER.md:247-253).  Seeded with std::mt19937_64 — the reference's RNG
(test_fft.cpp:15) — implemented here bit-exactly, with explicit transforms
(uniform = (x >> 11) * 2^-53, normal by Box-Muller) because libstdc++'s
distributions are implementation-defined.  A C++ caller seeding
std::mt19937_64 identically reproduces every draw.

Configs (BASELINE.json "configs"):
  C1  n=64    u = sin(2 pi x) sin(2 pi y) sin(2 pi z), f = 12 pi^2 u
              (= exact_f(TestCase::oscillatory(1)), problems.cpp:65-67,75-77)
  C2  n=256   32 Fourier modes, k uniform in [-8,8]^3 \\ {0}, a ~ N(0,1) + i N(0,1)
  C3  n=512   periodised Gaussian, alpha = 1e4, c ~ U[0,1)^3, 27 images
  C4  n=1024  64 modes, k in [-32,32]^3 (headline bench config)
  C5  n=2048  periodised Gaussian, alpha = 1e5 (multi-GPU pencil); C4 in fp32
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

_MASK64 = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (Matsumoto & Nishimura 64-bit Mersenne Twister), default seeding."""

    def __init__(self, seed: int = 5489):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK64
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK64
        self.idx = 312

    def _twist(self) -> None:
        mt = self.mt
        upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
        for i in range(312):
            x = (mt[i] & upper) | (mt[(i + 1) % 312] & lower)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def next_u64(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK64

    def uniform(self) -> float:
        """[0, 1) with 53 random bits."""
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)

    def randint(self, lo: int, hi: int) -> int:
        """Uniform integer in [lo, hi] (rejection-free for small ranges via floor(u*span))."""
        span = hi - lo + 1
        return lo + min(int(self.uniform() * span), span - 1)

    def normal_pair(self) -> Tuple[float, float]:
        """Box-Muller: two independent N(0,1)."""
        u1 = self.uniform()
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        return r * math.cos(2.0 * math.pi * u2), r * math.sin(2.0 * math.pi * u2)


@dataclass
class ModeSource:
    """f = sum_m Re(a_m e^{2 pi i k_m.x}); analytic u = sum_m Re(a_m / (4 pi^2 |k_m|^2) e^{...})."""

    n: int
    k: np.ndarray  # (M, 3) int
    a: np.ndarray  # (M,) complex128
    kind: str = "modes"

    def f_coef(self) -> np.ndarray:
        return self.a

    def u_coef(self) -> np.ndarray:
        k2 = (self.k.astype(np.float64) ** 2).sum(axis=1)
        return self.a / (4.0 * math.pi * math.pi * k2)


@dataclass
class GaussianSource:
    """u = sum_{m in {-1,0,1}^3} exp(-alpha |x - c - m|^2), f = -Lap u."""

    n: int
    alpha: float
    center: Tuple[float, float, float]
    kind: str = "gaussian"


def oscillatory_modes(n: int, kw: int = 1) -> ModeSource:
    """exact_f of TestCase::oscillatory(kw) (problems.cpp:65-67,75-77) as 8 modes:
    sin a sin b sin c = (i/8) sum_{s in {+-1}^3} s1 s2 s3 e^{i(s1 a + s2 b + s3 c)}; f = 3 w^2 u."""
    ks, cs = [], []
    w2 = (2.0 * math.pi * kw) ** 2
    for s1 in (1, -1):
        for s2 in (1, -1):
            for s3 in (1, -1):
                ks.append((s1 * kw, s2 * kw, s3 * kw))
                cs.append(1j / 8.0 * s1 * s2 * s3 * 3.0 * w2)
    return ModeSource(n, np.array(ks, dtype=np.int64), np.array(cs, dtype=np.complex128))


def random_modes(n: int, nmodes: int, kmax: int, seed: int) -> ModeSource:
    rng = MT19937_64(seed)
    ks, cs = [], []
    while len(ks) < nmodes:
        k = (rng.randint(-kmax, kmax), rng.randint(-kmax, kmax), rng.randint(-kmax, kmax))
        if k == (0, 0, 0):
            continue  # rejection: k = 0 excluded
        re, im = rng.normal_pair()
        ks.append(k)
        cs.append(complex(re, im))
    return ModeSource(n, np.array(ks, dtype=np.int64), np.array(cs, dtype=np.complex128))


def gaussian(n: int, alpha: float, seed: int) -> GaussianSource:
    rng = MT19937_64(seed)
    c = (rng.uniform(), rng.uniform(), rng.uniform())
    return GaussianSource(n, alpha, c)


# BASELINE.json configs, seeds 1..5 ("fix and record one per config").
def config(idx: int, n: Optional[int] = None):
    if idx == 1:
        return oscillatory_modes(n or 64, 1)
    if idx == 2:
        return random_modes(n or 256, 32, 8, seed=2)
    if idx == 3:
        return gaussian(n or 512, 1.0e4, seed=3)
    if idx == 4:
        return random_modes(n or 1024, 64, 32, seed=4)
    if idx == 5:
        return gaussian(n or 2048, 1.0e5, seed=5)
    raise ValueError(f"unknown config {idx}")


CONFIG_TEXT = {
    1: "N=64^3 fp64 single mode sin(2pi x)sin(2pi y)sin(2pi z), f=12pi^2 u",
    2: "N=256^3 fp64, 32 random Fourier modes k in [-8,8]^3, a~N(0,1)+iN(0,1), seed 2",
    3: "N=512^3 fp64 periodised Gaussian alpha=1e4, c~U[0,1)^3, seed 3",
    4: "N=1024^3 fp64, 64 random Fourier modes k in [-32,32]^3, a~N(0,1)+iN(0,1), seed 4",
    5: "N=2048^3 fp64 periodised Gaussian alpha=1e5, seed 5",
}


def fill_device(src, which: str, out, precision: int = 64, stream: int = 0, i0: int = 0, ni=None, j0: int = 0,
                nj=None) -> None:
    """Write f (which='f') or the analytic u (which='u') of `src` into device buffer `out`
    (block i0..i0+ni-1 x j0..j0+nj-1 x all k of the n^3 field; default all)."""
    from . import source_gaussian, source_modes

    if isinstance(src, ModeSource):
        coef = src.f_coef() if which == "f" else src.u_coef()
        source_modes(src.n, src.k, coef, out, precision, stream, i0, ni, j0, nj)
    else:
        source_gaussian(src.n, src.alpha, src.center, 1 if which == "f" else 0, out, precision, stream, i0, ni, j0, nj)


def host_field(src, which: str = "f", workers: Optional[int] = None) -> np.ndarray:
    """f (or the analytic u) of `src` on the host at any n, without the GPU.

    Mode sources are band-limited, so the field is the c2r transform of a sparse
    half spectrum (scipy pocketfft, `workers` threads): with N = n^3 and kz taken
    mod n, a mode with 0 < kz < n/2 puts a N/2 at (kx, ky, kz), n/2 < kz puts
    conj(a) N/2 at -k, and the self-conjugate planes kz = 0, n/2 take a N, whose
    imaginary part the c2r's last axis drops — Re(a e^{2 pi i k.x}) in every case.  Other sources: eval_host (small n)."""
    if not isinstance(src, ModeSource):
        return eval_host(src, which)
    import os

    import scipy.fft as sf

    n = src.n
    N = float(n) ** 3
    nc = n // 2 + 1
    coef = src.f_coef() if which == "f" else src.u_coef()
    H = np.zeros((n, n, nc), dtype=np.complex128)
    for (kx, ky, kz), c in zip(src.k, coef):
        kz = int(kz) % n  # the grid aliases k to k mod n
        if kz == 0 or 2 * kz == n:  # self-conjugate planes (DC, Nyquist): c2r keeps Re
            H[kx % n, ky % n, kz] += c * N
        elif kz < nc:
            H[kx % n, ky % n, kz] += 0.5 * c * N
        else:
            H[-kx % n, -ky % n, n - kz] += 0.5 * np.conj(c) * N
    w = workers or len(os.sched_getaffinity(0))
    out = sf.irfftn(H, s=(n, n, n), workers=w, overwrite_x=True)
    del H
    return np.ascontiguousarray(out)


def eval_host(src, which: str) -> np.ndarray:
    """Host (numpy) evaluation of f or analytic u — for small n only (tests, oracle inputs)."""
    n = src.n
    x = np.arange(n, dtype=np.float64) / n
    if isinstance(src, ModeSource):
        coef = src.f_coef() if which == "f" else src.u_coef()
        idx = np.arange(n, dtype=np.int64)
        out = np.zeros((n, n, n))
        for (kx, ky, kz), c in zip(src.k, coef):
            # exact phase reduction mod n, as on the device
            p = (kx * idx[:, None, None] + ky * idx[None, :, None] + kz * idx[None, None, :]) % n
            th = 2.0 * math.pi * p / n
            out += c.real * np.cos(th) - c.imag * np.sin(th)
        return out
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    out = np.zeros((n, n, n))
    a = src.alpha
    cx, cy, cz = src.center
    for i in (-1, 0, 1):
        for j in (-1, 0, 1):
            for k in (-1, 0, 1):
                r2 = (X - cx - i) ** 2 + (Y - cy - j) ** 2 + (Z - cz - k) ** 2
                g = np.exp(-a * r2)
                out += g if which == "u" else (6.0 * a - 4.0 * a * a * r2) * g
    return out
