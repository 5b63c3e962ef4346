"""CPU oracle for the spectral Poisson path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or
as the reported CPU baseline; the product (paper_1408_6497_b200/) never does.

Two CPU implementations, both built by oracle/Makefile:

* ``ref``  — oracle/_ref/libref_poisson.so: the reference's own
  /root/reference/proj/src/fft_solver.cpp:13-87, compiled unmodified over the
  FFTW3-API shim (oracle/fftw_shim) whose transforms are oracle/offt.c.
  Pinned by the reference's own tests (oracle/_ref/test_fft_ref runs
  test_fft.cpp T1-T12 unmodified against it).
* ``port`` — oracle/lib/libofft.so: offt_poisson_solve, the C restatement of
  fft_solver.cpp:51-87 (same op order), built from repo sources only.

Both run the 3D transforms with OpenMP over lines (``threads``); the
reference's FFTW itself is single-threaded (no fftw_init_threads,
proj/src/CMakeLists.txt:3,17), so threads=1 is the reference-faithful setting.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_PATH = os.path.join(HERE, "lib", "libofft.so")
REF_PATH = os.path.join(HERE, "_ref", "libref_poisson.so")
TEST_FFT_REF = os.path.join(HERE, "_ref", "test_fft_ref")
TEST_PROBLEMS_REF = os.path.join(HERE, "_ref", "test_problems_ref")
TEST_FFT_DROPIN = os.path.join(HERE, "_ref", "test_fft_dropin")

_vp = ctypes.c_void_p
_libs = {}


def _load(kind: str):
    if kind in _libs:
        return _libs[kind]
    path = REF_PATH if kind == "ref" else PORT_PATH
    if not os.path.exists(path):
        return None
    lib = ctypes.CDLL(path)
    pre = "ref_" if kind == "ref" else "offt_"
    getattr(lib, pre + "poisson_solve").argtypes = [ctypes.c_int, _vp, _vp]
    getattr(lib, pre + "dft3_forward").argtypes = [ctypes.c_int, _vp, _vp]
    getattr(lib, pre + "dft3_inverse").argtypes = [ctypes.c_int, _vp, _vp]
    getattr(lib, pre + "set_threads").argtypes = [ctypes.c_int]
    getattr(lib, pre + "get_threads").restype = ctypes.c_int
    _libs[kind] = lib
    return lib


def available(kind: str = "ref") -> bool:
    return _load(kind) is not None


def best_kind() -> str:
    """'ref' when the reference's own solver was built here (this container), else 'port'."""
    return "ref" if available("ref") else "port"


def _lib(kind: Optional[str]):
    kind = kind or best_kind()
    lib = _load(kind)
    if lib is None:
        raise FileNotFoundError(f"oracle '{kind}' not built (make -C oracle)")
    return lib, ("ref_" if kind == "ref" else "offt_")


def set_threads(n: int, kind: Optional[str] = None) -> None:
    lib, pre = _lib(kind)
    getattr(lib, pre + "set_threads")(int(n))


def get_threads(kind: Optional[str] = None) -> int:
    lib, pre = _lib(kind)
    return getattr(lib, pre + "get_threads")()


def poisson_solve(f: np.ndarray, kind: Optional[str] = None) -> np.ndarray:
    """fft_solver.cpp:51-87 on the CPU: fp64 n^3 in, n^3 out."""
    lib, pre = _lib(kind)
    f = np.ascontiguousarray(f, dtype=np.float64)
    n = f.shape[0]
    u = np.empty_like(f)
    rc = getattr(lib, pre + "poisson_solve")(n, _vp(f.ctypes.data), _vp(u.ctypes.data))
    if rc != 0:
        raise ValueError("oracle poisson_solve failed (n < 2?)")
    return u


def dft3_forward(g: np.ndarray, kind: Optional[str] = None) -> np.ndarray:
    lib, pre = _lib(kind)
    g = np.ascontiguousarray(g, dtype=np.float64)
    out = np.empty(g.shape, dtype=np.complex128)
    if getattr(lib, pre + "dft3_forward")(g.shape[0], _vp(g.ctypes.data), _vp(out.ctypes.data)) != 0:
        raise ValueError("oracle dft3_forward failed")
    return out


def dft3_inverse(spec: np.ndarray, n: int, kind: Optional[str] = None) -> np.ndarray:
    lib, pre = _lib(kind)
    spec = np.ascontiguousarray(spec, dtype=np.complex128).reshape(n, n, n)
    out = np.empty((n, n, n), dtype=np.float64)
    if getattr(lib, pre + "dft3_inverse")(n, _vp(spec.ctypes.data), _vp(out.ctypes.data)) != 0:
        raise ValueError("oracle dft3_inverse failed")
    return out


def pocketfft_poisson(f: np.ndarray, workers: Optional[int] = None) -> np.ndarray:
    """fft_solver.cpp:51-87 restated on scipy.fft (pocketfft, `workers` threads): the
    strongest CPU engine in this image ("B-all" of BASELINE.md §3) — rfftn, the
    symbol (k2 == 0 ? 0 : (1/n^3) / (4 pi^2 k2)) applied plane block by plane block
    on a thread pool (numpy releases the GIL), irfftn."""
    from concurrent.futures import ThreadPoolExecutor

    import scipy.fft as sf

    f = np.ascontiguousarray(f, dtype=np.float64)
    n = f.shape[0]
    w = workers or len(os.sched_getaffinity(0))
    F = sf.rfftn(f, workers=w)
    sfreq = np.where(np.arange(n) <= n // 2, np.arange(n), np.arange(n) - n).astype(np.float64)  # fft_solver.hpp:19
    kk2 = np.arange(n // 2 + 1, dtype=np.float64) ** 2
    kj2 = sfreq ** 2
    four_pi2 = 4.0 * np.pi * np.pi  # fft_solver.cpp:66
    scale = 1.0 / (float(n) ** 3)

    def block(i0, i1):
        for i in range(i0, i1):
            k2 = sfreq[i] ** 2 + kj2[:, None] + kk2[None, :]
            with np.errstate(divide="ignore"):
                s = np.where(k2 == 0.0, 0.0, scale / (four_pi2 * k2))  # fft_solver.cpp:76
            F[i] *= s

    step = max(1, n // (4 * w))
    with ThreadPoolExecutor(w) as ex:
        list(ex.map(lambda a: block(a, min(n, a + step)), range(0, n, step)))
    return sf.irfftn(F, s=f.shape, workers=w, overwrite_x=True, norm="forward")  # unnormalised, as FFTW c2r


def direct_dft3(g: np.ndarray) -> np.ndarray:
    """O(N^2) direct-summation DFT (the algorithm of oracle::direct_dft3,
    /root/reference/proj/tests/oracles.cpp:13-29), vectorised per output mode.
    For n <= 8 only."""
    n = g.shape[0]
    idx = np.arange(n)
    X = np.empty((n, n, n), dtype=np.complex128)
    I, J, K = np.meshgrid(idx, idx, idx, indexing="ij")
    for ki in range(n):
        for kj in range(n):
            for kk in range(n):
                ph = -2.0 * np.pi * (ki * I + kj * J + kk * K) / n
                X[ki, kj, kk] = np.sum(g * (np.cos(ph) + 1j * np.sin(ph)))
    return X
