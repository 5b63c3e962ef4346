"""B200-native spectral Poisson solver — Python host mirror of the reference API.

The product is the C ABI in ``include/arena_fft.h`` (``lib/libarena_fft.so``,
sm_100a CUDA kernels) and the C++ drop-in ``include/arena/fft_solver.hpp``
(``lib/libarena_core.so``).  This module is a thin ctypes binding used by the
tests and by ``bench.py``; it mirrors the reference's function names and
error behaviour (/root/reference/proj/include/arena/fft_solver.hpp:11-23):

    poisson_spectral_solve(f)   fft_solver.cpp:51-87
    dft3_forward(g)             fft_solver.cpp:13-29
    dft3_inverse(spec, n)       fft_solver.cpp:31-49
    signed_freq(k, n)           fft_solver.hpp:19

n < 2 raises ValueError (std::invalid_argument in the reference, grid.hpp:18).
There is no CPU path: if the shared library is missing this import fails, and
without an sm_100a device every solve raises RuntimeError.
"""
from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.environ.get("ARENA_FFT_LIB_DIR", os.path.join(_HERE, "lib"))  # override: kernel-variant experiments
LIB_PATH = os.path.join(LIB_DIR, "libarena_fft.so")
CORE_PATH = os.path.join(LIB_DIR, "libarena_core.so")
REPO_ROOT = os.path.dirname(_HERE)
HEADER_PATH = os.path.join(REPO_ROOT, "include", "arena_fft.h")

ARENA_OK, ARENA_EINVAL, ARENA_ENOMEM, ARENA_ECUDA, ARENA_ENCCL, ARENA_EUNSUPPORTED = range(6)
PATH_POW2, PATH_GENERIC = 0, 1
_STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "EUNSUPPORTED"}

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or `make -C paper_1408_6497_b200`). There is no CPU fallback."
    )


_vp = ctypes.c_void_p
_i = ctypes.c_int
_sig = {
    "arena_fft_plan_create": (_i, [ctypes.POINTER(_vp), _i, _i, _i]),
    "arena_fft_plan_destroy": (None, [_vp]),
    "arena_fft_plan_info": (_i, [_vp, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(_i),
                                  ctypes.POINTER(_i), ctypes.POINTER(ctypes.c_size_t)]),
    "arena_poisson_solve_device": (_i, [_vp, _vp, _vp, _vp]),
    "arena_poisson_solve_host": (_i, [_vp, _vp, _vp]),
    "arena_poisson_solve_host_batch": (_i, [_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "arena_dft3_forward_host": (_i, [_vp, _vp, _vp]),
    "arena_dft3_forward_device": (_i, [_vp, _vp, _vp, _vp]),
    "arena_dft3_inverse_host": (_i, [_vp, _vp, _vp]),
    "arena_dft3_inverse_device": (_i, [_vp, _vp, _vp, _vp]),
    "arena_fft_set_stage_timing": (_i, [_vp, _i]),
    "arena_fft_stage_times": (_i, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_char_p), _i,
                                   ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "arena_poisson_launches_per_solve": (_i, [_vp]),
    "arena_source_modes": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp]),
    "arena_source_gaussian": (_i, [_i, _i, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                   _i, _vp, _vp]),
    "arena_source_modes_slab": (_i, [_i, _i, _i, _vp, _vp, _i, _i, _vp, _vp]),
    "arena_source_gaussian_slab": (_i, [_i, _i, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                        _i, _i, _i, _vp, _vp]),
    "arena_source_modes_block": (_i, [_i, _i, _i, _vp, _vp, _i, _i, _i, _i, _vp, _vp]),
    "arena_source_gaussian_block": (_i, [_i, _i, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                         _i, _i, _i, _i, _i, _vp, _vp]),
    "arena_nccl_unique_id_bytes": (_i, []),
    "arena_nccl_unique_id": (_i, [_vp, _i]),
    "arena_slab_create": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _i, _i, _vp]),
    "arena_slab_create_loopback": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _i]),
    "arena_slab_destroy": (None, [_vp]),
    "arena_slab_info": (_i, [_vp, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(ctypes.c_size_t),
                             ctypes.POINTER(ctypes.c_size_t)]),
    "arena_slab_solve_device": (_i, [_vp, _vp, _vp, _vp]),
    "arena_slab_create_peer": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _i, _i]),
    "arena_slab_peer_handle_bytes": (_i, []),
    "arena_slab_peer_export": (_i, [_vp, _vp, _i]),
    "arena_slab_peer_attach": (_i, [_vp, _vp, _i]),
    "arena_slab_set_exchange": (_i, [_vp, _i]),
    "arena_slab_solve_phase": (_i, [_vp, _i, _vp, _vp, _vp]),
    "arena_slab_barrier_status": (_i, [_vp]),
    "arena_slab_set_stage_timing": (_i, [_vp, _i]),
    "arena_slab_set_chunking": (_i, [_vp, _i, _i]),
    "arena_slab_get_chunking": (_i, [_vp, ctypes.POINTER(_i), ctypes.POINTER(_i)]),
    "arena_slab_exchange_pieces": (_i, [_i, _i, _i, _i, _i, ctypes.POINTER(ctypes.c_size_t),
                                        ctypes.POINTER(ctypes.c_size_t), _i]),
    "arena_slab_wait": (_i, [_vp, _vp, ctypes.c_double]),
    "arena_slab_stage_times": (_i, [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i)]),
    "arena_peer_barrier_selftest": (_i, [_i, _i, _i, ctypes.POINTER(_i)]),
    "arena_pencil_create_peer": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _i, _i, _i]),
    "arena_pencil_peer_handle_bytes": (_i, []),
    "arena_pencil_peer_export": (_i, [_vp, _vp, _i]),
    "arena_pencil_peer_attach": (_i, [_vp, _vp, _i]),
    "arena_pencil_set_exchange": (_i, [_vp, _i]),
    "arena_pencil_solve_phase": (_i, [_vp, _i, _vp, _vp, _vp]),
    "arena_pencil_barrier_status": (_i, [_vp]),
    "arena_pencil_set_layout": (_i, [_vp, _i]),
    "arena_field_stats": (_i, [ctypes.c_size_t, _i, _vp, ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_double)]),
    "arena_field_compare": (_i, [ctypes.c_size_t, _i, _vp, _vp, ctypes.POINTER(ctypes.c_double),
                                 ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "arena_pow2_kernel_geometry": (_i, [_i, _i, ctypes.POINTER(_i)]),
    "arena_pencil_create": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _i, _i, _i, _vp]),
    "arena_pencil_create_loopback": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _i, _i]),
    "arena_pencil_destroy": (None, [_vp]),
    "arena_pencil_launches_per_solve": (_i, [_vp]),
    "arena_slab_launches_per_solve": (_i, [_vp]),
    "arena_pencil_info": (_i, [_vp, ctypes.POINTER(_i), ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]),
    "arena_pencil_solve_device": (_i, [_vp, _vp, _vp, _vp]),
    "arena_interpolant_eval": (_i, [_i, _i, _vp, _vp, _i, _vp, _vp]),
    "arena_last_error": (ctypes.c_char_p, []),
    "arena_fft_abi_version": (_i, []),
    "arena_current_device": (_i, []),
    "arena_mgpu_create": (_i, [ctypes.POINTER(_vp), _i, _i, _i, ctypes.POINTER(_i)]),
    "arena_mgpu_destroy": (None, [_vp]),
    "arena_mgpu_info": (_i, [_vp, ctypes.POINTER(_i), ctypes.POINTER(_i), ctypes.POINTER(ctypes.c_size_t)]),
    "arena_mgpu_solve_device": (_i, [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.POINTER(_vp)]),
    "arena_mgpu_solve_host": (_i, [_vp, _vp, _vp]),
}
_lib = None
_lib_lock = threading.Lock()


def _load_lib() -> ctypes.CDLL:
    """Load libarena_fft.so on first use (not at import: importing the package —
    e.g. problems.py for a CPU-only reference run — must not map the CUDA library)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            h = ctypes.CDLL(LIB_PATH)
            for _name, (_res, _args) in _sig.items():
                _fn = getattr(h, _name)
                _fn.restype = _res
                _fn.argtypes = _args
            _lib = h
    return _lib


class _LazyLib:
    """Attribute access loads the library (``arena.lib.arena_...`` as before)."""

    def __getattr__(self, name):
        return getattr(_load_lib(), name)


lib = _LazyLib()


class ArenaError(RuntimeError):
    def __init__(self, status: int, what: str):
        msg = lib.arena_last_error().decode(errors="replace")
        super().__init__(f"{what}: {_STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def _check(status: int, what: str) -> None:
    if status == ARENA_OK:
        return
    if status == ARENA_EINVAL:
        raise ValueError(f"{what}: {lib.arena_last_error().decode(errors='replace')}")
    if status == ARENA_ENOMEM:
        raise MemoryError(f"{what}: {lib.arena_last_error().decode(errors='replace')}")
    raise ArenaError(status, what)


def signed_freq(k: int, n: int) -> int:
    """fft_solver.hpp:19 — signed frequency in (-n/2, n/2]."""
    return k if k <= n // 2 else k - n


def _ptr(x) -> int:
    """Raw pointer of a numpy array or torch tensor."""
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _check_buffer(x, numel: int, itemsize: int, what: str, device: Optional[int] = None) -> None:
    """Validate a buffer before its raw pointer crosses the C ABI: contiguous,
    `numel` elements of `itemsize` bytes, and (device is not None) a CUDA tensor
    on that device — or (device is None) host memory.  The kernels and copies
    trust the sizes, so a short or mistyped buffer would be read past its end."""
    if isinstance(x, np.ndarray):
        if device is not None:
            raise TypeError(f"{what}: expected a CUDA tensor on device {device}, got a numpy array")
        ok_c, n_el, isz = x.flags.c_contiguous, x.size, x.itemsize
    else:
        is_cuda = bool(getattr(x, "is_cuda", False))
        if device is not None and (not is_cuda or x.device.index != device):
            raise TypeError(f"{what}: expected a CUDA tensor on device {device}, got {x.device}")
        if device is None and is_cuda:
            raise TypeError(f"{what}: expected host memory, got a CUDA tensor")
        ok_c, n_el, isz = x.is_contiguous(), x.numel(), x.element_size()
    if not ok_c:
        raise ValueError(f"{what}: buffer must be contiguous")
    if isz != itemsize:
        raise TypeError(f"{what}: element size {isz} B, the plan needs {itemsize} B")
    if n_el != numel:
        raise ValueError(f"{what}: {n_el} elements, the plan needs {numel}")


class Plan:
    """Owns an ``arena_fft_plan`` (Setup: twiddles + device half-spectrum workspace)."""

    def __init__(self, n: int, precision: int = 64, device: int = -1):
        self._p = _vp()
        _check(lib.arena_fft_plan_create(ctypes.byref(self._p), int(n), int(precision), int(device)),
               "arena_fft_plan_create")
        self.n = int(n)
        self.precision = int(precision)
        self.dtype = np.float64 if precision == 64 else np.float32
        self.lock = threading.Lock()
        nn, pb, path, dev, ws = _i(), _i(), _i(), _i(), ctypes.c_size_t()
        _check(lib.arena_fft_plan_info(self._p, ctypes.byref(nn), ctypes.byref(pb), ctypes.byref(path),
                                       ctypes.byref(dev), ctypes.byref(ws)), "arena_fft_plan_info")
        self.path, self.device, self.workspace_bytes = path.value, dev.value, ws.value

    @property
    def handle(self) -> _vp:
        return self._p

    def close(self) -> None:
        if getattr(self, "_p", None) and self._p.value:
            lib.arena_fft_plan_destroy(self._p)
            self._p = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches_per_solve(self) -> int:
        return lib.arena_poisson_launches_per_solve(self._p)

    # ---- device-resident solve (the timed hot path)
    def solve_device(self, f, u, stream: Optional[int] = None) -> None:
        """Enqueue u = solve(f) on `stream` (cudaStream_t as int; None = torch's current stream).
        f, u: CUDA tensors of n^3 values of the plan's precision (may be the same tensor)."""
        n3, isz = self.n ** 3, self.precision // 8
        _check_buffer(f, n3, isz, "solve_device f", self.device)
        _check_buffer(u, n3, isz, "solve_device u", self.device)
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(f.device).cuda_stream
        _check(lib.arena_poisson_solve_device(self._p, _vp(_ptr(f)), _vp(_ptr(u)), _vp(stream)),
               "arena_poisson_solve_device")

    # ---- host boundary (the drop-in path)
    def solve_host(self, f, u) -> None:
        n3, isz = self.n ** 3, self.precision // 8
        _check_buffer(f, n3, isz, "solve_host f")
        _check_buffer(u, n3, isz, "solve_host u")
        _check(lib.arena_poisson_solve_host(self._p, _vp(_ptr(f)), _vp(_ptr(u))), "arena_poisson_solve_host")

    def solve_host_batch(self, fs, us) -> None:
        """Solve fields fs[s] -> us[s] (host arrays / pinned tensors) with copy/compute overlap."""
        if len(fs) != len(us):
            raise ValueError("fs and us must have the same length")
        n3, isz = self.n ** 3, self.precision // 8
        for x in list(fs) + list(us):
            _check_buffer(x, n3, isz, "solve_host_batch field")
        fa = (_vp * len(fs))(*[_ptr(x) for x in fs])
        ua = (_vp * len(us))(*[_ptr(x) for x in us])
        _check(lib.arena_poisson_solve_host_batch(self._p, len(fs), fa, ua), "arena_poisson_solve_host_batch")

    def dft3_forward_host(self, g: np.ndarray) -> np.ndarray:
        _check_buffer(g, self.n ** 3, self.precision // 8, "dft3_forward g")
        out = np.empty(g.shape, dtype=np.complex128 if self.precision == 64 else np.complex64)
        _check(lib.arena_dft3_forward_host(self._p, _vp(g.ctypes.data), _vp(out.ctypes.data)), "dft3_forward")
        return out

    def dft3_inverse_host(self, spec: np.ndarray) -> np.ndarray:
        _check_buffer(spec, self.n ** 3, self.precision // 4, "dft3_inverse spec")
        out = np.empty(spec.shape, dtype=self.dtype)
        _check(lib.arena_dft3_inverse_host(self._p, _vp(spec.ctypes.data), _vp(out.ctypes.data)), "dft3_inverse")
        return out

    # ---- measurement hooks
    def set_stage_timing(self, enable: bool) -> None:
        _check(lib.arena_fft_set_stage_timing(self._p, int(bool(enable))), "arena_fft_set_stage_timing")

    def stage_times(self):
        """-> (dict name -> total ms over recorded solves, number of solves)."""
        ms = (ctypes.c_double * 16)()
        names = (ctypes.c_char_p * 16)()
        ns, nsol = _i(), _i()
        _check(lib.arena_fft_stage_times(self._p, ms, names, 16, ctypes.byref(ns), ctypes.byref(nsol)),
               "arena_fft_stage_times")
        return {names[i].decode(): ms[i] for i in range(ns.value)}, nsol.value


XCHG_COPY, XCHG_PEER = 0, 1


def _resolve_device(device: int) -> int:
    return int(device) if device >= 0 else lib.arena_current_device()


class _Decomposition:
    """Peer-exchange / phase methods shared by Slab and Pencil (prefix arena_slab_ / arena_pencil_)."""

    _pfx = ""

    def _fn(self, name):
        return getattr(lib, f"arena_{self._pfx}_{name}")

    def _check_fields(self, f, u, what):
        _check_buffer(f, self.field_numel, self.precision // 8, f"{what} f", self.device)
        _check_buffer(u, self.field_numel, self.precision // 8, f"{what} u", self.device)

    def solve_device(self, f, u, stream: Optional[int] = None) -> None:
        self._check_fields(f, u, "solve_device")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(f.device).cuda_stream
        _check(self._fn("solve_device")(self._s, _vp(_ptr(f)), _vp(_ptr(u)), _vp(stream)),
               f"arena_{self._pfx}_solve_device")

    def solve_phase(self, phase: int, f, u, stream: Optional[int] = None) -> None:
        """One phase of a solve (slab 0-2, pencil 0-4); peer mode: synchronise the ranks in between."""
        self._check_fields(f, u, "solve_phase")
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(f.device).cuda_stream
        _check(self._fn("solve_phase")(self._s, int(phase), _vp(_ptr(f)), _vp(_ptr(u)), _vp(stream)),
               f"arena_{self._pfx}_solve_phase")

    def peer_handles(self) -> bytes:
        nb = self._fn("peer_handle_bytes")()
        buf = ctypes.create_string_buffer(nb)
        _check(self._fn("peer_export")(self._s, buf, nb), f"arena_{self._pfx}_peer_export")
        return buf.raw

    def peer_attach(self, all_handles: bytes) -> None:
        buf = ctypes.create_string_buffer(bytes(all_handles), len(all_handles))
        _check(self._fn("peer_attach")(self._s, buf, len(all_handles)), f"arena_{self._pfx}_peer_attach")

    def set_exchange(self, mode: int) -> None:
        _check(self._fn("set_exchange")(self._s, int(mode)), f"arena_{self._pfx}_set_exchange")

    def barrier_status(self) -> None:
        _check(self._fn("barrier_status")(self._s), f"arena_{self._pfx}_barrier_status")

    @property
    def launches_per_solve(self) -> int:
        return self._fn("launches_per_solve")(self._s)

    def close(self) -> None:
        if getattr(self, "_s", None) and self._s.value:
            self._fn("destroy")(self._s)
            self._s = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Slab(_Decomposition):
    """Slab decomposition over P ranks (include/arena_fft.h, arena_slab_*).

    Slab(n, P, rank=r, nccl_id=bytes) — one rank of a multi-GPU solve (NCCL all-to-alls);
    Slab(n, P, rank=r, peer=True)     — one rank, exchange fused into K2 / K3 as stores
                                        into the peers' workspaces (CUDA IPC); call
                                        peer_attach(all ranks' peer_handles()) first;
    Slab(n, P, loopback=True)         — P virtual ranks on one device (testing);
                                        set_exchange(XCHG_PEER) for the peer-store kernels.
    """

    _pfx = "slab"

    def __init__(self, n: int, nranks: int, rank: int = 0, nccl_id: Optional[bytes] = None,
                 precision: int = 64, device: int = -1, loopback: bool = False, peer: bool = False):
        self._s = _vp()
        if loopback:
            _check(lib.arena_slab_create_loopback(ctypes.byref(self._s), int(n), int(precision), int(device),
                                                  int(nranks)), "arena_slab_create_loopback")
        elif peer:
            _check(lib.arena_slab_create_peer(ctypes.byref(self._s), int(n), int(precision), int(device),
                                              int(nranks), int(rank)), "arena_slab_create_peer")
        else:
            if nccl_id is None:
                raise ValueError("nccl_id required (see nccl_unique_id())")
            buf = ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
            _check(lib.arena_slab_create(ctypes.byref(self._s), int(n), int(precision), int(device), int(nranks),
                                         int(rank), buf), "arena_slab_create")
        self.n, self.nranks, self.rank, self.loopback = int(n), int(nranks), int(rank), loopback
        ni, nj, cb, wb = _i(), _i(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib.arena_slab_info(self._s, ctypes.byref(ni), ctypes.byref(nj), ctypes.byref(cb), ctypes.byref(wb)),
               "arena_slab_info")
        self.ni, self.nj, self.chunk_bytes, self.workspace_bytes = ni.value, nj.value, cb.value, wb.value
        self.precision = int(precision)
        self.device = _resolve_device(device)
        self.field_numel = self.n ** 3 if loopback else (self.n // self.nranks) * self.n * self.n

    STAGES = ("k1k2", "xchg1", "k3", "xchg2", "k4k5")

    def set_chunking(self, fwd: int, bwd: int) -> None:
        """Sub-steps of the COPY exchange per direction (1, 1: whole chunks after whole passes)."""
        _check(lib.arena_slab_set_chunking(self._s, int(fwd), int(bwd)), "arena_slab_set_chunking")

    @property
    def chunking(self):
        f, b = _i(), _i()
        _check(lib.arena_slab_get_chunking(self._s, ctypes.byref(f), ctypes.byref(b)), "arena_slab_get_chunking")
        return f.value, b.value

    def wait(self, stream: Optional[int] = None, timeout_s: float = 60.0) -> None:
        """Block until the solves enqueued on `stream` finish, with NCCL error / hang detection
        (the communicator is aborted and ArenaError raised on an async error or timeout)."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.device).cuda_stream
        _check(lib.arena_slab_wait(self._s, _vp(stream), float(timeout_s)), "arena_slab_wait")

    def set_stage_timing(self, enable: bool) -> None:
        _check(lib.arena_slab_set_stage_timing(self._s, int(bool(enable))), "arena_slab_set_stage_timing")

    def stage_times(self):
        """-> (dict stage -> total ms over the timed solves, number of solves)."""
        ms = (ctypes.c_double * 5)()
        ns = _i()
        _check(lib.arena_slab_stage_times(self._s, ms, ctypes.byref(ns)), "arena_slab_stage_times")
        return {k: ms[i] for i, k in enumerate(self.STAGES)}, ns.value


class Pencil(_Decomposition):
    """Pencil decomposition over a Pr x Pc process grid (include/arena_fft.h, arena_pencil_*).

    Pencil(n, Pr, Pc, rank=r, nccl_id=bytes) — one rank (its block (n/Pr) x (n/Pc) x n), NCCL;
    Pencil(n, Pr, Pc, rank=r, peer=True)    — one rank, exchanges fused into K1-K4 as stores
                                              into the peers' buffers (peer_attach first);
    Pencil(n, Pr, Pc, loopback=True)        — all ranks on one device (full field in/out).
    folded=True: the folded distribution (include/arena_fft.h ARENA_PENCIL_FOLDED; a rank's
    block is fold_blocks(n, Pr, Pc, r, c)), quadrant z passes and n/2-point strided passes.
    """

    _pfx = "pencil"

    def __init__(self, n: int, pr: int, pc: int, rank: int = 0, nccl_id: Optional[bytes] = None,
                 precision: int = 64, device: int = -1, loopback: bool = False, peer: bool = False,
                 folded: bool = False):
        self._s = _vp()
        if loopback:
            _check(lib.arena_pencil_create_loopback(ctypes.byref(self._s), int(n), int(precision), int(device),
                                                    int(pr), int(pc)), "arena_pencil_create_loopback")
        elif peer:
            _check(lib.arena_pencil_create_peer(ctypes.byref(self._s), int(n), int(precision), int(device),
                                                int(pr), int(pc), int(rank)), "arena_pencil_create_peer")
        else:
            if nccl_id is None:
                raise ValueError("nccl_id required (see nccl_unique_id())")
            buf = ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
            _check(lib.arena_pencil_create(ctypes.byref(self._s), int(n), int(precision), int(device), int(pr),
                                           int(pc), int(rank), buf), "arena_pencil_create")
        self.n, self.pr, self.pc, self.rank = int(n), int(pr), int(pc), int(rank)
        kq, bb, kb = _i(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib.arena_pencil_info(self._s, ctypes.byref(kq), ctypes.byref(bb), ctypes.byref(kb)), "arena_pencil_info")
        self.kq, self.buffer_bytes, self.block_bytes = kq.value, bb.value, kb.value
        self.precision = int(precision)
        self.device = _resolve_device(device)
        self.field_numel = self.n ** 3 if loopback else (self.n // self.pr) * (self.n // self.pc) * self.n
        self.folded = bool(folded)
        if folded:
            _check(lib.arena_pencil_set_layout(self._s, 1), "arena_pencil_set_layout")


def fold_blocks(n: int, pr: int, pc: int, r: int, c: int):
    """Sub-blocks of rank (r, c)'s folded pencil block: [(i0, j0, li0, lj0, ni, nj)] — global
    plane / line offsets of the n^3 field, local offsets in the (n/Pr) x (n/Pc) x n block."""
    H, hi, hj = n // 2, n // (2 * pr), n // (2 * pc)
    return [(a * H + r * hi, b * H + c * hj, a * hi, b * hj, hi, hj) for a in (0, 1) for b in (0, 1)]


class MultiGPU:
    """P GPUs driven by this process (include/arena_fft.h arena_mgpu_*): rank v on
    devices[v] owns planes [v n/P, (v+1) n/P); the exchanges are peer stores fused
    into K2 / K3, the phases ordered by cross-device events.  The drop-in C++
    poisson_spectral_solve uses it when ARENA_FFT_NGPU > 1."""

    def __init__(self, n: int, nranks: int, devices=None, precision: int = 64):
        self._m = _vp()
        dv = None
        if devices is not None:
            if len(devices) != nranks:
                raise ValueError("one device per rank")
            dv = (_i * nranks)(*[int(d) for d in devices])
        _check(lib.arena_mgpu_create(ctypes.byref(self._m), int(n), int(precision), int(nranks), dv),
               "arena_mgpu_create")
        self.n, self.nranks, self.precision = int(n), int(nranks), int(precision)
        P, sb = _i(), ctypes.c_size_t()
        devs = (_i * nranks)()
        _check(lib.arena_mgpu_info(self._m, ctypes.byref(P), devs, ctypes.byref(sb)), "arena_mgpu_info")
        self.devices, self.slab_bytes = list(devs), sb.value

    def solve_device(self, fs, us, streams=None) -> None:
        """fs[v], us[v]: rank v's (n/P) x n x n CUDA tensors on devices[v] (may alias)."""
        P = self.nranks
        numel = (self.n // P) * self.n * self.n
        if len(fs) != P or len(us) != P:
            raise ValueError("one shard per rank")
        for v in range(P):
            _check_buffer(fs[v], numel, self.precision // 8, f"shard f[{v}]", self.devices[v])
            _check_buffer(us[v], numel, self.precision // 8, f"shard u[{v}]", self.devices[v])
        fa = (_vp * P)(*[_ptr(x) for x in fs])
        ua = (_vp * P)(*[_ptr(x) for x in us])
        sa = (_vp * P)(*[int(x) for x in streams]) if streams is not None else None
        _check(lib.arena_mgpu_solve_device(self._m, fa, ua, sa), "arena_mgpu_solve_device")

    def solve_host(self, f, u) -> None:
        """Whole n^3 host field in, whole field out (synchronous)."""
        n3 = self.n ** 3
        _check_buffer(f, n3, self.precision // 8, "solve_host f")
        _check_buffer(u, n3, self.precision // 8, "solve_host u")
        _check(lib.arena_mgpu_solve_host(self._m, _vp(_ptr(f)), _vp(_ptr(u))), "arena_mgpu_solve_host")

    def close(self) -> None:
        if getattr(self, "_m", None) and self._m.value:
            lib.arena_mgpu_destroy(self._m)
            self._m = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def slab_exchange_pieces(n: int, nranks: int, forward: bool, lo: int, hi: int):
    """Host-only: in-chunk row ranges [(first, rows), ...] that one sub-step [lo, hi) of the
    slab's chunked all-to-all moves between every pair of ranks (include/arena_fft.h)."""
    first = (ctypes.c_size_t * 4096)()
    rows = (ctypes.c_size_t * 4096)()
    k = lib.arena_slab_exchange_pieces(int(n), int(nranks), int(bool(forward)), int(lo), int(hi), first, rows, 4096)
    if k < 0:
        raise ValueError("bad exchange sub-step")
    return [(first[i], rows[i]) for i in range(k)]


def nccl_unique_id() -> bytes:
    nb = lib.arena_nccl_unique_id_bytes()
    buf = ctypes.create_string_buffer(nb)
    _check(lib.arena_nccl_unique_id(buf, nb), "arena_nccl_unique_id")
    return buf.raw


_plans: dict = {}
_plans_lock = threading.Lock()


def get_plan(n: int, precision: int = 64, device: int = -1) -> Plan:
    """Plan cache keyed by (n, precision, device) — the analogue of the reference's
    planner mutex (fft_solver.cpp:10-11), created once instead of per call."""
    key = (int(n), int(precision), int(device))
    with _plans_lock:
        p = _plans.get(key)
        if p is None:
            p = Plan(n, precision, device)
            _plans[key] = p
        return p


def clear_plan_cache() -> None:
    """Destroy the cached plans (their workspaces and host-path buffers)."""
    with _plans_lock:
        plans = list(_plans.values())
        _plans.clear()
    for p in plans:
        p.close()


def _as_grid(f: np.ndarray, dtype) -> np.ndarray:
    f = np.ascontiguousarray(f, dtype=dtype)
    if f.ndim != 3 or not (f.shape[0] == f.shape[1] == f.shape[2]):
        raise ValueError("GridField: expected an n x n x n array")
    if f.shape[0] < 2:
        raise ValueError("GridField: n >= 2 required")
    return f


def poisson_spectral_solve(f: np.ndarray, precision: int = 64) -> np.ndarray:
    """u with -Lap u = f - mean(f), mean(u) = 0 (fft_solver.cpp:51-87) — host arrays in/out."""
    dtype = np.float64 if precision == 64 else np.float32
    f = _as_grid(f, dtype)
    u = np.empty_like(f)
    p = get_plan(f.shape[0], precision)
    with p.lock:
        p.solve_host(f, u)
    return u


def dft3_forward(g: np.ndarray) -> np.ndarray:
    """Full n^3 complex spectrum, unnormalised, sign -1 (fft_solver.cpp:13-29)."""
    g = _as_grid(g, np.float64)
    p = get_plan(g.shape[0], 64)
    with p.lock:
        return p.dft3_forward_host(g)


def dft3_inverse(spec: np.ndarray, n: int) -> np.ndarray:
    """Re(backward DFT)/n^3 (fft_solver.cpp:31-49); size mismatch -> ValueError."""
    spec = np.ascontiguousarray(spec, dtype=np.complex128)
    if spec.size != n * n * n:
        raise ValueError("dft3_inverse: size mismatch")
    if n < 2:
        raise ValueError("GridField: n >= 2 required")
    p = get_plan(n, 64)
    with p.lock:
        return p.dft3_inverse_host(spec.reshape(n, n, n))


def _prec_of(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return 64
    if t.dtype == torch.float32:
        return 32
    raise TypeError("field must be float64 or float32")


def field_stats(t):
    """(mean, max_abs) of a contiguous CUDA tensor (GridField::mean / max_abs, grid.cpp:9-19), on the device."""
    m, a = ctypes.c_double(), ctypes.c_double()
    _check(lib.arena_field_stats(t.numel(), _prec_of(t), _vp(_ptr(t)), ctypes.byref(m), ctypes.byref(a)),
           "arena_field_stats")
    return m.value, a.value


def field_compare(num, exact) -> dict:
    """Gauge-aligned errors of num vs exact (problems.cpp:88-106 on the grid), on the device:
    {"rel_l2", "linf_rel", "gauge_shift"}."""
    if num.numel() != exact.numel() or num.dtype != exact.dtype:
        raise ValueError("fields must have the same size and dtype")
    r, li, sh = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _check(lib.arena_field_compare(num.numel(), _prec_of(num), _vp(_ptr(num)), _vp(_ptr(exact)), ctypes.byref(r),
                                   ctypes.byref(li), ctypes.byref(sh)), "arena_field_compare")
    return {"rel_l2": r.value, "linf_rel": li.value, "gauge_shift": sh.value}


class SpectralInterpolant:
    """Mirror of arena::SpectralInterpolant (fft_solver.hpp:27-36, fft_solver.cpp:89-114):
    modes of the full spectrum above rel_cut * max|mode| (spectrum from the GPU
    dft3_forward); evaluation of many points at once on the GPU."""

    def __init__(self, k: np.ndarray, amp: np.ndarray):
        self.k = np.ascontiguousarray(k, dtype=np.int32).reshape(-1, 3)
        self.amp = np.ascontiguousarray(amp, dtype=np.complex128).ravel()

    @classmethod
    def build(cls, g: np.ndarray, rel_cut: float = 1e-14) -> "SpectralInterpolant":
        spec = dft3_forward(g)
        n = g.shape[0]
        mag = np.abs(spec)
        keep = np.nonzero(mag > rel_cut * mag.max())
        sf = np.where(np.arange(n) <= n // 2, np.arange(n), np.arange(n) - n)
        k = np.stack([sf[keep[0]], sf[keep[1]], sf[keep[2]]], axis=1)
        return cls(k, spec[keep] / float(n) ** 3)

    def __call__(self, pts, device: int = -1) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.empty(pts.shape[0], dtype=np.float64)
        a = np.ascontiguousarray(np.stack([self.amp.real, self.amp.imag], axis=-1))
        _check(lib.arena_interpolant_eval(int(device), self.k.shape[0], _vp(self.k.ctypes.data), _vp(a.ctypes.data),
                                          pts.shape[0], _vp(pts.ctypes.data), _vp(out.ctypes.data)),
               "arena_interpolant_eval")
        return out


def source_modes(n: int, kvec: np.ndarray, coef: np.ndarray, out, precision: int = 64, stream: int = 0,
                 i0: int = 0, ni: Optional[int] = None, j0: int = 0, nj: Optional[int] = None) -> None:
    """Device buffer `out` = sum_m Re(coef_m e^{2 pi i k_m.x}) on the block i0..i0+ni-1 x j0..j0+nj-1 x all k
    (default: all n^3).  kvec: (M, 3) ints, coef: (M,) complex."""
    kvec = np.ascontiguousarray(kvec, dtype=np.int32).reshape(-1, 3)
    c = np.ascontiguousarray(np.stack([np.real(coef), np.imag(coef)], axis=-1), dtype=np.float64)
    _check(lib.arena_source_modes_block(int(n), int(precision), int(kvec.shape[0]), _vp(kvec.ctypes.data),
                                        _vp(c.ctypes.data), int(i0), int(n if ni is None else ni), int(j0),
                                        int(n if nj is None else nj), _vp(_ptr(out)), _vp(stream)),
           "arena_source_modes")


def source_gaussian(n: int, alpha: float, center, which: int, out, precision: int = 64, stream: int = 0,
                    i0: int = 0, ni: Optional[int] = None, j0: int = 0, nj: Optional[int] = None) -> None:
    """Device buffer `out` = periodised Gaussian u (which=0) or f = -Lap u (which=1) on a block."""
    cx, cy, cz = (float(c) for c in center)
    _check(lib.arena_source_gaussian_block(int(n), int(precision), float(alpha), cx, cy, cz, int(which), int(i0),
                                           int(n if ni is None else ni), int(j0), int(n if nj is None else nj),
                                           _vp(_ptr(out)), _vp(stream)), "arena_source_gaussian")


__all__ = [
    "Plan", "Slab", "Pencil", "MultiGPU", "fold_blocks", "SpectralInterpolant", "nccl_unique_id", "get_plan", "poisson_spectral_solve", "dft3_forward", "dft3_inverse", "signed_freq",
    "source_modes", "source_gaussian", "ArenaError", "lib", "LIB_PATH", "CORE_PATH", "HEADER_PATH",
    "PATH_POW2", "PATH_GENERIC",
]
