"""CPU tests of the drop-in boundary: the C-ABI library loads and exports every
declared symbol, the C++ drop-in exports the reference's fft_solver API, and
argument errors behave like the reference's (no GPU calls here)."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1408_6497_b200 as arena


def _declared(header):
    text = open(header).read()
    return sorted(set(re.findall(r"\b(arena_[a-z0-9_]+)\s*\(", text)))


def _exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line}


def test_c_abi_exports_every_declared_symbol():
    declared = _declared(arena.HEADER_PATH)
    assert "arena_poisson_solve_device" in declared and "arena_poisson_solve_host" in declared
    exported = _exported(arena.LIB_PATH)
    missing = [s for s in declared if s not in exported]
    assert not missing, missing


def test_cpp_dropin_exports_reference_api():
    out = subprocess.run(["nm", "-DC", "--defined-only", arena.CORE_PATH], capture_output=True, text=True,
                         check=True).stdout
    for sym in ("arena::poisson_spectral_solve(arena::GridField const&)",
                "arena::dft3_forward(arena::GridField const&)",
                "arena::dft3_inverse(std::vector<std::complex<double>, std::allocator<std::complex<double> > > const&, int)",
                "arena::SpectralInterpolant::build(arena::GridField const&, double)",
                "arena::SpectralInterpolant::operator()(std::array<double, 3ul> const&) const",
                "arena::sample_grid(", "arena::grid_write(", "arena::grid_read("):
        assert sym in out, sym


def test_kernels_are_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", arena.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out, out[:500]


def test_abi_version():
    assert arena.lib.arena_fft_abi_version() == 101


def test_invalid_n_raises_like_gridfield():
    """GridField(n < 2) throws std::invalid_argument (grid.hpp:18) -> EINVAL / ValueError."""
    with pytest.raises(ValueError):
        arena.Plan(1)
    with pytest.raises(ValueError):
        arena.poisson_spectral_solve(np.zeros((1, 1, 1)))
    with pytest.raises(ValueError):
        arena.dft3_inverse(np.zeros(7, dtype=complex), 2)
    with pytest.raises(ValueError):
        arena.Plan(8, precision=16)


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(arena.ArenaError) as ei:
        arena.Plan(8)
    assert ei.value.status == 5  # ARENA_EUNSUPPORTED


def test_reference_tests_against_dropin_fail_loudly_without_gpu(tmp_path):
    import torch
    import oracle

    if torch.cuda.is_available():
        pytest.skip("GPU present (covered by the gpu parity tests)")
    if not os.path.exists(oracle.TEST_FFT_DROPIN):
        pytest.skip("dropin test binary not built")
    r = subprocess.run([oracle.TEST_FFT_DROPIN], cwd=tmp_path, capture_output=True, text=True, timeout=120)
    assert r.returncode != 0  # every solve throws: there is no CPU path
    assert "TEST CASE THREW" in r.stderr
