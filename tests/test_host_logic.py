"""CPU tests of host-side logic: the bench launcher, the lazy library load, buffer
validation before pointers cross the C ABI, and the host-side config sources."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_gpus2_self_launches_two_ranks():
    """`python bench.py --gpus 2` outside torchrun spawns two ranks (gloo dry run here)
    and rank 0 alone prints one JSON line with n_gpus = 2."""
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["world_size"] == 2 and d["max_over_ranks"] == 2.0


def test_bench_rejects_gpus_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "4", "--steps", "1"],
                       capture_output=True, text=True, timeout=120, cwd=REPO, env=env)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


def test_package_import_maps_no_cuda_library():
    """Importing the package (e.g. problems.py for the CPU reference arm) must not load
    libarena_fft.so; the first library call does."""
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1408_6497_b200 import problems\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libarena_fft' not in maps, 'mapped at import'\n"
            "import paper_1408_6497_b200 as a\n"
            "a.lib.arena_fft_abi_version()\n"
            "assert 'libarena_fft' in open('/proc/self/maps').read()\n" % REPO)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-2000:]


def test_check_buffer_rejects_bad_fields():
    from paper_1408_6497_b200 import _check_buffer

    ok = np.zeros((4, 4, 4))
    _check_buffer(ok, 64, 8, "f")
    with pytest.raises(TypeError):
        _check_buffer(ok.astype(np.float32), 64, 8, "f")  # fp32 buffer on a fp64 plan
    with pytest.raises(ValueError):
        _check_buffer(np.zeros((4, 4, 3)), 64, 8, "f")  # short
    with pytest.raises(ValueError):
        _check_buffer(np.zeros((4, 4, 8))[:, :, ::2], 64, 8, "f")  # not contiguous
    with pytest.raises(TypeError):
        _check_buffer(ok, 64, 8, "f", device=0)  # host array where a CUDA tensor is required
    import torch

    t = torch.zeros(64, dtype=torch.float64)
    _check_buffer(t, 64, 8, "f")
    with pytest.raises(TypeError):
        _check_buffer(t, 64, 8, "f", device=0)


@pytest.mark.parametrize("n", [15, 16, 33])
def test_host_field_matches_direct_evaluation(n):
    """problems.host_field (c2r of a sparse half spectrum — the CPU arm's 1024^3 source)
    equals direct per-point evaluation, including aliased and self-conjugate planes."""
    from paper_1408_6497_b200 import problems

    for src in (problems.config(4, n), problems.config(2, n), problems.random_modes(n, 16, n // 2, seed=3)):
        for which in "fu":
            a, b = problems.host_field(src, which), problems.eval_host(src, which)
            assert np.abs(a - b).max() <= 1e-14 * np.abs(b).max()


def test_bench_reference_arm_small():
    """--impl reference at a small n: one JSON line, the same workload as the GPU arm
    (same_config), a 1-core and a pocketfft line, and no repo CUDA library mapped."""
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference", "--n", "80",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["config"]["same_config"] and d["config"]["n"] == 80
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["one_core"]["cores"] == 1 and cb["b_all"]["rel_l2_vs_reference"] < 1e-13
    assert d["parity"]["rel_l2_vs_analytic"] < 1e-12
    assert not any(m.startswith("paper_1408_6497_b200") for m in d["repo_libs_mapped"])
    assert "invalid" not in d
