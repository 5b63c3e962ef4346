"""Generate the committed golden vectors for the spectral Poisson path.

Run in the build container (needs /root/reference for the reference build):
    make -C oracle ref && python tests/golden/make_golden.py

Outputs (committed): tests/golden/poisson_golden.npz, dft3_golden.npz, MANIFEST.json.

Each output is produced by the REFERENCE'S OWN solver code
(/root/reference/proj/src/fft_solver.cpp:13-87 compiled unmodified over the
FFTW3-API shim, oracle/_ref/libref_poisson.so) and cross-checked here against
scipy.fft (pocketfft, an independent engine) before it is written; dft3 at
n <= 6 is also checked against the O(N^2) direct DFT (oracles.cpp:13-29).
Inputs are seeded numpy draws (uniform(-1,1)) plus structured cases from the
reference's tests (test_fft.cpp:44-99).
"""
import json
import os
import sys

import numpy as np
import scipy.fft as sf

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import oracle  # noqa: E402


def scipy_poisson(f):
    n = f.shape[0]
    F = sf.rfftn(f)
    k = np.array([i if i <= n // 2 else i - n for i in range(n)], dtype=float)
    kk = np.arange(n // 2 + 1, dtype=float)
    k2 = k[:, None, None] ** 2 + k[None, :, None] ** 2 + kk[None, None, :] ** 2
    with np.errstate(divide="ignore"):
        s = np.where(k2 == 0, 0.0, (1.0 / (float(n) ** 3)) / (4.0 * np.pi * np.pi * k2))
    return sf.irfftn(F * s, s=f.shape) * n ** 3


def rel(a, b):
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))


def main():
    assert oracle.available("ref"), "build the reference oracle first: make -C oracle ref"
    out, man = {}, {"generator": "tests/golden/make_golden.py", "engine": "oracle/_ref/libref_poisson.so "
                    "(reference fft_solver.cpp over the FFTW3-API shim)", "cases": {}}
    # --- Poisson solve
    cases = []
    for n in (2, 3, 4, 5, 6, 8, 10, 12, 16, 32):
        cases.append((f"rand_n{n}", np.random.default_rng(1000 + n).uniform(-1, 1, (n, n, n))))
    for n in (4, 8, 16):  # test_fft.cpp:82-92 single mode
        x = np.arange(n) / n
        cases.append((f"sinx_n{n}", np.broadcast_to(4 * np.pi ** 2 * np.sin(2 * np.pi * x)[:, None, None], (n, n, n)).copy()))
    cases.append(("const7_n8", np.full((8, 8, 8), 7.0)))  # test_fft.cpp:94-99
    x = np.arange(32) / 32  # test_fft.cpp:101-114, osc k=8
    w = 2 * np.pi * 8
    cases.append(("osc8_n32", 3 * w * w * np.sin(w * x)[:, None, None] * np.sin(w * x)[None, :, None] * np.sin(w * x)[None, None, :]))
    for name, f in cases:
        u = oracle.poisson_solve(f, "ref")
        e = rel(u, scipy_poisson(f))
        assert e < 1e-13 or np.linalg.norm(u) < 1e-12, (name, e)
        out[f"{name}_f"], out[f"{name}_u"] = f, u
        man["cases"][name] = {"op": "poisson_spectral_solve", "n": f.shape[0], "scipy_rel_l2": e}
    np.savez_compressed(os.path.join(HERE, "poisson_golden.npz"), **out)
    # --- dft3_forward / dft3_inverse
    out = {}
    for n in (2, 4, 6, 8, 10):
        g = np.random.default_rng(2000 + n).uniform(-1, 1, (n, n, n))
        s = oracle.dft3_forward(g, "ref")
        e = rel(s, sf.fftn(g))
        if n <= 6:
            e = max(e, rel(s, oracle.direct_dft3(g)))
        assert e < 1e-13, (n, e)
        back = oracle.dft3_inverse(s, n, "ref")
        assert rel(back, g) < 1e-13
        out[f"dft_n{n}_g"], out[f"dft_n{n}_spec"] = g, s
        man["cases"][f"dft_n{n}"] = {"op": "dft3_forward", "n": n, "max_rel_vs_scipy_direct": e}
    np.savez_compressed(os.path.join(HERE, "dft3_golden.npz"), **out)
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump(man, fh, indent=1)
    print("wrote", len(man["cases"]), "golden cases")


if __name__ == "__main__":
    main()
