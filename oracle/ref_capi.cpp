// C entry points into the reference's own arena::poisson_spectral_solve /
// dft3_forward / dft3_inverse (fft_solver.cpp:13-87 compiled unmodified over
// oracle/fftw_shim).  TEST INFRASTRUCTURE ONLY: loaded by tests/ and by
// bench.py's --impl reference / cpu_baseline leg, never by the product.
#include <algorithm>
#include <complex>

#include "arena/fft_solver.hpp"
#include "offt.h"

extern "C" {

void ref_set_threads(int nthreads) { offt_set_threads(nthreads); }
int ref_get_threads(void) { return offt_get_threads(); }

int ref_poisson_solve(int n, const double* f, double* u) {
  try {
    arena::GridField g(n);
    std::copy(f, f + g.size(), g.data.begin());
    const arena::GridField r = arena::poisson_spectral_solve(g);
    std::copy(r.data.begin(), r.data.end(), u);
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_dft3_forward(int n, const double* g, double* spec) {
  try {
    arena::GridField a(n);
    std::copy(g, g + a.size(), a.data.begin());
    const auto s = arena::dft3_forward(a);
    std::copy(reinterpret_cast<const double*>(s.data()), reinterpret_cast<const double*>(s.data()) + 2 * s.size(),
              spec);
    return 0;
  } catch (...) {
    return -1;
  }
}

int ref_dft3_inverse(int n, const double* spec, double* g) {
  try {
    const size_t N = size_t(n) * n * n;
    std::vector<std::complex<double>> s(N);
    std::copy(spec, spec + 2 * N, reinterpret_cast<double*>(s.data()));
    const arena::GridField r = arena::dft3_inverse(s, n);
    std::copy(r.data.begin(), r.data.end(), g);
    return 0;
  } catch (...) {
    return -1;
  }
}
}
