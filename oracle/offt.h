/*
 * offt — CPU restatement of the reference's FFT spectral Poisson path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_1408_6497_b200/ links, loads or
 * calls this code; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may use it, and there only as the checker
 * or the CPU baseline being reported.
 *
 * What it restates:
 *   - FFTW 3 (the reference's third-party FFT, `find_library(FFTW3_LIB fftw3)`,
 *     /root/reference/proj/src/CMakeLists.txt:3-4, version unpinned) — only the
 *     published DFT definitions the reference relies on:
 *       forward  X[k] = sum_x x[x] exp(-2 pi i k.x / n)   (FFTW_FORWARD = -1)
 *       backward x[x] = sum_k X[k] exp(+2 pi i k.x / n)   (FFTW_BACKWARD = +1)
 *     both unnormalised; r2c keeps k_last in [0, n/2]; c2r reads that half
 *     spectrum as Hermitian (imaginary parts of the self-conjugate modes are
 *     ignored).  Algorithm: recursive mixed-radix decimation-in-time
 *     Cooley-Tukey (radix 4/2/3/5 butterflies + O(p^2) DFT for other primes),
 *     twiddles from an 80-bit long-double table.  This is deliberately NOT the
 *     Stockham formulation the CUDA kernels use.
 *   - arena::poisson_spectral_solve, /root/reference/proj/src/fft_solver.cpp:51-87
 *     (offt_poisson_solve below, same op order incl. the k2==0 test and the
 *     `scale / (four_pi2 * k2)` expression at fft_solver.cpp:66-79).
 *   - arena::dft3_forward / dft3_inverse, fft_solver.cpp:13-49.
 *
 * Parity pins: tests/test_oracle.py checks this file against the reference's
 * own known-answer tests (test_fft.cpp T1-T12, run unmodified through
 * oracle/_ref/test_fft_ref), against oracle::direct_dft3 semantics, and against
 * the committed golden vectors in tests/golden/ (scipy pocketfft, a third
 * independent engine).
 */
#ifndef OFFT_H
#define OFFT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Interleaved complex double (re, im), the FFTW / std::complex<double> layout. */

/* Set the number of OpenMP threads used by the 3D routines (<=0: all). */
void offt_set_threads(int nthreads);
int offt_get_threads(void);

/* 1D unnormalised c2c DFT of length n, in place on x (interleaved), sign -1/+1. */
int offt_c2c_1d(int n, double* x, int sign);

/* 3D c2c on an n0 x n1 x n2 row-major interleaved complex array (out may == in). */
int offt_c2c_3d(int n0, int n1, int n2, const double* in, double* out, int sign);

/* 3D r2c: real n0 x n1 x n2 -> complex n0 x n1 x (n2/2+1), FFTW layout. */
int offt_r2c_3d(int n0, int n1, int n2, const double* in, double* out);

/* 3D c2r: complex n0 x n1 x (n2/2+1) (Hermitian) -> real n0 x n1 x n2, unnormalised.
 * `in` is used as scratch (destroyed), like FFTW's default c2r. */
int offt_c2r_3d(int n0, int n1, int n2, double* in, double* out);

/* Restatement of arena::poisson_spectral_solve (fft_solver.cpp:51-87) on an
 * n^3 GridField.data buffer.  Returns 0 on success. */
int offt_poisson_solve(int n, const double* f, double* u);

/* Restatements of arena::dft3_forward / dft3_inverse (fft_solver.cpp:13-49).
 * spec is interleaved complex n^3; dft3_inverse returns Re(.)/n^3. */
int offt_dft3_forward(int n, const double* g, double* spec);
int offt_dft3_inverse(int n, const double* spec, double* g);

#ifdef __cplusplus
}
#endif
#endif
