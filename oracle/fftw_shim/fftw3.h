/*
 * Minimal FFTW3 API declaration — TEST INFRASTRUCTURE ONLY (oracle).
 *
 * Declares exactly the FFTW3 entry points the reference's fft_solver.cpp
 * calls (/root/reference/proj/src/fft_solver.cpp:20-26,37-43,60-65,80-84) so
 * that file compiles UNMODIFIED here, where libfftw3 is not installed.  The
 * definitions live in fftw3_shim.c and run oracle/offt.c (the DFT
 * definitions FFTW documents: unnormalised, FFTW_FORWARD = -1 exponent sign,
 * r2c halves the last dimension, c2r treats its input as Hermitian).
 * Builder-written; not FFTW's header.
 */
#ifndef ORACLE_FFTW3_SHIM_H
#define ORACLE_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct oracle_fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out, unsigned flags);
fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out, unsigned flags);
void fftw_execute(const fftw_plan p);
void fftw_destroy_plan(fftw_plan p);

#ifdef __cplusplus
}
#endif
#endif
