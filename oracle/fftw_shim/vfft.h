/* vfft.h — FFTW stand-in engine of the shim (TEST INFRASTRUCTURE ONLY; see vfft.c).
 * Same contracts as the offt_*_3d routines in ../offt.h. */
#ifndef VFFT_H
#define VFFT_H
#ifdef __cplusplus
extern "C" {
#endif
int vfft_c2c_3d(int n0, int n1, int n2, const double* in, double* out, int sign);
int vfft_r2c_3d(int n0, int n1, int n2, const double* in, double* out);
int vfft_c2r_3d(int n0, int n1, int n2, double* in, double* out);
#ifdef __cplusplus
}
#endif
#endif
