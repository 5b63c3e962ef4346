/*
 * FFTW3-API shim over oracle/offt.c — TEST INFRASTRUCTURE ONLY.
 * Lets the reference's own fft_solver.cpp run unmodified as the CPU oracle /
 * CPU baseline (oracle/_ref/libref_poisson.so).  A plan just records its
 * arguments; fftw_execute runs the vfft.c transform (the FFTW stand-in engine,
 * cross-checked against the independent oracle/offt.c in tests/test_oracle.py)
 * on the recorded buffers.
 */
#include <stdlib.h>

#include "../offt.h"
#include "fftw3.h"
#include "vfft.h"

enum { K_C2C, K_R2C, K_C2R };

struct oracle_fftw_plan_s {
  int kind, n0, n1, n2, sign;
  void* in;
  void* out;
};

static fftw_plan mk(int kind, int n0, int n1, int n2, int sign, void* in, void* out) {
  fftw_plan p = (fftw_plan)malloc(sizeof *p);
  if (!p) return NULL;
  p->kind = kind; p->n0 = n0; p->n1 = n1; p->n2 = n2; p->sign = sign;
  p->in = in; p->out = out;
  return p;
}

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
  (void)flags;
  return mk(K_C2C, n0, n1, n2, sign, in, out);
}

fftw_plan fftw_plan_dft_r2c_3d(int n0, int n1, int n2, double* in, fftw_complex* out, unsigned flags) {
  (void)flags;
  return mk(K_R2C, n0, n1, n2, -1, in, out);
}

fftw_plan fftw_plan_dft_c2r_3d(int n0, int n1, int n2, fftw_complex* in, double* out, unsigned flags) {
  (void)flags;
  return mk(K_C2R, n0, n1, n2, +1, in, out);
}

void fftw_execute(const fftw_plan p) {
  if (!p) return;
  switch (p->kind) {
    case K_C2C: vfft_c2c_3d(p->n0, p->n1, p->n2, (const double*)p->in, (double*)p->out, p->sign); break;
    case K_R2C: vfft_r2c_3d(p->n0, p->n1, p->n2, (const double*)p->in, (double*)p->out); break;
    case K_C2R: vfft_c2r_3d(p->n0, p->n1, p->n2, (double*)p->in, (double*)p->out); break;
  }
}

void fftw_destroy_plan(fftw_plan p) { free(p); }
