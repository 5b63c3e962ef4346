/*
 * vfft.c — the transform engine behind the FFTW3-API shim (TEST INFRASTRUCTURE
 * ONLY: it is what oracle/_ref/libref_poisson.so, i.e. the reference's own
 * fft_solver.cpp, executes when it calls fftw_execute).
 *
 * It stands in for FFTW 3 (unpinned, `find_library(FFTW3_LIB fftw3)`,
 * /root/reference/proj/src/CMakeLists.txt:3-4) and restates only FFTW's
 * published transform definitions:
 *   forward  X[k] = sum_x x[x] exp(-2 pi i k.x / n)   (FFTW_FORWARD = -1)
 *   backward x[x] = sum_k X[k] exp(+2 pi i k.x / n)   (FFTW_BACKWARD = +1)
 * unnormalised; r2c keeps the last axis' k in [0, n/2]; c2r reads that half
 * spectrum as Hermitian and ignores the imaginary parts of the self-conjugate
 * modes (DC and, for even n, Nyquist).
 *
 * Why a second engine next to oracle/offt.c: the shim is also the timed CPU
 * baseline (bench.py --impl reference), so it should be a reasonable stand-in
 * for FFTW's speed, not just its definitions.  offt.c (recursive DIT, one line
 * at a time, r2c through a full complex FFT) stays the independent restatement
 * the tests cross-check this engine against.  Here:
 *   - mixed-radix Stockham autosort (radix 4/2/3 butterflies, O(R^2) DFT for
 *     other factors), twiddles from an 80-bit long-double table;
 *   - VB = 8 lines transformed together, split re/im, so every butterfly is
 *     one SIMD loop over the 8 lines and every twiddle is loaded once per 8;
 *   - r2c / c2r transform two real rows per complex FFT (z = x0 + i x1, split
 *     on the way out / merged on the way in), FFTW's half-cost real transforms;
 *   - OpenMP over blocks of lines (threads: offt_set_threads).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../offt.h"
#include "vfft.h"

#define VB 8

typedef struct {
  int n, ns;
  int rad[64];
  double *wr, *wi; /* W_n^m = exp(-2 pi i m / n), m in [0, n) */
} vplan;

static int vplan_init(vplan* p, int n) {
  if (n < 1) return -1;
  p->n = n;
  p->ns = 0;
  int m = n;
  while (m % 4 == 0) { p->rad[p->ns++] = 4; m /= 4; }
  while (m % 2 == 0) { p->rad[p->ns++] = 2; m /= 2; }
  for (int q = 3; m > 1; q += 2) {
    while (m % q == 0) { p->rad[p->ns++] = q; m /= q; }
    if ((long)q * q > m && m > 1) { p->rad[p->ns++] = m; m = 1; }
  }
  p->wr = (double*)malloc(sizeof(double) * (size_t)n);
  p->wi = (double*)malloc(sizeof(double) * (size_t)n);
  if (!p->wr || !p->wi) return -1;
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int k = 0; k < n; ++k) {
    const long double a = two_pi * (long double)k / (long double)n;
    p->wr[k] = (double)cosl(a);
    p->wi[k] = (double)-sinl(a);
  }
  return 0;
}

static void vplan_free(vplan* p) {
  free(p->wr);
  free(p->wi);
}

/* One Stockham stage over VB lines: x -> y, radix R, Ns = product of the
 * previous radices.  Element t of line b lives at [t * VB + b]. */
static void vstage(const vplan* p, int R, int Ns, int sign, const double* restrict xr, const double* restrict xi,
                   double* restrict yr, double* restrict yi) {
  const int n = p->n, m = n / R, tstep = n / (Ns * R);
  const double sg = (double)sign;
  double wr[64], wi[64];
  double* gwr = R > 64 ? (double*)malloc(sizeof(double) * (size_t)R * 2) : wr;
  double* gwi = R > 64 ? gwr + R : wi;
  for (int j = 0; j < m; ++j) {
    const int jm = j % Ns;
    const int ob = (j / Ns) * Ns * R + jm;
    for (int r = 0; r < R; ++r) {
      const int e = jm * r * tstep; /* < n */
      gwr[r] = p->wr[e];
      gwi[r] = sign > 0 ? -p->wi[e] : p->wi[e]; /* table holds -sin: sign -1 keeps it, +1 flips it */
    }
#define LD(r) const double* restrict ar##r = xr + (size_t)(j + (r) * m) * VB; \
              const double* restrict ai##r = xi + (size_t)(j + (r) * m) * VB;
#define ST(r) double* restrict br##r = yr + (size_t)(ob + (r) * Ns) * VB; \
              double* restrict bi##r = yi + (size_t)(ob + (r) * Ns) * VB;
    if (R == 2) {
      LD(0) LD(1) ST(0) ST(1)
      const double w1r = gwr[1], w1i = gwi[1];
#pragma omp simd
      for (int b = 0; b < VB; ++b) {
        const double v1r = ar1[b] * w1r - ai1[b] * w1i, v1i = ar1[b] * w1i + ai1[b] * w1r;
        br0[b] = ar0[b] + v1r; bi0[b] = ai0[b] + v1i;
        br1[b] = ar0[b] - v1r; bi1[b] = ai0[b] - v1i;
      }
    } else if (R == 4) {
      LD(0) LD(1) LD(2) LD(3) ST(0) ST(1) ST(2) ST(3)
      const double w1r = gwr[1], w1i = gwi[1], w2r = gwr[2], w2i = gwi[2], w3r = gwr[3], w3i = gwi[3];
#pragma omp simd
      for (int b = 0; b < VB; ++b) {
        const double v0r = ar0[b], v0i = ai0[b];
        const double v1r = ar1[b] * w1r - ai1[b] * w1i, v1i = ar1[b] * w1i + ai1[b] * w1r;
        const double v2r = ar2[b] * w2r - ai2[b] * w2i, v2i = ar2[b] * w2i + ai2[b] * w2r;
        const double v3r = ar3[b] * w3r - ai3[b] * w3i, v3i = ar3[b] * w3i + ai3[b] * w3r;
        const double s02r = v0r + v2r, s02i = v0i + v2i, d02r = v0r - v2r, d02i = v0i - v2i;
        const double s13r = v1r + v3r, s13i = v1i + v3i, d13r = v1r - v3r, d13i = v1i - v3i;
        /* y1 = d02 + sign * i * d13, y3 = d02 - sign * i * d13 */
        br0[b] = s02r + s13r; bi0[b] = s02i + s13i;
        br2[b] = s02r - s13r; bi2[b] = s02i - s13i;
        br1[b] = d02r - sg * d13i; bi1[b] = d02i + sg * d13r;
        br3[b] = d02r + sg * d13i; bi3[b] = d02i - sg * d13r;
      }
    } else if (R == 3) {
      LD(0) LD(1) LD(2) ST(0) ST(1) ST(2)
      const double w1r = gwr[1], w1i = gwi[1], w2r = gwr[2], w2i = gwi[2];
      const double s3 = sg * 0.86602540378443864676372317075294; /* sign * sin(2 pi / 3) */
#pragma omp simd
      for (int b = 0; b < VB; ++b) {
        const double v1r = ar1[b] * w1r - ai1[b] * w1i, v1i = ar1[b] * w1i + ai1[b] * w1r;
        const double v2r = ar2[b] * w2r - ai2[b] * w2i, v2i = ar2[b] * w2i + ai2[b] * w2r;
        const double tr = v1r + v2r, ti = v1i + v2i;
        const double mr = ar0[b] - 0.5 * tr, mi = ai0[b] - 0.5 * ti;
        const double dr = s3 * (v1r - v2r), di = s3 * (v1i - v2i);
        br0[b] = ar0[b] + tr; bi0[b] = ai0[b] + ti;
        br1[b] = mr - di; bi1[b] = mi + dr;
        br2[b] = mr + di; bi2[b] = mi - dr;
      }
    } else {
      /* generic radix: y_s = sum_r (x_r w_r) W_R^{rs}, W_R^q = W_n^{q n / R} */
      const int rstep = n / R;
      for (int s = 0; s < R; ++s) {
        double* restrict brs = yr + (size_t)(ob + s * Ns) * VB;
        double* restrict bis = yi + (size_t)(ob + s * Ns) * VB;
        double accr[VB], acci[VB];
        for (int b = 0; b < VB; ++b) accr[b] = acci[b] = 0.0;
        for (int r = 0; r < R; ++r) {
          const int q = (int)(((long)r * s) % R) * rstep;
          const double cr = p->wr[q], ci = sign > 0 ? -p->wi[q] : p->wi[q];
          /* combined factor (w_r * W_R^{rs}) */
          const double fr = gwr[r] * cr - gwi[r] * ci, fi = gwr[r] * ci + gwi[r] * cr;
          const double* restrict xrr = xr + (size_t)(j + r * m) * VB;
          const double* restrict xir = xi + (size_t)(j + r * m) * VB;
#pragma omp simd
          for (int b = 0; b < VB; ++b) {
            accr[b] += xrr[b] * fr - xir[b] * fi;
            acci[b] += xrr[b] * fi + xir[b] * fr;
          }
        }
        for (int b = 0; b < VB; ++b) { brs[b] = accr[b]; bis[b] = acci[b]; }
      }
    }
#undef LD
#undef ST
  }
  if (gwr != wr) free(gwr);
}

/* Transform the VB lines in (r0, i0); scratch (r1, i1).  Returns 1 when the
 * result ended in the scratch pair, 0 when in (r0, i0). */
static int vlines(const vplan* p, int sign, double* r0, double* i0, double* r1, double* i1) {
  int Ns = 1, flip = 0;
  for (int s = 0; s < p->ns; ++s) {
    const int R = p->rad[s];
    if (R == 1) continue;
    if (!flip) vstage(p, R, Ns, sign, r0, i0, r1, i1);
    else vstage(p, R, Ns, sign, r1, i1, r0, i0);
    flip ^= 1;
    Ns *= R;
  }
  return flip;
}

/* c2c along one axis of an [outer][len][inner] interleaved complex array. */
static void vaxis(double* a, long outer, int len, long inner, int sign) {
  vplan p;
  if (vplan_init(&p, len)) return;
  const long lines = outer * inner;
  const long nblk = (lines + VB - 1) / VB;
#pragma omp parallel num_threads(offt_get_threads())
  {
    double* buf = (double*)malloc(sizeof(double) * (size_t)len * VB * 4);
    double *r0 = buf, *i0 = buf + (size_t)len * VB, *r1 = buf + 2 * (size_t)len * VB, *i1 = buf + 3 * (size_t)len * VB;
#pragma omp for schedule(static)
    for (long blk = 0; blk < nblk; ++blk) {
      const long L0 = blk * VB;
      const int nb = (int)((lines - L0) < VB ? (lines - L0) : VB);
      double* base[VB];
      for (int b = 0; b < VB; ++b) {
        const long L = L0 + (b < nb ? b : nb - 1);
        base[b] = a + 2 * ((L / inner) * (long)len * inner + (L % inner));
      }
      const long st = 2 * inner;
      for (int t = 0; t < len; ++t)
        for (int b = 0; b < VB; ++b) {
          r0[(size_t)t * VB + b] = base[b][t * st];
          i0[(size_t)t * VB + b] = base[b][t * st + 1];
        }
      const int fl = vlines(&p, sign, r0, i0, r1, i1);
      const double* orr = fl ? r1 : r0;
      const double* oi = fl ? i1 : i0;
      for (int t = 0; t < len; ++t)
        for (int b = 0; b < nb; ++b) {
          base[b][t * st] = orr[(size_t)t * VB + b];
          base[b][t * st + 1] = oi[(size_t)t * VB + b];
        }
    }
    free(buf);
  }
  vplan_free(&p);
}

int vfft_c2c_3d(int n0, int n1, int n2, const double* in, double* out, int sign) {
  const size_t N = (size_t)n0 * n1 * n2;
  if (out != in) memcpy(out, in, sizeof(double) * 2 * N);
  vaxis(out, (long)n0 * n1, n2, 1, sign);
  vaxis(out, n0, n1, n2, sign);
  vaxis(out, 1, n0, (long)n1 * n2, sign);
  return 0;
}

/* Rows of the last axis: two real rows per complex FFT, VB complex lines per block. */
int vfft_r2c_3d(int n0, int n1, int n2, const double* in, double* out) {
  const int nc = n2 / 2 + 1;
  vplan p;
  if (vplan_init(&p, n2)) return -1;
  const long rows = (long)n0 * n1;
  const long pairs = (rows + 1) / 2;
  const long nblk = (pairs + VB - 1) / VB;
#pragma omp parallel num_threads(offt_get_threads())
  {
    double* buf = (double*)malloc(sizeof(double) * (size_t)n2 * VB * 4);
    double *r0 = buf, *i0 = buf + (size_t)n2 * VB, *r1 = buf + 2 * (size_t)n2 * VB, *i1 = buf + 3 * (size_t)n2 * VB;
#pragma omp for schedule(static)
    for (long blk = 0; blk < nblk; ++blk) {
      const long c0 = blk * VB;
      const int nb = (int)((pairs - c0) < VB ? (pairs - c0) : VB);
      for (int b = 0; b < VB; ++b) {
        const long c = c0 + (b < nb ? b : nb - 1);
        const double* x0 = in + (2 * c) * (long)n2;
        const double* x1 = (2 * c + 1 < rows) ? in + (2 * c + 1) * (long)n2 : NULL;
        for (int t = 0; t < n2; ++t) {
          r0[(size_t)t * VB + b] = x0[t];
          i0[(size_t)t * VB + b] = x1 ? x1[t] : 0.0;
        }
      }
      const int fl = vlines(&p, -1, r0, i0, r1, i1);
      const double* zr = fl ? r1 : r0;
      const double* zi = fl ? i1 : i0;
      for (int b = 0; b < nb; ++b) {
        const long c = c0 + b;
        double* X0 = out + 2 * (2 * c) * (long)nc;
        double* X1 = (2 * c + 1 < rows) ? out + 2 * (2 * c + 1) * (long)nc : NULL;
        for (int k = 0; k < nc; ++k) {
          const int kk = k ? n2 - k : 0;
          const double ar = zr[(size_t)k * VB + b], ai = zi[(size_t)k * VB + b];
          const double br = zr[(size_t)kk * VB + b], bi = zi[(size_t)kk * VB + b];
          /* X0 = (Z[k] + conj Z[-k]) / 2, X1 = (Z[k] - conj Z[-k]) / (2i) */
          X0[2 * k] = 0.5 * (ar + br);
          X0[2 * k + 1] = 0.5 * (ai - bi);
          if (X1) {
            X1[2 * k] = 0.5 * (ai + bi);
            X1[2 * k + 1] = -0.5 * (ar - br);
          }
        }
      }
    }
    free(buf);
  }
  vplan_free(&p);
  vaxis(out, n0, n1, nc, -1);
  vaxis(out, 1, n0, (long)n1 * nc, -1);
  return 0;
}

int vfft_c2r_3d(int n0, int n1, int n2, double* in, double* out) {
  const int nc = n2 / 2 + 1;
  vaxis(in, 1, n0, (long)n1 * nc, +1);
  vaxis(in, n0, n1, nc, +1);
  vplan p;
  if (vplan_init(&p, n2)) return -1;
  const long rows = (long)n0 * n1;
  const long pairs = (rows + 1) / 2;
  const long nblk = (pairs + VB - 1) / VB;
#pragma omp parallel num_threads(offt_get_threads())
  {
    double* buf = (double*)malloc(sizeof(double) * (size_t)n2 * VB * 4);
    double *r0 = buf, *i0 = buf + (size_t)n2 * VB, *r1 = buf + 2 * (size_t)n2 * VB, *i1 = buf + 3 * (size_t)n2 * VB;
#pragma omp for schedule(static)
    for (long blk = 0; blk < nblk; ++blk) {
      const long c0 = blk * VB;
      const int nb = (int)((pairs - c0) < VB ? (pairs - c0) : VB);
      for (int b = 0; b < VB; ++b) {
        const long c = c0 + (b < nb ? b : nb - 1);
        const double* h0 = in + 2 * (2 * c) * (long)nc;
        const double* h1 = (2 * c + 1 < rows) ? in + 2 * (2 * c + 1) * (long)nc : NULL;
        for (int k = 0; k < n2; ++k) {
          /* Hermitian completion; self-conjugate modes keep their real part only */
          double a_r, a_i, b_r = 0.0, b_i = 0.0;
          if (k < nc) {
            a_r = h0[2 * k]; a_i = h0[2 * k + 1];
            if (h1) { b_r = h1[2 * k]; b_i = h1[2 * k + 1]; }
          } else {
            a_r = h0[2 * (n2 - k)]; a_i = -h0[2 * (n2 - k) + 1];
            if (h1) { b_r = h1[2 * (n2 - k)]; b_i = -h1[2 * (n2 - k) + 1]; }
          }
          if (k == 0 || 2 * k == n2) { a_i = 0.0; b_i = 0.0; }
          /* Z = H0 + i H1 */
          r0[(size_t)k * VB + b] = a_r - b_i;
          i0[(size_t)k * VB + b] = a_i + b_r;
        }
      }
      const int fl = vlines(&p, +1, r0, i0, r1, i1);
      const double* zr = fl ? r1 : r0;
      const double* zi = fl ? i1 : i0;
      for (int b = 0; b < nb; ++b) {
        const long c = c0 + b;
        double* x0 = out + (2 * c) * (long)n2;
        double* x1 = (2 * c + 1 < rows) ? out + (2 * c + 1) * (long)n2 : NULL;
        for (int t = 0; t < n2; ++t) x0[t] = zr[(size_t)t * VB + b];
        if (x1)
          for (int t = 0; t < n2; ++t) x1[t] = zi[(size_t)t * VB + b];
      }
    }
    free(buf);
  }
  vplan_free(&p);
  return 0;
}
