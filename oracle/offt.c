/*
 * offt.c — CPU restatement (TEST INFRASTRUCTURE ONLY; see offt.h for the
 * contract, the reference lines restated and how it is pinned).
 *
 * Recursive mixed-radix decimation-in-time Cooley-Tukey.  Twiddles are
 * computed once per length in 80-bit long double and rounded to double.
 */
#include "offt.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  double re, im;
} cplx;

static int g_threads = 0;

void offt_set_threads(int nthreads) { g_threads = nthreads; }

int offt_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

/* ------------------------------------------------------------------ plan */

typedef struct {
  int n;
  int nf;
  int fac[64];
  cplx* tw; /* W_n^m = exp(-2 pi i m / n), m in [0, n) */
} plan1d;

static int plan_init(plan1d* p, int n) {
  if (n < 1) return -1;
  p->n = n;
  p->nf = 0;
  int m = n;
  while (m % 4 == 0) { p->fac[p->nf++] = 4; m /= 4; }
  while (m % 2 == 0) { p->fac[p->nf++] = 2; m /= 2; }
  for (int q = 3; m > 1; q += 2) {
    while (m % q == 0) { p->fac[p->nf++] = q; m /= q; }
    if ((long)q * q > m && m > 1) { p->fac[p->nf++] = m; m = 1; }
  }
  if (p->nf == 0) p->fac[p->nf++] = 1;
  p->tw = (cplx*)malloc(sizeof(cplx) * (size_t)n);
  if (!p->tw) return -1;
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int k = 0; k < n; ++k) {
    const long double a = two_pi * (long double)k / (long double)n;
    p->tw[k].re = (double)cosl(a);
    p->tw[k].im = (double)-sinl(a);
  }
  return 0;
}

static void plan_free(plan1d* p) {
  free(p->tw);
  p->tw = NULL;
}

static inline cplx cmul(cplx a, cplx b) {
  cplx r = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return r;
}

/* twiddle W_N^e with the requested sign (-1 forward, +1 backward) */
static inline cplx twid(const cplx* tw, int N, long e, int sign) {
  cplx w = tw[e % N];
  if (sign > 0) w.im = -w.im;
  return w;
}

/* in-place DFT of a[0..R) (R small), sign -1/+1 */
static void small_dft(cplx* a, int R, const cplx* tw, int N, int sign) {
  if (R == 1) return;
  if (R == 2) {
    cplx t = a[1];
    a[1].re = a[0].re - t.re; a[1].im = a[0].im - t.im;
    a[0].re += t.re; a[0].im += t.im;
    return;
  }
  if (R == 4) {
    cplx s02 = {a[0].re + a[2].re, a[0].im + a[2].im};
    cplx d02 = {a[0].re - a[2].re, a[0].im - a[2].im};
    cplx s13 = {a[1].re + a[3].re, a[1].im + a[3].im};
    cplx d13 = {a[1].re - a[3].re, a[1].im - a[3].im};
    /* forward: y1 = d02 - i d13 ; backward: y1 = d02 + i d13 */
    /* jd = (sign * i) * d13 = sign * (-y + i x) */
    cplx jd = {sign * -d13.im, sign * d13.re};
    a[0].re = s02.re + s13.re; a[0].im = s02.im + s13.im;
    a[2].re = s02.re - s13.re; a[2].im = s02.im - s13.im;
    a[1].re = d02.re + jd.re; a[1].im = d02.im + jd.im;
    a[3].re = d02.re - jd.re; a[3].im = d02.im - jd.im;
    return;
  }
  /* generic O(R^2) DFT using the length-N table (R divides N) */
  cplx tmp[64];
  cplx* t = R <= 64 ? tmp : (cplx*)malloc(sizeof(cplx) * (size_t)R);
  const int step = N / R;
  for (int s = 0; s < R; ++s) {
    double re = 0, im = 0;
    for (int r = 0; r < R; ++r) {
      cplx w = twid(tw, N, (long)((long)r * s % R) * step, sign);
      re += a[r].re * w.re - a[r].im * w.im;
      im += a[r].re * w.im + a[r].im * w.re;
    }
    t[s].re = re;
    t[s].im = im;
  }
  memcpy(a, t, sizeof(cplx) * (size_t)R);
  if (t != tmp) free(t);
}

/* DFT of length n of in[0], in[is], ..., into out[0..n) (contiguous).
 * Twiddle table is for length N; W_n^e = tw[e * (N/n)]. */
static void rec(const cplx* in, cplx* out, int n, long is, const int* fac, const cplx* tw, int N,
                int sign) {
  const int R = fac[0];
  const int m = n / R;
  if (m == 1) {
    cplx a[64];
    cplx* b = R <= 64 ? a : (cplx*)malloc(sizeof(cplx) * (size_t)R);
    for (int r = 0; r < R; ++r) b[r] = in[r * is];
    small_dft(b, R, tw, N, sign);
    for (int s = 0; s < R; ++s) out[s] = b[s];
    if (b != a) free(b);
    return;
  }
  for (int r = 0; r < R; ++r) rec(in + r * is, out + (long)r * m, m, is * R, fac + 1, tw, N, sign);
  const int step = N / n;
  cplx a[64];
  cplx* b = R <= 64 ? a : (cplx*)malloc(sizeof(cplx) * (size_t)R);
  for (int k = 0; k < m; ++k) {
    b[0] = out[k];
    for (int r = 1; r < R; ++r) b[r] = cmul(out[(long)r * m + k], twid(tw, N, (long)r * k * step, sign));
    small_dft(b, R, tw, N, sign);
    for (int s = 0; s < R; ++s) out[k + (long)s * m] = b[s];
  }
  if (b != a) free(b);
}

/* transform a contiguous line x (length p->n) in place using scratch y */
static void line_fft(const plan1d* p, cplx* x, cplx* y, int sign) {
  rec(x, y, p->n, 1, p->fac, p->tw, p->n, sign);
  memcpy(x, y, sizeof(cplx) * (size_t)p->n);
}

int offt_c2c_1d(int n, double* x, int sign) {
  plan1d p;
  if (plan_init(&p, n)) return -1;
  cplx* y = (cplx*)malloc(sizeof(cplx) * (size_t)n);
  if (!y) { plan_free(&p); return -1; }
  line_fft(&p, (cplx*)x, y, sign);
  free(y);
  plan_free(&p);
  return 0;
}

/* Transform every line of a strided axis.  The array is viewed as
 * [outer][len][inner] complex; lines run along `len`.  Lines that are adjacent
 * in `inner` are gathered in blocks of 8 for cache-friendly access. */
static void axis_fft(cplx* a, long outer, int len, long inner, int sign) {
  plan1d p;
  if (plan_init(&p, len)) return;
  const int B = inner >= 8 ? 8 : (int)inner;
  const long nblk_inner = (inner + B - 1) / B;
  const long nwork = outer * nblk_inner;
#pragma omp parallel num_threads(offt_get_threads())
  {
    cplx* buf = (cplx*)malloc(sizeof(cplx) * (size_t)len * (size_t)(B + 1));
    cplx* scratch = buf + (size_t)len * B;
#pragma omp for schedule(static)
    for (long w = 0; w < nwork; ++w) {
      const long o = w / nblk_inner;
      const long i0 = (w % nblk_inner) * B;
      const int nb = (int)((inner - i0) < B ? (inner - i0) : B);
      cplx* base = a + o * (long)len * inner + i0;
      for (int t = 0; t < len; ++t)
        for (int b = 0; b < nb; ++b) buf[(size_t)b * len + t] = base[(long)t * inner + b];
      for (int b = 0; b < nb; ++b) line_fft(&p, buf + (size_t)b * len, scratch, sign);
      for (int t = 0; t < len; ++t)
        for (int b = 0; b < nb; ++b) base[(long)t * inner + b] = buf[(size_t)b * len + t];
    }
    free(buf);
  }
  plan_free(&p);
}

int offt_c2c_3d(int n0, int n1, int n2, const double* in, double* out, int sign) {
  const size_t N = (size_t)n0 * n1 * n2;
  if (out != in) memcpy(out, in, sizeof(cplx) * N);
  cplx* a = (cplx*)out;
  axis_fft(a, (long)n0 * n1, n2, 1, sign);
  axis_fft(a, n0, n1, n2, sign);
  axis_fft(a, 1, n0, (long)n1 * n2, sign);
  return 0;
}

int offt_r2c_3d(int n0, int n1, int n2, const double* in, double* out) {
  const int nc = n2 / 2 + 1;
  cplx* a = (cplx*)out;
  plan1d p;
  if (plan_init(&p, n2)) return -1;
  const long rows = (long)n0 * n1;
#pragma omp parallel num_threads(offt_get_threads())
  {
    cplx* x = (cplx*)malloc(sizeof(cplx) * (size_t)n2 * 2);
    cplx* y = x + n2;
#pragma omp for schedule(static)
    for (long r = 0; r < rows; ++r) {
      for (int k = 0; k < n2; ++k) { x[k].re = in[r * n2 + k]; x[k].im = 0.0; }
      line_fft(&p, x, y, -1);
      memcpy(a + r * nc, x, sizeof(cplx) * (size_t)nc);
    }
    free(x);
  }
  plan_free(&p);
  axis_fft(a, n0, n1, nc, -1);
  axis_fft(a, 1, n0, (long)n1 * nc, -1);
  return 0;
}

int offt_c2r_3d(int n0, int n1, int n2, double* in, double* out) {
  const int nc = n2 / 2 + 1;
  cplx* a = (cplx*)in;
  axis_fft(a, 1, n0, (long)n1 * nc, +1);
  axis_fft(a, n0, n1, nc, +1);
  plan1d p;
  if (plan_init(&p, n2)) return -1;
  const long rows = (long)n0 * n1;
#pragma omp parallel num_threads(offt_get_threads())
  {
    cplx* x = (cplx*)malloc(sizeof(cplx) * (size_t)n2 * 2);
    cplx* y = x + n2;
#pragma omp for schedule(static)
    for (long r = 0; r < rows; ++r) {
      const cplx* h = a + r * nc;
      for (int k = 0; k < nc; ++k) x[k] = h[k];
      for (int k = nc; k < n2; ++k) { x[k].re = h[n2 - k].re; x[k].im = -h[n2 - k].im; }
      x[0].im = 0.0;                          /* self-conjugate modes: imaginary part ignored */
      if (n2 % 2 == 0) x[n2 / 2].im = 0.0;
      line_fft(&p, x, y, +1);
      for (int k = 0; k < n2; ++k) out[r * n2 + k] = x[k].re;
    }
    free(x);
  }
  plan_free(&p);
  return 0;
}

static inline int signed_freq(int k, int n) { return k <= n / 2 ? k : k - n; } /* fft_solver.hpp:19 */

int offt_poisson_solve(int n, const double* f, double* u) {
  if (n < 2) return -1; /* GridField(n) throws for n < 2, grid.hpp:18 */
  const int nc = n / 2 + 1;
  const size_t ns = (size_t)n * n * nc;
  double* spec = (double*)malloc(sizeof(double) * 2 * ns);
  if (!spec) return -1;
  offt_r2c_3d(n, n, n, f, spec); /* fft_solver.cpp:60-61,65 */
  const double four_pi2 = 4.0 * M_PI * M_PI; /* fft_solver.cpp:66 */
  const double scale = 1.0 / ((double)n * n * n);
#pragma omp parallel for num_threads(offt_get_threads()) schedule(static)
  for (int i = 0; i < n; ++i) {
    const double ki = signed_freq(i, n);
    for (int j = 0; j < n; ++j) {
      const double kj = signed_freq(j, n);
      for (int k = 0; k < nc; ++k) {
        const double kk = k;
        const size_t idx = ((size_t)i * n + j) * nc + k;
        const double k2 = ki * ki + kj * kj + kk * kk;
        const double s = (k2 == 0.0) ? 0.0 : scale / (four_pi2 * k2); /* fft_solver.cpp:76 */
        spec[2 * idx] *= s;
        spec[2 * idx + 1] *= s;
      }
    }
  }
  offt_c2r_3d(n, n, n, spec, u); /* fft_solver.cpp:62-63,80 */
  free(spec);
  return 0;
}

int offt_dft3_forward(int n, const double* g, double* spec) {
  const size_t N = (size_t)n * n * n;
  for (size_t i = 0; i < N; ++i) { spec[2 * i] = g[i]; spec[2 * i + 1] = 0.0; } /* fft_solver.cpp:16 */
  return offt_c2c_3d(n, n, n, spec, spec, -1);
}

int offt_dft3_inverse(int n, const double* spec, double* g) {
  const size_t N = (size_t)n * n * n;
  double* tmp = (double*)malloc(sizeof(double) * 2 * N);
  if (!tmp) return -1;
  offt_c2c_3d(n, n, n, spec, tmp, +1);
  const double scale = 1.0 / (double)N; /* fft_solver.cpp:46-47 */
  for (size_t i = 0; i < N; ++i) g[i] = tmp[2 * i] * scale;
  free(tmp);
  return 0;
}
