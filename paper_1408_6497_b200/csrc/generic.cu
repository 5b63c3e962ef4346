// generic.cu — mixed-radix path for any n >= 2 (the reference accepts any
// n, grid.hpp:18; its own tests solve at n = 12 and transform at n = 6, 10,
// test_fft.cpp:45,77,136).  Not the benchmarked path: one CTA per line, the
// line staged in shared memory, Stockham stages whose butterflies are direct
// O(R) sums with the stage twiddle folded into one exact table index, so every
// factor of n (2, 3, 5, 7, any prime) is handled by the same code.
//
// Same conventions as fft_solver.cpp: r2c along the last axis keeping
// k in [0, n/2], c2r treating its input as Hermitian (imaginary parts of the
// self-conjugate modes ignored), the Poisson symbol of fft_solver.cpp:66-79.
#include <cuda_runtime.h>

#include <cmath>

#include "fft_engine.cuh"
#include "launchers.h"

namespace arena_fft {

namespace {

enum GenMode { G_R2C = 0, G_C2R = 1, G_C2C = 2, G_R2C_FULL = 3, G_C2C_TO_REAL = 4 };

// Line q -> (a, b) = (q / cnt_b, q % cnt_b); element x of the line at
// base + a*sa + b*sb + x*es.  Lines with b >= valid_b are skipped.
struct GenGeom {
  long long sa, sb, es;    // input geometry (elements of the input type)
  long long osa, osb, oes; // output geometry
  int cnt_b, valid_b;
};

template <typename T>
__device__ __forceinline__ vec2_t<T> twn(const vec2_t<T>* __restrict__ tw, long long e, int n, int sign) {
  vec2_t<T> w = __ldg(tw + (e % n));
  if (sign > 0) w.y = -w.y;
  return w;
}

template <typename T, int MODE>
__global__ void k_gen_lines(const void* in, void* out, GenPlan pl, GenGeom g,
                            const vec2_t<T>* __restrict__ tw, int sign, int nc, T out_scale) {
  using V = vec2_t<T>;
  extern __shared__ __align__(16) unsigned char gen_smem_raw[];
  V* b0 = reinterpret_cast<V*>(gen_smem_raw);
  V* b1 = b0 + pl.n;
  const int n = pl.n;
  const long long q = blockIdx.x;
  const long long a = q / g.cnt_b, b = q % g.cnt_b;
  if (b >= g.valid_b) return;  // whole block: no barrier skipped by a subset
  const long long ib = a * g.sa + b * g.sb, ob = a * g.osa + b * g.osb;

  // ---- load
  if (MODE == G_R2C || MODE == G_R2C_FULL) {
    const T* src = static_cast<const T*>(in) + ib;
    for (int x = threadIdx.x; x < n; x += blockDim.x) b0[x] = V{src[x * g.es], T(0)};
  } else if (MODE == G_C2R) {
    const V* src = static_cast<const V*>(in) + ib;
    for (int k = threadIdx.x; k < nc; k += blockDim.x) {
      V h = src[k * g.es];
      if (k == 0 || 2 * k == n) h.y = T(0);  // self-conjugate modes: imaginary part ignored
      b0[k] = h;
      if (k > 0 && n - k != k) b0[n - k] = V{h.x, -h.y};
    }
  } else {
    const V* src = static_cast<const V*>(in) + ib;
    for (int x = threadIdx.x; x < n; x += blockDim.x) b0[x] = src[x * g.es];
  }
  __syncthreads();

  // ---- Stockham stages: out[grp*NS*R + jj + s*NS] = sum_r in[j + r*n/R] W^{r (jj + s NS)} on the NS*R grid
  int NS = 1;
  for (int st = 0; st < pl.nst; ++st) {
    const int R = pl.radix[st];
    const int NSR = NS * R, nR = n / R, step = n / NSR;
    for (int o = threadIdx.x; o < n; o += blockDim.x) {
      const int jj = o % NS, s = (o % NSR) / NS, grp = o / NSR;
      const int j = grp * NS + jj;
      const int es = jj + s * NS;
      T re = 0, im = 0;
      for (int r = 0; r < R; ++r) {
        const V x = b0[j + r * nR];
        const V w = twn<T>(tw, (long long)((long long)r * es % NSR) * step, n, sign);
        re = fma(x.x, w.x, fma(-x.y, w.y, re));
        im = fma(x.x, w.y, fma(x.y, w.x, im));
      }
      b1[o] = V{re, im};
    }
    __syncthreads();
    V* t = b0;
    b0 = b1;
    b1 = t;
    NS = NSR;
  }

  // ---- store
  if (MODE == G_R2C) {
    V* dst = static_cast<V*>(out) + ob;
    for (int k = threadIdx.x; k < nc; k += blockDim.x) dst[k * g.oes] = b0[k];
  } else if (MODE == G_C2R || MODE == G_C2C_TO_REAL) {
    T* dst = static_cast<T*>(out) + ob;
    for (int x = threadIdx.x; x < n; x += blockDim.x) dst[x * g.oes] = b0[x].x * out_scale;
  } else {
    V* dst = static_cast<V*>(out) + ob;
    for (int x = threadIdx.x; x < n; x += blockDim.x) dst[x * g.oes] = b0[x];
  }
}

// Poisson symbol on the half spectrum S[(i*n+j)*ncp + k], fft_solver.cpp:66-79.
template <typename T>
__global__ void k_gen_scale(vec2_t<T>* __restrict__ S, int n, int nc, int ncp, T scale, T four_pi2) {
  const long long total = (long long)n * n * nc;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int k = int(idx % nc);
    const long long ij = idx / nc;
    const int j = int(ij % n), i = int(ij / n);
    const T ki = T(i <= n / 2 ? i : i - n), kj = T(j <= n / 2 ? j : j - n), kk = T(k);
    const T k2 = ki * ki + kj * kj + kk * kk;
    const T m = (k2 == T(0)) ? T(0) : scale / (four_pi2 * k2);
    vec2_t<T>& v = S[ij * ncp + k];
    v.x *= m;
    v.y *= m;
  }
}

template <typename T, int MODE>
cudaError_t run_lines(const GenArgs& a, const void* in, void* out, long long nlines, const GenGeom& g, int sign,
                      T out_scale) {
  const size_t smem = gen_smem_bytes(a.n, int(2 * sizeof(T)));
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > 48 * 1024 && !attr_done[dev & 63]) {
    const int most = int(gen_smem_bytes(gen_max_n(int(2 * sizeof(T))), int(2 * sizeof(T))));
    cudaError_t e = cudaFuncSetAttribute(k_gen_lines<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, most);
    if (e != cudaSuccess) return e;
    attr_done[dev & 63] = true;
  }
  const int threads = a.n >= 256 ? 256 : (a.n >= 64 ? 64 : 32);
  k_gen_lines<T, MODE><<<unsigned(nlines), threads, smem, a.stream>>>(
      in, out, *a.plan, g, static_cast<const vec2_t<T>*>(a.tw), sign, a.nc, out_scale);
  return cudaGetLastError();
}

inline void gmark(const GenArgs& a, int i) {
  if (a.ev) cudaEventRecord(a.ev[i], a.stream);
}

template <typename T>
cudaError_t gen_poisson(const GenArgs& a, const void* f, void* u, void* spec) {
  const int n = a.n, nc = a.nc, ncp = a.ncp;
  const long long nn = (long long)n * n;
  cudaError_t e;
  // z r2c: rows of f -> rows of S
  gmark(a, 0);
  e = run_lines<T, G_R2C>(a, f, spec, nn, GenGeom{n, 0, 1, ncp, 0, 1, 1, 1}, -1, T(1));
  if (e) return e;
  // y c2c forward: lines (i, k), element j at i*n*ncp + k + j*ncp
  GenGeom gy{(long long)n * ncp, 1, ncp, (long long)n * ncp, 1, ncp, ncp, nc};
  gmark(a, 1);
  if ((e = run_lines<T, G_C2C>(a, spec, spec, (long long)n * ncp, gy, -1, T(1)))) return e;
  // x c2c forward: lines (j, k), element i at j*ncp + k + i*n*ncp
  GenGeom gx{ncp, 1, (long long)n * ncp, ncp, 1, (long long)n * ncp, ncp, nc};
  gmark(a, 2);
  if ((e = run_lines<T, G_C2C>(a, spec, spec, (long long)n * ncp, gx, -1, T(1)))) return e;
  gmark(a, 3);
  k_gen_scale<T><<<1184, 256, 0, a.stream>>>(static_cast<vec2_t<T>*>(spec), n, nc, ncp,
                                             T(1.0 / (double(n) * n * n)), T(4.0 * M_PI * M_PI));
  if ((e = cudaGetLastError())) return e;
  gmark(a, 4);
  if ((e = run_lines<T, G_C2C>(a, spec, spec, (long long)n * ncp, gx, +1, T(1)))) return e;
  gmark(a, 5);
  if ((e = run_lines<T, G_C2C>(a, spec, spec, (long long)n * ncp, gy, +1, T(1)))) return e;
  // z c2r: rows of S -> rows of u
  gmark(a, 6);
  e = run_lines<T, G_C2R>(a, spec, u, nn, GenGeom{ncp, 0, 1, n, 0, 1, 1, 1}, +1, T(1));
  gmark(a, 7);
  return e;
}

// Full complex n^3 array C (pitch n): c2c along y and x, in place.
template <typename T>
cudaError_t gen_c2c_yx(const GenArgs& a, void* C, int sign) {
  const long long n = a.n;
  cudaError_t e;
  GenGeom gy{n * n, 1, n, n * n, 1, n, int(n), int(n)};
  if ((e = run_lines<T, G_C2C>(a, C, C, n * n, gy, sign, T(1)))) return e;
  GenGeom gx{n, 1, n * n, n, 1, n * n, int(n), int(n)};
  return run_lines<T, G_C2C>(a, C, C, n * n, gx, sign, T(1));
}

template <typename T>
cudaError_t gen_dft3_forward(const GenArgs& a, const void* g, void* spec) {
  const long long n = a.n;
  cudaError_t e = run_lines<T, G_R2C_FULL>(a, g, spec, n * n, GenGeom{n, 0, 1, n, 0, 1, 1, 1}, -1, T(1));
  if (e) return e;
  return gen_c2c_yx<T>(a, spec, -1);
}

template <typename T>
cudaError_t gen_dft3_inverse(const GenArgs& a, const void* spec, void* g, void* work) {
  const long long n = a.n;
  cudaError_t e = cudaMemcpyAsync(work, spec, size_t(n * n * n) * 2 * sizeof(T), cudaMemcpyDeviceToDevice, a.stream);
  if (e) return e;
  if ((e = gen_c2c_yx<T>(a, work, +1))) return e;
  const T scale = T(1.0 / double(n * n * n));  // fft_solver.cpp:46
  return run_lines<T, G_C2C_TO_REAL>(a, work, g, n * n, GenGeom{n, 0, 1, n, 0, 1, 1, 1}, +1, scale);
}

}  // namespace

bool gen_plan_make(int n, GenPlan* p) {
  if (n < 2) return false;
  p->n = n;
  p->nst = 0;
  int m = n;
  // radix 4 first, then 2, then odd primes ascending
  while (m % 4 == 0 && p->nst < kGenMaxStages) { p->radix[p->nst++] = 4; m /= 4; }
  while (m % 2 == 0 && p->nst < kGenMaxStages) { p->radix[p->nst++] = 2; m /= 2; }
  for (int q = 3; m > 1 && p->nst < kGenMaxStages; q += 2) {
    while (m % q == 0 && p->nst < kGenMaxStages) { p->radix[p->nst++] = q; m /= q; }
    if ((long long)q * q > m && m > 1) { p->radix[p->nst++] = m; m = 1; }
  }
  return m == 1;
}

size_t gen_smem_bytes(int n, int elem_bytes) { return size_t(2) * n * elem_bytes; }
int gen_max_n(int elem_bytes) { return (227 * 1024) / (2 * elem_bytes); }

cudaError_t gen_poisson_f64(const GenArgs& a, const void* f, void* u, void* spec) {
  return gen_poisson<double>(a, f, u, spec);
}
cudaError_t gen_poisson_f32(const GenArgs& a, const void* f, void* u, void* spec) {
  return gen_poisson<float>(a, f, u, spec);
}
cudaError_t gen_dft3_forward_f64(const GenArgs& a, const void* g, void* spec) {
  return gen_dft3_forward<double>(a, g, spec);
}
cudaError_t gen_dft3_inverse_f64(const GenArgs& a, const void* spec, void* g, void* work) {
  return gen_dft3_inverse<double>(a, spec, g, work);
}
cudaError_t gen_dft3_forward_f32(const GenArgs& a, const void* g, void* spec) {
  return gen_dft3_forward<float>(a, g, spec);
}
cudaError_t gen_dft3_inverse_f32(const GenArgs& a, const void* spec, void* g, void* work) {
  return gen_dft3_inverse<float>(a, spec, g, work);
}

}  // namespace arena_fft
