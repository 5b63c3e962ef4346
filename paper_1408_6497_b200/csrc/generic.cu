// generic.cu — mixed-radix path for any n >= 2 (the reference accepts any
// n, grid.hpp:18; its own tests solve at n = 12 and transform at n = 6, 10,
// test_fft.cpp:45,77,136).  Not the benchmarked path: up to 8 adjacent lines
// per CTA staged in shared memory (so the strided y / x passes load and store
// 128-byte rows), Stockham stages with compile-time radix-2/3/4/5/7/8
// butterflies (constant twiddles) and a direct O(R) sum for larger prime
// factors; every n >= 2 is handled.  Five sweeps: the x pass runs forward *
// symbol * backward in one kernel (G_XPOISSON), the z passes transform two real
// rows per complex line (G_R2C_PAIR / G_C2R_PAIR).  B200, fp64: 384^3 in 3.9 ms,
// 768^3 in 28 ms, 1000^3 in 61 ms (seven sweeps, table twiddles, one row per
// line: 6.8 / 83 / 156 ms; the power-of-two path: 1024^3 in 16.4 ms).  Sizes
// n = 3 * 2^k and 5 * 2^k only use the z passes here: their y / x passes run on
// the power-of-two kernels through the radix-3 / radix-5 split (poisson_split3.cuh).
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

// G_XPOISSON: the x pass of the solve in one sweep — forward stages, the
// Poisson symbol of fft_solver.cpp:66-79, backward stages (as K3 of the
// power-of-two path), so the solve is five sweeps instead of seven.
// G_R2C_PAIR / G_C2R_PAIR: the solve's z passes with two real rows packed into
// one complex line (row 2q in the real part, row 2q+1 in the imaginary part), so
// one n-point complex FFT serves two rows; the Hermitian split / merge happens on
// the way out / in.
enum GenMode { G_R2C = 0, G_C2R = 1, G_C2C = 2, G_R2C_FULL = 3, G_C2C_TO_REAL = 4, G_XPOISSON = 5,
               G_R2C_PAIR = 6, G_C2R_PAIR = 7 };

// cos / sin(2 pi m / R), 0 <= m < R, for the odd radices with compile-time
// butterflies (literal constants: folded once the loops are unrolled).
template <int R>
__host__ __device__ constexpr double cosR(int m) {
  if (R == 3) return m == 0 ? 1.0 : -0.5;
  if (R == 5) return m == 0 ? 1.0 : (m == 1 || m == 4) ? 0.30901699437494745 : -0.8090169943749475;
  return m == 0 ? 1.0 : (m == 1 || m == 6) ? 0.6234898018587336 : (m == 2 || m == 5) ? -0.22252093395631434 : -0.9009688679024191;
}
template <int R>
__host__ __device__ constexpr double sinR(int m) {
  if (R == 3) return m == 0 ? 0.0 : m == 1 ? 0.8660254037844386 : -0.8660254037844386;
  if (R == 5) {
    const double s1 = 0.9510565162951535, s2 = 0.5877852522924731;
    return m == 0 ? 0.0 : m == 1 ? s1 : m == 2 ? s2 : m == 3 ? -s2 : -s1;
  }
  const double s1 = 0.7818314824680298, s2 = 0.9749279121818236, s3 = 0.4338837391175582;
  return m == 0 ? 0.0 : m == 1 ? s1 : m == 2 ? s2 : m == 3 ? s3 : m == 4 ? -s3 : m == 5 ? -s2 : -s1;
}

// R-point DFT of a[] in registers, sign S, every twiddle a compile-time constant:
// the power-of-two radices by the engine's Dft, 3 / 5 / 7 by the direct sum.
template <typename T, int R, int S>
__device__ __forceinline__ void small_dft(vec2_t<T> (&a)[R]) {
  using V = vec2_t<T>;
  if constexpr ((R & (R - 1)) == 0) {
    Dft<R, S>::run(a);
  } else {
    V o[R];
#pragma unroll
    for (int s2 = 0; s2 < R; ++s2) {
      T re = a[0].x, im = a[0].y;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        // a * exp(S 2 pi i m / R) = a * (c + i sn), c = cos, sn = S sin (m = r s2 mod R)
        const T c = T(cosR<R>((r * s2) % R)), sn = T(S * sinR<R>((r * s2) % R));
        re = fma(a[r].x, c, fma(-a[r].y, sn, re));
        im = fma(a[r].y, c, fma(a[r].x, sn, im));
      }
      o[s2] = V{re, im};
    }
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = o[r];
  }
}

// Line q -> (a, b) = (q / cnt_b, q % cnt_b); element x of the line at
// base + a*sa + b*sb + x*es.  Lines with b >= valid_b are skipped.
struct GenGeom {
  long long sa, sb, es;    // input geometry (elements of the input type)
  long long osa, osb, oes; // output geometry
  int cnt_b, valid_b;
};

// W_n^e for 0 <= e < n (conjugated for the backward sign).
template <typename T>
__device__ __forceinline__ vec2_t<T> twi(const vec2_t<T>* __restrict__ tw, int e, int sign) {
  vec2_t<T> w = __ldg(tw + e);
  if (sign > 0) w.y = -w.y;
  return w;
}

// One Stockham radix-R stage over the L lines of the tile ([x][line] layout):
// butterfly j = grp*NS + jj reads inputs j + r*n/R, multiplies input r by
// W_{NS R}^{r jj} and writes the R-point DFT to grp*NS*R + jj + s*NS.
template <typename T, int R>
__device__ __forceinline__ void gen_stage_bfly(const vec2_t<T>* b0, vec2_t<T>* b1, int L, int n, int NS,
                                               const vec2_t<T>* __restrict__ tw, int sign) {
  using V = vec2_t<T>;
  const int NSR = NS * R, nR = n / R, tstep = n / NSR;
  for (int idx = threadIdx.x; idx < L * nR; idx += blockDim.x) {
    const int l = idx % L, j = idx / L;
    const int grp = j / NS, jj = j - grp * NS;
    V a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      V x = b0[(j + r * nR) * L + l];
      if (r > 0 && jj > 0) {
        const V w = twi<T>(tw, r * jj * tstep, sign);
        x = V{x.x * w.x - x.y * w.y, x.x * w.y + x.y * w.x};
      }
      a[r] = x;
    }
    if (sign < 0) small_dft<T, R, -1>(a);
    else small_dft<T, R, +1>(a);
    const int obase = grp * NSR + jj;
#pragma unroll
    for (int s2 = 0; s2 < R; ++s2) b1[(obase + s2 * NS) * L + l] = a[s2];
  }
}

// Any radix (large prime factors): one output per thread, inputs from shared memory.
template <typename T>
__device__ __forceinline__ void gen_stage_direct(const vec2_t<T>* b0, vec2_t<T>* b1, int L, int n, int NS, int R,
                                                 const vec2_t<T>* __restrict__ tw, int sign) {
  using V = vec2_t<T>;
  const int NSR = NS * R, nR = n / R, tstep = n / NSR;
  for (int idx = threadIdx.x; idx < L * n; idx += blockDim.x) {
    const int l = idx % L, o = idx / L;
    const int grp = o / NSR, rem = o - grp * NSR, s2 = rem / NS, jj = rem - s2 * NS;
    const int j = grp * NS + jj, es = jj + s2 * NS;
    T re = 0, im = 0;
    int e = 0;  // (r * es) mod NSR
    for (int r = 0; r < R; ++r) {
      const V x = b0[(j + r * nR) * L + l];
      const V w = twi<T>(tw, e * tstep, sign);
      re = fma(x.x, w.x, fma(-x.y, w.y, re));
      im = fma(x.x, w.y, fma(x.y, w.x, im));
      e += es;
      if (e >= NSR) e -= NSR;
    }
    b1[o * L + l] = V{re, im};
  }
}

// L lines per CTA (lines q0 .. q0+L-1, consecutive b: adjacent k for the y / x
// passes, so every x row of the tile is one contiguous L*16-byte segment and the
// strided loads coalesce).  Shared memory holds two L x n buffers laid out
// [x][line] (line fastest: a warp's accesses are contiguous).  Each stage is a
// Stockham radix-R step: butterfly j = grp*NS + jj takes inputs j + r*n/R,
// multiplies input r by W_{NS R}^{r jj}, runs a direct R-point DFT and writes
// outputs grp*NS*R + jj + s*NS.
template <typename T, int MODE>
__global__ void k_gen_lines(const void* in, void* out, GenPlan pl, GenGeom g,
                            const vec2_t<T>* __restrict__ tw, int sign, int nc, T out_scale, int L, long long nlines) {
  using V = vec2_t<T>;
  extern __shared__ __align__(16) unsigned char gen_smem_raw[];
  V* b0 = reinterpret_cast<V*>(gen_smem_raw);
  V* b1 = b0 + size_t(L) * pl.n;
  const int n = pl.n;
  const long long q0 = (long long)blockIdx.x * L;
  const bool lfast = g.es != 1;  // strided axis: adjacent threads take adjacent lines
  auto line_ok = [&](int l) {
    const long long q = q0 + l;
    return q < nlines && (q % g.cnt_b) < g.valid_b;
  };
  auto in_base = [&](int l) {
    const long long q = q0 + l;
    return (q / g.cnt_b) * g.sa + (q % g.cnt_b) * g.sb;
  };
  auto out_base = [&](int l) {
    const long long q = q0 + l;
    return (q / g.cnt_b) * g.osa + (q % g.cnt_b) * g.osb;
  };
  // element idx of an (L x cnt) sweep -> (line, position)
  auto split = [&](int idx, int cnt, int& l, int& x) {
    if (lfast) {
      l = idx % L;
      x = idx / L;
    } else {
      x = idx % cnt;
      l = idx / cnt;
    }
  };

  // pair modes: line l packs rows 2q and 2q+1 (q = q0 + l); nlines counts rows, cnt_b == 1
  auto row_ok = [&](long long r) { return r < nlines; };

  // ---- load
  if constexpr (MODE == G_R2C_PAIR) {
    const T* src = static_cast<const T*>(in);
    for (int idx = threadIdx.x; idx < L * n; idx += blockDim.x) {
      int l, x;
      split(idx, n, l, x);
      const long long ra = 2 * (q0 + l), rb = ra + 1;
      b0[x * L + l] = V{row_ok(ra) ? src[ra * g.sa + x] : T(0), row_ok(rb) ? src[rb * g.sa + x] : T(0)};
    }
  } else if constexpr (MODE == G_C2R_PAIR) {
    const V* src = static_cast<const V*>(in);
    for (int idx = threadIdx.x; idx < L * nc; idx += blockDim.x) {
      int l, k;
      split(idx, nc, l, k);
      const long long ra = 2 * (q0 + l), rb = ra + 1;
      V A = row_ok(ra) ? src[ra * g.sa + k] : V{T(0), T(0)};
      V B = row_ok(rb) ? src[rb * g.sa + k] : V{T(0), T(0)};
      if (k == 0 || 2 * k == n) {  // self-conjugate modes: imaginary parts ignored
        A.y = T(0);
        B.y = T(0);
      }
      b0[k * L + l] = V{A.x - B.y, A.y + B.x};                                  // A + i B
      if (k > 0 && n - k != k) b0[(n - k) * L + l] = V{A.x + B.y, B.x - A.y};  // conj(A) + i conj(B)
    }
  } else if (MODE == G_C2R) {
    const V* src = static_cast<const V*>(in);
    for (int idx = threadIdx.x; idx < L * nc; idx += blockDim.x) {
      int l, k;
      split(idx, nc, l, k);
      V h = line_ok(l) ? src[in_base(l) + k * g.es] : V{T(0), T(0)};
      if (k == 0 || 2 * k == n) h.y = T(0);  // self-conjugate modes: imaginary part ignored
      b0[k * L + l] = h;
      if (k > 0 && n - k != k) b0[(n - k) * L + l] = V{h.x, -h.y};
    }
  } else {
    for (int idx = threadIdx.x; idx < L * n; idx += blockDim.x) {
      int l, x;
      split(idx, n, l, x);
      V v{T(0), T(0)};
      if (line_ok(l)) {
        if (MODE == G_R2C || MODE == G_R2C_FULL) v = V{static_cast<const T*>(in)[in_base(l) + x * g.es], T(0)};
        else v = static_cast<const V*>(in)[in_base(l) + x * g.es];
      }
      b0[x * L + l] = v;
    }
  }
  __syncthreads();

  // ---- Stockham stages (result in b0)
  auto stages = [&](int sgn) {
    int NS = 1;
    for (int st = 0; st < pl.nst; ++st) {
      const int R = pl.radix[st];
      switch (R) {
        case 2: gen_stage_bfly<T, 2>(b0, b1, L, n, NS, tw, sgn); break;
        case 3: gen_stage_bfly<T, 3>(b0, b1, L, n, NS, tw, sgn); break;
        case 4: gen_stage_bfly<T, 4>(b0, b1, L, n, NS, tw, sgn); break;
        case 5: gen_stage_bfly<T, 5>(b0, b1, L, n, NS, tw, sgn); break;
        case 7: gen_stage_bfly<T, 7>(b0, b1, L, n, NS, tw, sgn); break;
        case 8: gen_stage_bfly<T, 8>(b0, b1, L, n, NS, tw, sgn); break;
        default: gen_stage_direct<T>(b0, b1, L, n, NS, R, tw, sgn); break;
      }
      __syncthreads();
      V* t = b0;
      b0 = b1;
      b1 = t;
      NS *= R;
    }
  };
  if constexpr (MODE == G_XPOISSON) {
    // line q = (j, k) of the x pass (geometry gx: a = j, b = k); position x = i
    stages(-1);
    const T four_pi2 = T(4.0 * M_PI * M_PI);  // fft_solver.cpp:66
    for (int idx = threadIdx.x; idx < L * n; idx += blockDim.x) {
      int l, x;
      split(idx, n, l, x);
      const long long q = q0 + l;
      const int j = int(q / g.cnt_b), k = int(q % g.cnt_b);
      const T ki = T(x <= n / 2 ? x : x - n), kj = T(j <= n / 2 ? j : j - n), kk = T(k);
      const T k2 = ki * ki + kj * kj + kk * kk;
      const T m = (k2 == T(0)) ? T(0) : out_scale / (four_pi2 * k2);  // out_scale = 1/n^3
      V& v = b0[x * L + l];
      v.x *= m;
      v.y *= m;
    }
    __syncthreads();
    stages(+1);
  } else {
    stages(sign);
  }

  // ---- store
  if constexpr (MODE == G_R2C_PAIR) {
    V* dst = static_cast<V*>(out);
    for (int idx = threadIdx.x; idx < L * nc; idx += blockDim.x) {
      int l, k;
      split(idx, nc, l, k);
      const long long ra = 2 * (q0 + l), rb = ra + 1;
      const V Z = b0[k * L + l], Zm = b0[((n - k) % n) * L + l];
      // row a: (Z + conj(Zm)) / 2, row b: (Z - conj(Zm)) / 2i
      if (row_ok(ra)) dst[ra * g.osa + k] = V{T(0.5) * (Z.x + Zm.x), T(0.5) * (Z.y - Zm.y)};
      if (row_ok(rb)) dst[rb * g.osa + k] = V{T(0.5) * (Z.y + Zm.y), T(0.5) * (Zm.x - Z.x)};
    }
    return;
  }
  if constexpr (MODE == G_C2R_PAIR) {
    T* dst = static_cast<T*>(out);
    for (int idx = threadIdx.x; idx < L * n; idx += blockDim.x) {
      int l, x;
      split(idx, n, l, x);
      const long long ra = 2 * (q0 + l), rb = ra + 1;
      const V v = b0[x * L + l];
      if (row_ok(ra)) dst[ra * g.osa + x] = v.x * out_scale;
      if (row_ok(rb)) dst[rb * g.osa + x] = v.y * out_scale;
    }
    return;
  }
  const int cnt = MODE == G_R2C ? nc : n;
  for (int idx = threadIdx.x; idx < L * cnt; idx += blockDim.x) {
    int l, x;
    split(idx, cnt, l, x);
    if (!line_ok(l)) continue;
    const V v = b0[x * L + l];
    if (MODE == G_C2R || MODE == G_C2C_TO_REAL) static_cast<T*>(out)[out_base(l) + x * g.oes] = v.x * out_scale;
    else if (MODE == G_XPOISSON) static_cast<V*>(out)[out_base(l) + x * g.oes] = v;
    else static_cast<V*>(out)[out_base(l) + x * g.oes] = v;
  }
}

// Lines per CTA.  Strided passes (es != 1): up to 8 adjacent lines (128-byte
// rows) within ~100 KB so two CTAs share an SM, else fewer; contiguous passes:
// rows are contiguous anyway, so at most 2 lines within ~48 KB (four CTAs per
// SM hide the load latency).  B200, 768^3: 83 ms with 8 lines everywhere.
#ifndef ARENA_GEN_ZCAP
#define ARENA_GEN_ZCAP (96 * 1024)  // shared-memory budget of a contiguous-axis CTA (B200 1000^3:
#endif                              // z passes 10.6 -> 8.5 ms with 96 KB instead of 48 KB)
inline int gen_lines_per_cta(int n, int vb, bool strided) {
  // contiguous axis: 4 lines (row pairs) up to n = 512, else 2 (B200: 384^3 z 0.56 -> 0.46 ms
  // with 4; 768^3 z 3.7 -> 4.5 ms with 4)
  int L = strided ? 8 : (n <= 512 ? 4 : 2);
  const size_t cap = strided ? 100 * 1024 : ARENA_GEN_ZCAP;
  while (L > 1 && size_t(2) * n * L * vb > cap) L /= 2;
  return L;
}

template <typename T, int MODE>
cudaError_t run_lines(const GenArgs& a, const void* in, void* out, long long nlines, const GenGeom& g, int sign,
                      T out_scale) {
  const int vb = int(2 * sizeof(T));
  const int L = gen_lines_per_cta(a.n, vb, g.es != 1);
  const size_t smem = size_t(2) * a.n * L * vb;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    cudaError_t e = cudaFuncSetAttribute(k_gen_lines<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr_done[dev & 63] = true;
  }
  const long long units = (MODE == G_R2C_PAIR || MODE == G_C2R_PAIR) ? (nlines + 1) / 2 : nlines;  // pairs of rows
  const long long blocks = (units + L - 1) / L;
  k_gen_lines<T, MODE><<<unsigned(blocks), 256, smem, a.stream>>>(
      in, out, *a.plan, g, static_cast<const vec2_t<T>*>(a.tw), sign, a.nc, out_scale, L, nlines);
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
  e = run_lines<T, G_R2C_PAIR>(a, f, spec, nn, GenGeom{n, 0, 1, ncp, 0, 1, 1, 1}, -1, T(1));
  if (e) return e;
  // y c2c forward: lines (i, k), element j at i*n*ncp + k + j*ncp
  GenGeom gy{(long long)n * ncp, 1, ncp, (long long)n * ncp, 1, ncp, ncp, nc};
  gmark(a, 1);
  if ((e = run_lines<T, G_C2C>(a, spec, spec, (long long)n * ncp, gy, -1, T(1)))) return e;
  // x c2c forward: lines (j, k), element i at j*ncp + k + i*n*ncp
  GenGeom gx{ncp, 1, (long long)n * ncp, ncp, 1, (long long)n * ncp, ncp, nc};
  // x: forward * Poisson symbol (fft_solver.cpp:66-79) * backward, one sweep
  gmark(a, 2);
  if ((e = run_lines<T, G_XPOISSON>(a, spec, spec, (long long)n * ncp, gx, -1, T(1.0 / (double(n) * n * n)))))
    return e;
  gmark(a, 3);
  if ((e = run_lines<T, G_C2C>(a, spec, spec, (long long)n * ncp, gy, +1, T(1)))) return e;
  // z c2r: rows of S -> rows of u
  gmark(a, 4);
  e = run_lines<T, G_C2R_PAIR>(a, spec, u, nn, GenGeom{ncp, 0, 1, n, 0, 1, 1, 1}, +1, T(1));
  gmark(a, 5);
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
  // radix 8, then 4, then 2, then odd primes ascending
  while (m % 8 == 0 && p->nst < kGenMaxStages) { p->radix[p->nst++] = 8; m /= 8; }
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

// The solve's z passes alone (the radix-3 split path runs its own y / x passes).
template <typename T>
cudaError_t gen_z_r2c(const GenArgs& a, const void* f, void* spec) {
  const long long nn = (long long)a.n * a.n;
  return run_lines<T, G_R2C_PAIR>(a, f, spec, nn, GenGeom{a.n, 0, 1, a.ncp, 0, 1, 1, 1}, -1, T(1));
}
template <typename T>
cudaError_t gen_z_c2r(const GenArgs& a, const void* spec, void* u) {
  const long long nn = (long long)a.n * a.n;
  return run_lines<T, G_C2R_PAIR>(a, spec, u, nn, GenGeom{a.ncp, 0, 1, a.n, 0, 1, 1, 1}, +1, T(1));
}
cudaError_t gen_z_r2c_f64(const GenArgs& a, const void* f, void* spec) { return gen_z_r2c<double>(a, f, spec); }
cudaError_t gen_z_r2c_f32(const GenArgs& a, const void* f, void* spec) { return gen_z_r2c<float>(a, f, spec); }
cudaError_t gen_z_c2r_f64(const GenArgs& a, const void* spec, void* u) { return gen_z_c2r<double>(a, spec, u); }
cudaError_t gen_z_c2r_f32(const GenArgs& a, const void* spec, void* u) { return gen_z_c2r<float>(a, spec, u); }

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
