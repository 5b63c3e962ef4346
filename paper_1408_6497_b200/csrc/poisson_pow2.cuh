// poisson_pow2.cuh — sm_100a kernels of the power-of-two spectral Poisson
// solve (the hot path of /root/reference/proj/src/fft_solver.cpp:51-87).
//
// Device layout of the half spectrum (internal; the boundary layout is the
// GridField one): S[(i*n + j)*ncp + k], k in [0, nc), nc = n/2 + 1, row pitch
// ncp = round_up(nc, 8) complex so every (i, j) row starts 128-byte aligned.
// This is the r2c layout FFTW produces at fft_solver.cpp:60-61 (index
// (i*n+j)*nc+k, fft_solver.cpp:74) with a padded row.
//
// Five kernels, one HBM sweep each:
//   K1 zfwd : f rows (k axis, contiguous)  -> S      real->half complex (r2c)
//   K2 yfwd : S lines along j (stride ncp) in place  c2c forward
//   K3 xmid : S lines along i (stride n*ncp) in place  c2c forward, Poisson
//             scale (fft_solver.cpp:66-79), c2c backward — one round trip
//   K4 yinv : as K2, backward
//   K5 zinv : S rows -> u rows              half complex->real (c2r)
// The r2c/c2r along the contiguous axis run an n/2-point complex FFT on the
// packed even/odd pairs (a double2 load of two reals) plus an O(n) split.
#pragma once

#include "fft_engine.cuh"

namespace arena_fft {

__host__ __device__ constexpr int imin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int imax(int a, int b) { return a > b ? a : b; }

// ------------------------------------------------------------ configuration
// E: points per thread; L: lines per CTA.  Shared memory per CTA is
// N*L*sizeof(V) (<= 64 KB so two or more CTAs fit per SM).
template <typename T, int N>
struct StridedCfg {  // y / x passes: lines along a strided axis, L adjacent k
  static constexpr int E = imin(16, N);
  static constexpr int VB = 2 * sizeof(T);
  static constexpr int L = imax(1, imin(8, (64 * 1024) / (N * VB)));
  static constexpr int P = N / E;
  static constexpr int THREADS = L * P;
  static constexpr int SMEM = N * L * VB;
};

template <typename T, int NR>
struct ContigCfg {  // z passes: rows of NR reals = M = NR/2 complex
  static constexpr int M = NR / 2;
  static constexpr int E = imin(16, M);
  static constexpr int P = M / E;
  static constexpr int VB = 2 * sizeof(T);
  // rows per CTA: aim for 256 threads, at least 8 rows, at most 64 KB smem,
  // never more rows than the grid has (n^2).
  static constexpr int L0 = imax(8, 256 / P);
  static constexpr int L1 = imin(L0, imax(1, (64 * 1024) / ((M + 1) * VB)));
  static constexpr int L = imin(L1, NR * NR);
  static constexpr int THREADS = L * P;
  static constexpr int SMEM = (M * L + L) * VB;
};

__device__ __forceinline__ int signed_freq(int k, int n) { return k <= n / 2 ? k : k - n; }  // fft_solver.hpp:19

template <typename V>
__device__ __forceinline__ V* smem_base() {
  extern __shared__ __align__(16) unsigned char arena_smem_raw[];
  return reinterpret_cast<V*>(arena_smem_raw);
}

// ------------------------------------------------------------------- K1 zfwd
// Rows of NR reals: z[m] = f[2m] + i f[2m+1] (one vector load), M-point FFT,
// then X[k] = 1/2 (A + B) - 1/2 i W_n^k (A - B), A = Z[k], B = conj(Z[M-k]),
// for k in [0, M]; X[M] = Re Z0 - Im Z0.
template <typename T, int NR>
__global__ void __launch_bounds__(ContigCfg<T, NR>::THREADS)
    k_zfwd(const T* __restrict__ f, vec2_t<T>* __restrict__ S, int ncp, const vec2_t<T>* __restrict__ tw) {
  using V = vec2_t<T>;
  using C = ContigCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L;
  constexpr int SW = engine_swizzle<M, E>();
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const size_t row = size_t(blockIdx.x) * L + l;
  const V* src = reinterpret_cast<const V*>(f + row * NR);
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  line_fft<M, E, L, -1>(v, sm, tw, 2, t, l);
#pragma unroll
  for (int e = 0; e < E; ++e) sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  __syncthreads();
  V* dst = S + row * ncp;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    const V A = v[e];
    const V Bc = sm[smem_idx<L, SW, V>((M - k) & (M - 1), l)];
    const V B{Bc.x, -Bc.y};
    const V W = __ldg(tw + k);  // W_n^k
    const V WD = cmul(W, csub(A, B));
    dst[k] = V{T(0.5) * (A.x + B.x + WD.y), T(0.5) * (A.y + B.y - WD.x)};
    if (k == 0) dst[M] = V{A.x - A.y, T(0)};
  }
}

// ------------------------------------------------------------------- K5 zinv
// Inverse of K1 with FFTW c2r semantics (imaginary parts of X[0] and X[M]
// ignored): Z[k] = (A + B) + i (A - B) conj(W_n^k), A = X[k], B = conj(X[M-k]),
// M-point backward FFT, u[2m] = Re z[m], u[2m+1] = Im z[m].
template <typename T, int NR>
__global__ void __launch_bounds__(ContigCfg<T, NR>::THREADS)
    k_zinv(const vec2_t<T>* __restrict__ S, T* __restrict__ u, int ncp, const vec2_t<T>* __restrict__ tw) {
  using V = vec2_t<T>;
  using C = ContigCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L;
  constexpr int SW = engine_swizzle<M, E>();
  V* sm = smem_base<V>();
  V* xm = sm + M * L;  // X[M] per line
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const size_t row = size_t(blockIdx.x) * L + l;
  const V* src = S + row * ncp;
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    v[e] = __ldcs(src + t + P * e);
    sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  }
  if (t == 0) xm[l] = __ldcs(src + M);
  __syncthreads();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    V A = v[e];
    V Bs = (k == 0) ? xm[l] : sm[smem_idx<L, SW, V>(M - k, l)];
    if (k == 0) {
      A.y = T(0);
      Bs.y = T(0);
    }
    const V B{Bs.x, -Bs.y};
    const V W = __ldg(tw + k);
    const V Ep = cadd(A, B);
    const V Op = cmulc(csub(A, B), W);
    v[e] = V{Ep.x - Op.y, Ep.y + Op.x};
  }
  __syncthreads();
  line_fft<M, E, L, +1>(v, sm, tw, 2, t, l);
  V* dst = reinterpret_cast<V*>(u + row * NR);
#pragma unroll
  for (int e = 0; e < E; ++e) __stcs(dst + t + P * e, v[e]);
}

// --------------------------------------------------------------- K2/K4 ypass
template <typename T, int N, int S>
__global__ void __launch_bounds__(StridedCfg<T, N>::THREADS)
    k_ypass(vec2_t<T>* __restrict__ spec, int ncp, int nc, const vec2_t<T>* __restrict__ tw) {
  using V = vec2_t<T>;
  using C = StridedCfg<T, N>;
  constexpr int E = C::E, P = C::P, L = C::L;
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int k = blockIdx.x * L + l;
  const bool valid = k < nc;
  V* base = spec + size_t(blockIdx.y) * N * ncp + k;
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = valid ? __ldcs(base + size_t(t + P * e) * ncp) : V{T(0), T(0)};
  line_fft<N, E, L, S>(v, sm, tw, 1, t, l);
  if (valid) {
#pragma unroll
    for (int e = 0; e < E; ++e) __stcs(base + size_t(t + P * e) * ncp, v[e]);
  }
}

// -------------------------------------------------------------- K3 xmid
// Forward FFT along i, multiply by the Poisson symbol of fft_solver.cpp:66-79
// (same expression: k2 == 0 ? 0 : scale / (four_pi2 * k2), k2 summed in T from
// exact integer squares), backward FFT along i.  The data never leaves
// registers between the two transforms.
template <typename T, int N>
__global__ void __launch_bounds__(StridedCfg<T, N>::THREADS)
    k_xmid(vec2_t<T>* __restrict__ spec, int ncp, int nc, const vec2_t<T>* __restrict__ tw, T scale, T four_pi2) {
  using V = vec2_t<T>;
  using C = StridedCfg<T, N>;
  constexpr int E = C::E, P = C::P, L = C::L;
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int k = blockIdx.x * L + l;
  const int j = blockIdx.y;
  const bool valid = k < nc;
  const size_t istride = size_t(N) * ncp;
  V* base = spec + size_t(j) * ncp + k;
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = valid ? __ldcs(base + size_t(t + P * e) * istride) : V{T(0), T(0)};
  line_fft<N, E, L, -1>(v, sm, tw, 1, t, l);
  const T kj = T(signed_freq(j, N)), kk = T(k);
  const T c = kj * kj + kk * kk;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const T ki = T(signed_freq(t + P * e, N));
    const T k2 = ki * ki + c;
    const T m = (k2 == T(0)) ? T(0) : scale / (four_pi2 * k2);
    v[e].x *= m;
    v[e].y *= m;
  }
  line_fft<N, E, L, +1>(v, sm, tw, 1, t, l);
  if (valid) {
#pragma unroll
    for (int e = 0; e < E; ++e) __stcs(base + size_t(t + P * e) * istride, v[e]);
  }
}

}  // namespace arena_fft
