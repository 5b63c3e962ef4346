// poisson_split3.cuh — the radix-3 split of the i and j transforms for
// n = 3M (M a power of two): the mixed-radix sizes 48 ... 1536 run their y / x
// passes on the power-of-two TMA kernels.
//
// As the quadrant formulation (poisson_quad.cuh) with radix 3: after the rows'
// r2c (the generic path's z pass, two rows per complex line), for the nine rows
// (i' + aM, j' + bM), a, b in {0, 1, 2},
//
//   Y_{ci,cj}[i', j', k] = W_n^{ci i' + cj j'} sum_{a,b} W_3^{a ci + b cj} X[i' + aM, j' + bM, k]
//
// and the M x M two-dimensional DFT of Y_{ci,cj} over (i', j') is the spectrum at
// (3i'' + ci, 3j'' + cj).  Nine independent problems with M-point y / x lines
// (k_strided_tma<..., SPL = 3>, symbol at ki = 3i'' + ci, kj = 3j'' + cj), then
// the inverse step and the rows' c2r.  Seven sweeps instead of five, but every
// one at the power-of-two kernels' efficiency instead of the generic stages'.
//
// Workspaces: S in the generic layout (row (i, j) at (i*n + j)*ncp) for the z
// passes, Q with nine chunks of Layout(M, M) (chunk 3ci + cj) for the strided
// passes; the split / merge kernels move between them.
#pragma once

#include "poisson_pow2.cuh"

namespace arena_fft {

// 3-point DFT of x[0..2], sign S (-1 forward): W_3 = -1/2 + S i sqrt(3)/2.
template <int S, typename V>
__device__ __forceinline__ void dft3(V& x0, V& x1, V& x2) {
  using T = decltype(x0.x);
  constexpr T h = T(0.8660254037844386);  // sqrt(3)/2
  const V s = cadd(x1, x2), d = csub(x1, x2);
  const V m{x0.x - T(0.5) * s.x, x0.y - T(0.5) * s.y};
  const V r{-S * h * d.y, S * h * d.x};  // S i h d
  x0 = cadd(x0, s);
  x1 = cadd(m, r);
  x2 = csub(m, r);
}

// 3x3 DFT y[ci][cj] = sum_{a,b} W_3^{S(a ci + b cj)} x[a][b] in place.
template <int S, typename V>
__device__ __forceinline__ void dft3x3(V (&x)[3][3]) {
#pragma unroll
  for (int a = 0; a < 3; ++a) dft3<S>(x[a][0], x[a][1], x[a][2]);  // over b -> cj
#pragma unroll
  for (int c = 0; c < 3; ++c) dft3<S>(x[0][c], x[1][c], x[2][c]);  // over a -> ci
}

// Forward split: S (generic layout) -> Q (nine chunks).  One CTA per (i', j'),
// threads over k (coalesced rows).
template <typename T>
__global__ void __launch_bounds__(128) k_split3_fwd(const vec2_t<T>* __restrict__ S, vec2_t<T>* __restrict__ Q,
                                                  const vec2_t<T>* __restrict__ tw, int n, int M, int nc, int ncp,
                                                  Layout gq) {
  using V = vec2_t<T>;
  const int ip = blockIdx.x / M, jp = blockIdx.x % M;
  const V* src[3][3];
  V* dst[3][3];
  V w[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      src[a][b] = S + (size_t(ip + a * M) * n + (jp + b * M)) * ncp;
      dst[a][b] = Q + lrow(gq, 3 * a + b, ip, jp) * ncp;
      w[a][b] = tw_load(tw, (a * ip + b * jp) % n);  // W_n^{ci i' + cj j'}, (ci, cj) = (a, b)
    }
  for (int k = threadIdx.x; k < nc; k += blockDim.x) {
    V x[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) x[a][b] = __ldcs(src[a][b] + k);
    dft3x3<-1>(x);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) st_out(dst[a][b] + k, cmul(x[a][b], w[a][b]));
  }
}

// Inverse merge: Q -> S, x_{a,b} = sum_{ci,cj} W_3^{-(a ci + b cj)} W_n^{-(ci i' + cj j')} Y'_{ci,cj}.
template <typename T>
__global__ void __launch_bounds__(128) k_split3_inv(const vec2_t<T>* __restrict__ Q, vec2_t<T>* __restrict__ S,
                                                  const vec2_t<T>* __restrict__ tw, int n, int M, int nc, int ncp,
                                                  Layout gq) {
  using V = vec2_t<T>;
  const int ip = blockIdx.x / M, jp = blockIdx.x % M;
  const V* src[3][3];
  V* dst[3][3];
  V w[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      src[a][b] = Q + lrow(gq, 3 * a + b, ip, jp) * ncp;
      dst[a][b] = S + (size_t(ip + a * M) * n + (jp + b * M)) * ncp;
      w[a][b] = tw_load(tw, (a * ip + b * jp) % n);
    }
  for (int k = threadIdx.x; k < nc; k += blockDim.x) {
    V x[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) x[a][b] = cmulc(__ldcs(src[a][b] + k), w[a][b]);
    dft3x3<+1>(x);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) st_out(dst[a][b] + k, x[a][b]);
  }
}

}  // namespace arena_fft
