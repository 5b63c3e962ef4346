// poisson_split3.cuh — the radix-R split (R = 3 or 5) of the i and j
// transforms for n = RM (M a power of two): the mixed-radix sizes 48 ... 1536
// (R = 3) and 80 ... 1280 (R = 5) run their y / x passes on the power-of-two
// TMA kernels.  Written below for R = 3; R = 5 is the same with 25 chunks.
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

// cos / sin(2 pi m / 5)
__host__ __device__ constexpr double cos5(int m) {
  return m == 0 ? 1.0 : (m == 1 || m == 4) ? 0.30901699437494745 : -0.8090169943749475;
}
__host__ __device__ constexpr double sin5(int m) {
  return m == 0 ? 0.0 : m == 1 ? 0.9510565162951535 : m == 2 ? 0.5877852522924731 : m == 3 ? -0.5877852522924731
                                                                                         : -0.9510565162951535;
}

// R-point DFT (R = 3 or 5) of x[0], x[s], ..., x[(R-1) s], sign S, in place.
template <int R, int S, typename V>
__device__ __forceinline__ void dftR(V* x, int s) {
  using T = decltype(x->x);
  if constexpr (R == 3) {
    dft3<S>(x[0], x[s], x[2 * s]);
  } else {
    V in[R], out[R];
#pragma unroll
    for (int r = 0; r < R; ++r) in[r] = x[r * s];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      T re = in[0].x, im = in[0].y;
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const T c = T(cos5((r * q) % R)), sn = T(S * sin5((r * q) % R));  // exp(S 2 pi i rq / 5) = c + i sn
        re = fma(in[r].x, c, fma(-in[r].y, sn, re));
        im = fma(in[r].y, c, fma(in[r].x, sn, im));
      }
      out[q] = V{re, im};
    }
#pragma unroll
    for (int r = 0; r < R; ++r) x[r * s] = out[r];
  }
}

// RxR DFT y[ci][cj] = sum_{a,b} W_R^{S(a ci + b cj)} x[a][b] in place.
template <int R, int S, typename V>
__device__ __forceinline__ void dftRxR(V (&x)[R][R]) {
#pragma unroll
  for (int a = 0; a < R; ++a) dftR<R, S>(&x[a][0], 1);  // over b -> cj
#pragma unroll
  for (int c = 0; c < R; ++c) dftR<R, S>(&x[0][c], R);  // over a -> ci
}

// Forward split: S (generic layout) -> Q (nine chunks).  One CTA per (i', j'),
// threads over k (coalesced rows).
template <typename T, int R>
__global__ void __launch_bounds__(128) k_split3_fwd(const vec2_t<T>* __restrict__ S, vec2_t<T>* __restrict__ Q,
                                                  const vec2_t<T>* __restrict__ tw, int n, int M, int nc, int ncp,
                                                  Layout gq) {
  using V = vec2_t<T>;
  const int ip = blockIdx.x / M, jp = blockIdx.x % M;
  const V* src[R][R];
  V* dst[R][R];
  V w[R][R];
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int b = 0; b < R; ++b) {
      src[a][b] = S + (size_t(ip + a * M) * n + (jp + b * M)) * ncp;
      dst[a][b] = Q + lrow(gq, R * a + b, ip, jp) * ncp;
      w[a][b] = tw_load(tw, (a * ip + b * jp) % n);  // W_n^{ci i' + cj j'}, (ci, cj) = (a, b)
    }
  for (int k = threadIdx.x; k < nc; k += blockDim.x) {
    V x[R][R];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) x[a][b] = __ldcs(src[a][b] + k);
    dftRxR<R, -1>(x);
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) st_out(dst[a][b] + k, cmul(x[a][b], w[a][b]));
  }
}

// Inverse merge: Q -> S, x_{a,b} = sum_{ci,cj} W_3^{-(a ci + b cj)} W_n^{-(ci i' + cj j')} Y'_{ci,cj}.
template <typename T, int R>
__global__ void __launch_bounds__(128) k_split3_inv(const vec2_t<T>* __restrict__ Q, vec2_t<T>* __restrict__ S,
                                                  const vec2_t<T>* __restrict__ tw, int n, int M, int nc, int ncp,
                                                  Layout gq) {
  using V = vec2_t<T>;
  const int ip = blockIdx.x / M, jp = blockIdx.x % M;
  const V* src[R][R];
  V* dst[R][R];
  V w[R][R];
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int b = 0; b < R; ++b) {
      src[a][b] = Q + lrow(gq, R * a + b, ip, jp) * ncp;
      dst[a][b] = S + (size_t(ip + a * M) * n + (jp + b * M)) * ncp;
      w[a][b] = tw_load(tw, (a * ip + b * jp) % n);
    }
  for (int k = threadIdx.x; k < nc; k += blockDim.x) {
    V x[R][R];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) x[a][b] = cmulc(__ldcs(src[a][b] + k), w[a][b]);
    dftRxR<R, +1>(x);
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) st_out(dst[a][b] + k, x[a][b]);
  }
}

}  // namespace arena_fft
