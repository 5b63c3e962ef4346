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
  } else if constexpr (R == 5) {
    // X1,4 = a1 -/+ S' i b1, X2,3 = a2 -/+ S' i b2 with t1 = x1 + x4, t2 = x2 + x3,
    // t3 = x1 - x4, t4 = x2 - x3, a1 = x0 + c1 t1 + c2 t2, a2 = x0 + c2 t1 + c1 t2,
    // b1 = s1 t3 + s2 t4, b2 = s2 t3 - s1 t4 (c_k, s_k = cos, sin(2 pi k / 5))
    constexpr T c1 = T(cos5(1)), c2 = T(cos5(2)), s1 = T(sin5(1)), s2 = T(sin5(2));
    const V x0 = x[0];
    const V t1 = cadd(x[s], x[4 * s]), t2 = cadd(x[2 * s], x[3 * s]);
    const V t3 = csub(x[s], x[4 * s]), t4 = csub(x[2 * s], x[3 * s]);
    const V a1{fma(c2, t2.x, fma(c1, t1.x, x0.x)), fma(c2, t2.y, fma(c1, t1.y, x0.y))};
    const V a2{fma(c1, t2.x, fma(c2, t1.x, x0.x)), fma(c1, t2.y, fma(c2, t1.y, x0.y))};
    const V b1{fma(s2, t4.x, s1 * t3.x), fma(s2, t4.y, s1 * t3.y)};
    const V b2{fma(-s1, t4.x, s2 * t3.x), fma(-s1, t4.y, s2 * t3.y)};
    // i b = (-b.y, b.x); forward (S = -1): X1 = a1 - i b1
    const V ib1{-b1.y, b1.x}, ib2{-b2.y, b2.x};
    x[0] = cadd(x0, cadd(t1, t2));
    x[s] = S < 0 ? csub(a1, ib1) : cadd(a1, ib1);
    x[4 * s] = S < 0 ? cadd(a1, ib1) : csub(a1, ib1);
    x[2 * s] = S < 0 ? csub(a2, ib2) : cadd(a2, ib2);
    x[3 * s] = S < 0 ? cadd(a2, ib2) : csub(a2, ib2);
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

// ------------------------------------------------ z passes for n = R * M rows
// A row of n reals is packed into NZ = n/2 = R * MH complex points (MH = M/2, a
// power of two).  Its NZ-point FFT is a radix-R step in registers (decimation in
// frequency: y_d[m] = W_NZ^{d m} sum_c W_R^{c d} z[m + MH c]) followed by R
// MH-point FFTs on the line engine, Z[R q + d] = FFT(y_d)[q]; the spectrum is
// staged in shared memory in natural order for the r2c split (as zfwd_rows).
// The inverse mirrors it.  Replaces the generic stages' z passes of the split
// path.
#ifndef ARENA_SPLITZ_E3
#define ARENA_SPLITZ_E3 8  // points per thread per sub-FFT, R = 3 (R * E values live)
#endif
#ifndef ARENA_SPLITZ_E5
#define ARENA_SPLITZ_E5 4
#endif
#ifndef ARENA_SPLITZ_THREADS
#define ARENA_SPLITZ_THREADS 32  // threads per CTA (at least: one row's P threads).  B200, 768^3: z passes
                                 // 1.85 / 2.16 ms at 64 threads, 1.52 / 1.82 at 32 (one warp: cheap barriers)
#endif
template <typename T, int R, int MH>
struct SplitZCfg {
  static constexpr int NZ = R * MH;
  static constexpr int E = imin(R == 3 ? ARENA_SPLITZ_E3 : ARENA_SPLITZ_E5, MH);
  static constexpr int P = MH / E;
  static constexpr int L = imax(1, ARENA_SPLITZ_THREADS / P);  // rows per CTA
  static constexpr int THREADS = L * P;
  static constexpr int SMEM = (NZ * L + L) * 2 * int(sizeof(T));
};

template <typename T, int R, int MH>
__global__ void __launch_bounds__(SplitZCfg<T, R, MH>::THREADS) k_zfwd_split(const T* __restrict__ f,
                                                                            vec2_t<T>* __restrict__ S,
                                                                            const vec2_t<T>* __restrict__ tw,
                                                                            const vec2_t<T>* __restrict__ stw,
                                                                            int ncp, long long nrows) {
  using V = vec2_t<T>;
  using C = SplitZCfg<T, R, MH>;
  constexpr int NZ = C::NZ, E = C::E, P = C::P, L = C::L, n = 2 * NZ;
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const long long row = (long long)blockIdx.x * L + l;
  const bool ok = row < nrows;
  const V* src = reinterpret_cast<const V*>(f + (ok ? row : 0) * n);
  V v[R][E];
#pragma unroll
  for (int c = 0; c < R; ++c)
#pragma unroll
    for (int e = 0; e < E; ++e) v[c][e] = ok ? __ldcs(src + t + P * e + MH * c) : V{T(0), T(0)};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    V x[R];
#pragma unroll
    for (int c = 0; c < R; ++c) x[c] = v[c][e];
    dftR<R, -1>(x, 1);
    const int m = t + P * e;
#pragma unroll
    for (int d = 0; d < R; ++d) v[d][e] = d ? cmul(x[d], tw_load(tw, (2 * d * m) % n)) : x[0];  // W_NZ^{d m}
  }
#pragma unroll
  for (int d = 0; d < R; ++d) line_fft<MH, E, L, -1, kSyncCta>(v[d], sm, stw, t, l);
#pragma unroll
  for (int d = 0; d < R; ++d)
#pragma unroll
    for (int e = 0; e < E; ++e) sm[(R * (t + P * e) + d) * L + l] = v[d][e];  // Z[R q + d]
  __syncthreads();
  if (!ok) return;
  V* dst = S + row * ncp;
#pragma unroll
  for (int e = 0; e < R * E; ++e) {
    const int k = t + P * e;
    const V A = sm[k * L + l];
    const V Bc = sm[((NZ - k) % NZ) * L + l];
    const V B{Bc.x, -Bc.y};
    const V W = tw_load(tw, k);  // W_n^k
    const V WD = cmul(W, csub(A, B));
    st_out(dst + k, V{T(0.5) * (A.x + B.x + WD.y), T(0.5) * (A.y + B.y - WD.x)});
    if (k == 0) st_out(dst + NZ, V{A.x - A.y, T(0)});
  }
}

template <typename T, int R, int MH>
__global__ void __launch_bounds__(SplitZCfg<T, R, MH>::THREADS) k_zinv_split(const vec2_t<T>* __restrict__ S,
                                                                            T* __restrict__ u,
                                                                            const vec2_t<T>* __restrict__ tw,
                                                                            const vec2_t<T>* __restrict__ stw,
                                                                            int ncp, long long nrows) {
  using V = vec2_t<T>;
  using C = SplitZCfg<T, R, MH>;
  constexpr int NZ = C::NZ, E = C::E, P = C::P, L = C::L, n = 2 * NZ;
  V* sm = smem_base<V>();
  V* xm = sm + NZ * L;
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const long long row = (long long)blockIdx.x * L + l;
  const bool ok = row < nrows;
  const V* src = S + (ok ? row : 0) * ncp;
  V z[R * E];
#pragma unroll
  for (int e = 0; e < R * E; ++e) {
    z[e] = ok ? __ldcs(src + t + P * e) : V{T(0), T(0)};
    sm[(t + P * e) * L + l] = z[e];
  }
  if (t == 0) xm[l] = ok ? __ldcs(src + NZ) : V{T(0), T(0)};
  __syncthreads();
#pragma unroll
  for (int e = 0; e < R * E; ++e) {  // Hermitian merge into the packed spectrum (as zinv_rows)
    const int k = t + P * e;
    V A = z[e];
    V Bs = (k == 0) ? xm[l] : sm[(NZ - k) * L + l];
    if (k == 0) {
      A.y = T(0);
      Bs.y = T(0);
    }
    const V B{Bs.x, -Bs.y};
    const V W = tw_load(tw, k);
    const V Ep = cadd(A, B);
    const V Op = cmulc(csub(A, B), W);
    z[e] = V{Ep.x - Op.y, Ep.y + Op.x};
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < R * E; ++e) sm[(t + P * e) * L + l] = z[e];
  __syncthreads();
  V v[R][E];
#pragma unroll
  for (int d = 0; d < R; ++d)
#pragma unroll
    for (int e = 0; e < E; ++e) v[d][e] = sm[(R * (t + P * e) + d) * L + l];  // Z[R q + d]
  __syncthreads();
#pragma unroll
  for (int d = 0; d < R; ++d) line_fft<MH, E, L, +1, kSyncCta>(v[d], sm, stw, t, l);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int m = t + P * e;
    V x[R];
#pragma unroll
    for (int d = 0; d < R; ++d) x[d] = d ? cmulc(v[d][e], tw_load(tw, (2 * d * m) % n)) : v[0][e];
    dftR<R, +1>(x, 1);
#pragma unroll
    for (int c = 0; c < R; ++c) v[c][e] = x[c];
  }
  if (!ok) return;
  V* dst = reinterpret_cast<V*>(u + row * n);
#pragma unroll
  for (int c = 0; c < R; ++c)
#pragma unroll
    for (int e = 0; e < E; ++e) st_out(dst + t + P * e + MH * c, v[c][e]);
}

}  // namespace arena_fft
