// poisson_hq.cuh — the i-split ("half-quadrant") formulation of the single-GPU
// power-of-two solve.
//
// The x pass (forward i transform * Poisson symbol * inverse i transform) is
// the only compute-heavy sweep: at n = 1024 fp64 its 32-point-per-thread lines
// need ~254 registers, so an SM runs 8 warps and the fp64 pipe and HBM overlap
// only partly (B200 r01: 59% of the HBM roofline, vs 81-88% for the other four
// sweeps).  Here the first radix-2 step of the i transform moves into the z
// passes, which hold two whole rows anyway:
//
//   for n = 2H and the row pair (i', j), (i'+H, j) (X = the rows' r2c spectra):
//   Y_c[i', j, k] = W_n^{c i'} (X[i', j, k] + (-1)^c X[i'+H, j, k]),   c = 0, 1,
//
// after which F[2 i'' + c, kj, k] is the H-point DFT over i' of the n-point
// DFT over j of Y_c: two chunk problems whose y lines keep all n points (the
// y passes are unchanged) and whose x lines are H points long, transformed with
// 16 points per thread at ~124 registers, two CTAs of 8 warps per SM.  The
// symbol reads the full-grid ki = 2 i'' + c (k_strided_tma<..., kSplitI>).  The
// inverse z pass undoes the step:
//   x[i'] = Z_0[i'] + W_n^{-i'} Z_1[i'],   x[i'+H] = Z_0[i'] - W_n^{-i'} Z_1[i'],
// then the rows' Hermitian split and c2r (FFTW c2r semantics, as k_zinv).
// The same DFT as fft_solver.cpp:60-80, evaluated in another order.
//
// Workspace: Layout(H, n) with two chunks (chunk c = the i parity of the
// frequency), the same n^2 rows of spec_pitch(n) complex as the plain path.
#pragma once

#include "poisson_pow2.cuh"

namespace arena_fft {

template <typename T, int NR>
struct HqZCfg {
  static constexpr int M = NR / 2;  // complex points of a packed row
  static constexpr int H = NR / 2;  // chunk extent in i
  static constexpr int E = ContigCfg<T, NR>::E;
  static constexpr int P = M / E;
  static constexpr int L = 2;  // the row pair (i', j), (i' + H, j)
  static constexpr int THREADS = L * P;
  static constexpr int SYNC = THREADS <= 32 ? kSyncWarp : kSyncCta;
  static constexpr int MINB = ContigCfg<T, NR>::MINB;
  static constexpr int SMEM = (2 * M + 2) * 2 * int(sizeof(T));
  static constexpr int PF = ARENA_Z_PF * ARENA_SMS * MINB;  // L2 prefetch distance (CTAs)
  static constexpr bool OK = NR >= 16 && THREADS <= 1024;
};

// K1 (i-split): r2c of the row pair, then the radix-2 step along i into the two chunks.
template <typename T, int NR>
__global__ void __launch_bounds__(HqZCfg<T, NR>::THREADS, HqZCfg<T, NR>::MINB)
    k_zfwd_hq(const T* __restrict__ f, vec2_t<T>* __restrict__ S, const vec2_t<T>* __restrict__ tw,
              const vec2_t<T>* __restrict__ stw) {
  using V = vec2_t<T>;
  using C = HqZCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L, H = C::H, SYNC = C::SYNC;
  constexpr int ncp = spec_pitch(NR);
  constexpr int SW = engine_swizzle<M, E>();
  constexpr Layout gh = fixed_geom<NR, kSplitI, 0>();  // (H, n), two chunks
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int ip = blockIdx.x / NR, j = blockIdx.x % NR;
  if constexpr (ARENA_Z_PF > 0) {  // the pair one resident wave ahead, into L2
    const unsigned b = blockIdx.x + C::PF;
    if (threadIdx.x < L && b < gridDim.x)
      bulk_prefetch_l2(f + (size_t(b / NR + threadIdx.x * H) * NR + b % NR) * NR, NR * sizeof(T));
  }
  const size_t row = size_t(ip + l * H) * NR + j;
  const V* src = reinterpret_cast<const V*>(f + row * NR);
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  line_fft<M, E, L, -1, SYNC>(v, sm, stw, t, l);
#pragma unroll
  for (int e = 0; e < E; ++e) sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  xbarrier<SYNC>();
  // Hermitian split of the packed row (as zfwd_rows): X[k], k in [0, M), and X[M]
  V xm{T(0), T(0)};
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    const V A = v[e];
    const V Bc = sm[smem_idx<L, SW, V>((M - k) & (M - 1), l)];
    const V B{Bc.x, -Bc.y};
    const V W = tw_load(tw, k);  // W_n^k
    const V WD = cmul(W, csub(A, B));
    if (k == 0) xm = V{A.x - A.y, T(0)};
    v[e] = V{T(0.5) * (A.x + B.x + WD.y), T(0.5) * (A.y + B.y - WD.x)};
  }
  xbarrier<SYNC>();  // split reads done: the rows' spectra go row-major into sm
  V* xs = sm;  // xs[r * (M + 1) + k], r = 0 (row i'), 1 (row i' + H)
#pragma unroll
  for (int e = 0; e < E; ++e) xs[l * (M + 1) + t + P * e] = v[e];
  if (t == 0) xs[l * (M + 1) + M] = xm;
  xbarrier<SYNC>();
  // chunk l: thread (l, t) forms Y_l at its k
  const V Wi = tw_load(tw, ip);  // W_n^{i'}
  V* dst = S + lrow(gh, l, ip, j) * ncp;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    const V a = xs[k], b = xs[M + 1 + k];
    st_out(dst + k, l == 0 ? cadd(a, b) : cmul(csub(a, b), Wi));
  }
  if (t == 0) {
    const V a = xs[M], b = xs[2 * M + 1];
    st_out(dst + M, l == 0 ? cadd(a, b) : cmul(csub(a, b), Wi));
  }
}

// K5 (i-split): the inverse radix-2 step of the pair from the two chunks, then
// each row's Hermitian split and c2r as zinv_rows.
template <typename T, int NR>
__global__ void __launch_bounds__(HqZCfg<T, NR>::THREADS, HqZCfg<T, NR>::MINB)
    k_zinv_hq(const vec2_t<T>* __restrict__ S, T* __restrict__ u, const vec2_t<T>* __restrict__ tw,
              const vec2_t<T>* __restrict__ stw) {
  using V = vec2_t<T>;
  using C = HqZCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L, H = C::H, SYNC = C::SYNC;
  constexpr int ncp = spec_pitch(NR);
  constexpr int SW = engine_swizzle<M, E>();
  constexpr Layout gh = fixed_geom<NR, kSplitI, 0>();
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int ip = blockIdx.x / NR, j = blockIdx.x % NR;
  if constexpr (ARENA_Z_PF > 0) {
    const unsigned b = blockIdx.x + C::PF;
    if (threadIdx.x < L && b < gridDim.x)
      bulk_prefetch_l2(S + lrow(gh, threadIdx.x, b / NR, b % NR) * ncp, ncp * sizeof(V));
  }
  const V* src = S + lrow(gh, l, ip, j) * ncp;
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  V ym{T(0), T(0)};
  if (t == 0) ym = __ldcs(src + M);
  V* ys = sm;  // ys[c * (M + 1) + k]: chunk c's row
#pragma unroll
  for (int e = 0; e < E; ++e) ys[l * (M + 1) + t + P * e] = v[e];
  if (t == 0) ys[l * (M + 1) + M] = ym;
  xbarrier<SYNC>();
  // row l of the pair: x_l = Z_0 + (-1)^l conj(W_n^{i'}) Z_1
  const V Wi = tw_load(tw, ip);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    const V z0 = ys[k], z1 = cmulc(ys[M + 1 + k], Wi);
    v[e] = l == 0 ? cadd(z0, z1) : csub(z0, z1);
  }
  if (t == 0) {
    const V z0 = ys[M], z1 = cmulc(ys[2 * M + 1], Wi);
    ym = l == 0 ? cadd(z0, z1) : csub(z0, z1);
  }
  xbarrier<SYNC>();  // chunk reads done: sm becomes the rows' split / FFT scratch
  V* xm = sm + M * L;  // X[M] per row
#pragma unroll
  for (int e = 0; e < E; ++e) sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  if (t == 0) xm[l] = ym;
  xbarrier<SYNC>();
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    V A = v[e];
    V Bs = (k == 0) ? xm[l] : sm[smem_idx<L, SW, V>(M - k, l)];
    if (k == 0) {  // FFTW c2r: imaginary parts of X[0] and X[M] ignored
      A.y = T(0);
      Bs.y = T(0);
    }
    const V B{Bs.x, -Bs.y};
    const V W = tw_load(tw, k);
    const V Ep = cadd(A, B);
    const V Op = cmulc(csub(A, B), W);
    v[e] = V{Ep.x - Op.y, Ep.y + Op.x};
  }
  xbarrier<SYNC>();
  line_fft<M, E, L, +1, SYNC>(v, sm, stw, t, l);
  V* dst = reinterpret_cast<V*>(u + (size_t(ip + l * H) * NR + j) * NR);
#pragma unroll
  for (int e = 0; e < E; ++e) st_out(dst + t + P * e, v[e]);
}

}  // namespace arena_fft
