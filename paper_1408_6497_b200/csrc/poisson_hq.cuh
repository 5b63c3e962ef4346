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
//   Y_c[i', j, k] = W_n^{c i'} (X[i', j, k] + (-1)^c X[i'+H, j, k]),   c = 0, 1
//                 = W_n^{c i'} r2c_k(f[i', j] + (-1)^c f[i'+H, j]),
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
  // rows l of a CTA: (i' + (l / JR) H, j + l % JR) — JR adjacent j of both rows of the
  // pair, so each half of the CTA streams JR contiguous rows (JR = 2: 16 KB at n = 1024)
#ifndef ARENA_HQ_JR
#define ARENA_HQ_JR 1  // B200 1024^3 fp64: z passes 3.32 / 4.01 / 5.93 ms (fwd) at JR = 1 / 2 / 4
#endif
  static constexpr int JR = ARENA_HQ_JR;
  static constexpr int L = 2 * JR;
  static constexpr int THREADS = L * P;
  static constexpr int SYNC = THREADS <= 32 ? kSyncWarp : kSyncCta;
  static constexpr int MINB = imin(32, imax(1, ContigCfg<T, NR>::MINB * ContigCfg<T, NR>::THREADS / THREADS));
  static constexpr int SMEM = (M * L + L) * 2 * int(sizeof(T));
  static constexpr int PF = ARENA_Z_PF * ARENA_SMS * MINB;  // L2 prefetch distance (CTAs)
  static constexpr bool OK = NR >= 16 && THREADS <= 1024;
};

// The radix-2 step commutes with the row transforms (both linear, different axes,
// W_n^{i'} is one complex scalar per row pair), so it runs on the REAL rows right
// after they are loaded: g_c = f[i'] + (-1)^c f[i'+H], exchanged between the two
// lanes that hold the same positions of the pair (lane l = row, partner lane ^ 1),
// then Y_c = W_n^{c i'} r2c(g_c) — the plain row kernel's work plus one shuffle
// per element and one complex product at the store.  K5h mirrors it on the half
// spectra before the Hermitian split and the c2r.
template <typename T, int THREADS, int X>
__device__ __forceinline__ vec2_t<T> shfl_pair(vec2_t<T> v) {
  constexpr unsigned mask = THREADS >= 32 ? 0xffffffffu : (1u << THREADS) - 1u;
  return vec2_t<T>{__shfl_xor_sync(mask, v.x, X), __shfl_xor_sync(mask, v.y, X)};
}

// K1 (i-split): butterfly of the row pair (i', j), (i'+H, j), r2c of g_0 / g_1 into the chunks.
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
  constexpr int JR = C::JR, NJB = NR / JR;
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int c = l / JR;                                              // chunk = which row of the pair
  const int ip = blockIdx.x / NJB, j = (blockIdx.x % NJB) * JR + l % JR;
  if constexpr (ARENA_Z_PF > 0) {  // the rows one resident wave ahead, into L2
    const unsigned b = blockIdx.x + C::PF;
    if (threadIdx.x < 2 && b < gridDim.x)
      bulk_prefetch_l2(f + (size_t(b / NJB + threadIdx.x * H) * NR + (b % NJB) * JR) * NR, JR * NR * sizeof(T));
  }
  const V* src = reinterpret_cast<const V*>(f + (size_t(ip + c * H) * NR + j) * NR);
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
#pragma unroll
  for (int e = 0; e < E; ++e) {  // g_0 = f_a + f_b (chunk c = 0), g_1 = f_a - f_b (c = 1)
    const V o = shfl_pair<T, C::THREADS, C::JR>(v[e]);
    v[e] = c == 0 ? cadd(v[e], o) : csub(o, v[e]);
  }
  line_fft<M, E, L, -1, SYNC>(v, sm, stw, t, l);
#pragma unroll
  for (int e = 0; e < E; ++e) sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  xbarrier<SYNC>();
  const V Wi = c == 0 ? V{T(1), T(0)} : tw_load(tw, ip);  // W_n^{c i'}
  V* dst = S + lrow(gh, c, ip, j) * ncp;
#pragma unroll
  for (int e = 0; e < E; ++e) {  // Hermitian split of the packed row (as zfwd_rows), times W_n^{c i'}
    const int k = t + P * e;
    const V A = v[e];
    const V Bc = sm[smem_idx<L, SW, V>((M - k) & (M - 1), l)];
    const V B{Bc.x, -Bc.y};
    const V W = tw_load(tw, k);  // W_n^k
    const V WD = cmul(W, csub(A, B));
    const V X{T(0.5) * (A.x + B.x + WD.y), T(0.5) * (A.y + B.y - WD.x)};
    st_out(dst + k, c == 0 ? X : cmul(X, Wi));
    if (k == 0) {
      const V XM{A.x - A.y, T(0)};
      st_out(dst + M, c == 0 ? XM : cmul(XM, Wi));
    }
  }
}

// K5 (i-split): the inverse radix-2 step of the pair on the chunks' half spectra
// (H_c = Y_0 + (-1)^c conj(W_n^{i'}) Y_1, exchanged between the pair's lanes), then
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
  V* xm = sm + M * L;  // X[M] per row
  constexpr int JR = C::JR, NJB = NR / JR;
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int c = l / JR;
  const int ip = blockIdx.x / NJB, j = (blockIdx.x % NJB) * JR + l % JR;
  if constexpr (ARENA_Z_PF > 0) {
    const unsigned b = blockIdx.x + C::PF;
    if (threadIdx.x < 2 && b < gridDim.x)
      bulk_prefetch_l2(S + lrow(gh, threadIdx.x, b / NJB, (b % NJB) * JR) * ncp, JR * ncp * sizeof(V));
  }
  const V* src = S + lrow(gh, c, ip, j) * ncp;
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  V ym = t == 0 ? __ldcs(src + M) : V{T(0), T(0)};
  const V Wi = tw_load(tw, ip);
  auto pair = [&](V own) {  // H_l from the pair's two chunk values at one k
    const V o = shfl_pair<T, C::THREADS, C::JR>(own);
    const V z0 = c == 0 ? own : o, z1 = cmulc(c == 0 ? o : own, Wi);
    return c == 0 ? cadd(z0, z1) : csub(z0, z1);
  };
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = pair(v[e]);
  ym = pair(ym);
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
  V* dst = reinterpret_cast<V*>(u + (size_t(ip + c * H) * NR + j) * NR);
#pragma unroll
  for (int e = 0; e < E; ++e) st_out(dst + t + P * e, v[e]);
}

}  // namespace arena_fft
