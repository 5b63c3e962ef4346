// poisson_xpp.cuh — the fused x pass (K3: forward FFT along i * Poisson symbol of
// /root/reference/proj/src/fft_solver.cpp:66-79 * backward FFT along i) as two
// half-CTA groups running out of phase ("ping-pong").
//
// Why: in k_strided_tma<…, 2> the eight warps of the one resident CTA run in
// lockstep through CTA-wide exchange barriers, so the kernel's phases — fp64
// butterflies (~8.2k clk per tile at the full DFMA rate), shared-memory
// exchanges (~5k clk) and the global stores (~2k clk) — follow each other instead
// of overlapping (17.7k clk per tile measured; neither the fp64 pipe, 50%, nor
// DRAM, 60%, is busy).  The register file only holds eight 32-point warps, so
// the overlap cannot come from more warps; it has to come from warps in
// different phases.
//
// Here one CTA per SM still takes 8-line tiles (128-byte TMA rows, the
// DRAM-friendly width), but its 256 threads form two groups of 128: group g
// transforms lines 4g .. 4g+3 on its own named barrier, with its own half-size
// exchange scratch (the split exchange of fft_engine.cuh: real parts, then
// imaginary parts).  The tile buffer is only the TMA landing zone: it is
// refilled as soon as both groups have read their lines into registers (the
// second group's leader issues the request), so the load of tile g+1 overlaps
// the transforms of tile g.  Group 1 starts half a transform late (a one-time
// named-barrier handshake after group 0's first forward FFT); the skew then
// sustains itself: group 0 is the one that waits for the next tile (if anyone
// does), group 1 finds it already landed.
#pragma once

#include "poisson_pow2.cuh"

namespace arena_fft {

#ifndef ARENA_XPP_SKEW
#define ARENA_XPP_SKEW 1  // 0: both groups start together (A/B of the skew itself)
#endif

template <typename T, int N>
struct XppCfg {
  using B = TmaCfg<T, N, false, true>;  // the wide x tile: 128-byte rows
  static constexpr int E = B::E, P = N / E, L = B::L;
  static constexpr int G = 2, LG = L / G;  // groups, lines per group
  static constexpr int GT = LG * P;        // threads per group
  static constexpr int THREADS = G * GT;
  static constexpr int VB = 2 * sizeof(T);
  static constexpr int TILE = N * L;                // complex elements of the landing tile
  static constexpr int TW = stage_tw_total(N, E);   // staged stage twiddles
  static constexpr int SMEM = TILE * VB + TILE * VB / 2 + TW * VB + 64;
  static constexpr bool OK = N >= 64 && L >= 2 && GT % 32 == 0 && GT <= 512 && num_stages(N, E) == 2 &&
                             SMEM <= 227 * 1024 && TILE * VB == 128 * 1024;
};

__device__ __forceinline__ void named_bar_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ unsigned atom_add_acq_rel_cta(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(smem_u32(p)), "r"(v) : "memory");
  return old;
}

// SPL = 0: the single-GPU n = N layout; SPL = 2: quadrant chunks of the n = 2N grid
// (poisson_quad.cuh).  Compile-time geometry (the FIXED case of k_strided_tma).
template <typename T, int N, int SPL = 0>
__global__ void __launch_bounds__(XppCfg<T, N>::THREADS, 1)
    k_xpass_pp(const __grid_constant__ CUtensorMap tmap, vec2_t<T>* __restrict__ spec,
               const vec2_t<T>* __restrict__ stw, T scale, T four_pi2) {
  using V = vec2_t<T>;
  using C = XppCfg<T, N>;
  constexpr int E = C::E, P = C::P, L = C::L, LG = C::LG, GT = C::GT, TILE = C::TILE;
  constexpr bool QUAD = SPL != 0;
  constexpr int NCH = spl_chunks(SPL);
  constexpr Layout g = fixed_geom<N, SPL, 2>();
  constexpr KSpan ks = fixed_kspan<N, SPL, 2>();
  constexpr int KT = (ks.kc + L - 1) / L;
  constexpr int NL = g.nj * KT;  // tiles per chunk
  constexpr int NT = NL * NCH;
  constexpr size_t kq = size_t(ks.kq);
  constexpr uint32_t TILE_BYTES = TILE * sizeof(V);
  constexpr int jbm = (1 << g.jbs) - 1;
  constexpr int IB = tma_ib(g.ni);

  V* land = smem_base<V>();
  const int tid = threadIdx.x;
  const int grp = tid / GT, gtid = tid % GT;
  const int lg = gtid % LG, t = gtid / LG;
  const int l = grp * LG + lg;
  // group scratch: N * LG real scalars (handed to the engine as V*)
  V* scratch = land + TILE + grp * (N * LG / 2);
  V* tws = land + TILE + TILE / 2;
  uint64_t* full = reinterpret_cast<uint64_t*>(tws + C::TW);
  unsigned* cnt = reinterpret_cast<unsigned*>(full + 1);

  if (tid == 0) {
    mbar_init(full, 1);
    *cnt = 0;
    fence_mbar_init();
  }
  for (int i = tid; i < C::TW; i += blockDim.x) tws[i] = __ldg(stw + i);
  __syncthreads();
  const SmemTable<V> twp{tws};

  auto issue = [&](int gt) {
    const int qd = QUAD ? gt / NL : 0;
    if constexpr (QUAD) gt -= qd * NL;
    const int outer = gt / KT, kt = gt % KT;
    mbar_arrive_expect_tx(full, TILE_BYTES);
#pragma unroll
    for (int q = 0; q < g.ni; q += IB)
      tma_load_5d(land + size_t(q) * L, &tmap, full, 2 * kt * L, outer & jbm, q, outer >> g.jbs, qd);
  };

  int gt = blockIdx.x;
  if (tid == 0 && gt < NT) issue(gt);
  for (int it = 0; gt < NT; ++it, gt += gridDim.x) {
    if constexpr (ARENA_XPP_SKEW) {
      if (it == 0 && grp == 1) named_bar_sync(3, C::THREADS);  // start once group 0 is through its first forward FFT
    }
    mbar_wait(full, it & 1);
    V v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = land[(t + P * e) * L + l];
    named_bar_sync(1 + grp, GT);  // the group's lines are in registers
    if (gtid == 0) {
      // the second group through releases the landing zone: request the next tile
      const unsigned old = atom_add_acq_rel_cta(cnt, 1u);
      const int gn = gt + gridDim.x;
      if ((old & 1u) && gn < NT) {
        fence_proxy_async_smem();
        issue(gn);
      }
    }
    const int qd = QUAD ? gt / NL : 0;
    const int gl = QUAD ? gt - qd * NL : gt;
    const int outer = gl / KT;
    const int k = (gl % KT) * L + l;
    line_fft_xs<N, E, LG, -1, GT>(v, scratch, twp, t, lg);
    if constexpr (ARENA_XPP_SKEW) {
      if (it == 0 && grp == 0) named_bar_arrive(3, C::THREADS);
    }
    constexpr int NG = SPL > 0 ? SPL * N : N;
    const T kj = SPL > 0 ? T(signed_freq(SPL * outer + qd % imax(SPL, 1), NG)) : T(signed_freq(outer, NG));
    const T kk = T(k);
    const T c = kj * kj + kk * kk;
    auto kiof = [&](int e) {
      return SPL > 0 ? T(signed_freq(SPL * (t + P * e) + qd / imax(SPL, 1), NG)) : T(signed_freq(t + P * e, NG));
    };
    constexpr bool LEAN = sizeof(T) == 8 && ARENA_LEAN_SYMBOL;
    const T cinv = four_pi2 / scale;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const T k2 = kiof(e) * kiof(e) + c;
      T m;
      if constexpr (LEAN) m = poisson_symbol_lean(k2, cinv);
      else m = poisson_symbol(k2, scale, four_pi2);
      v[e].x *= m;
      v[e].y *= m;
    }
    if constexpr (LEAN) {
      if (c == T(0) && t == 0 && kiof(0) == T(0)) v[0] = V{T(0), T(0)};  // k = 0: the mean, dropped
    }
    line_fft_xs<N, E, LG, +1, GT>(v, scratch, twp, t, lg);
    if (k < ks.kc) {
#pragma unroll
      for (int e = 0; e < E; ++e)
        st_out(spec + (QUAD ? lrow(g, qd, t + P * e, outer) : rowC(g, t + P * e, outer)) * kq + k, v[e]);
    }
  }
}

}  // namespace arena_fft
