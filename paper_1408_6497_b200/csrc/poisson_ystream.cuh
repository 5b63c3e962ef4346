// poisson_ystream.cuh — the y passes (K2, K4) with the tile load overlapping
// the whole FFT of the previous tile.
//
// The TMA kernel of poisson_pow2.cuh uses its tile buffer as the exchange
// scratch, so the next tile can only be requested after the last exchange: per
// tile the SM first waits for 128 KB to arrive (its share of HBM bandwidth
// makes that ~3 us) and then computes (~4.5 us).  Here the tile buffer is
// released as soon as the tile is in registers, and the exchanges go through a
// separate scratch of half a tile, used by the two halves of the CTA in turn:
//
//   * the L = 2*LH lines of a tile (adjacent k) are split in two groups of LH
//     lines (64-byte half rows, each loaded by its own TMA box so the group's
//     shared-memory reads are conflict-free); group g owns lines g*LH .. g*LH+LH-1;
//   * the groups alternate on the scratch (ping-pong): group 0 writes and reads
//     its lines while group 1 computes its butterflies, then the other way
//     round.  Named barriers: 1 + g inside group g, 3 "group 0 is done with the
//     scratch", 4 "group 1 is done", 5 "tile consumed" (its last warp issues the
//     next TMA load).
//
// Shared memory: tile (N*L elements) + scratch (N*LH) — 192 KB at n = 1024 fp64.
//
// Measured on B200 (1024^3 fp64): 3.75 ms vs 3.52 ms for k_strided_tma, so it is
// off by default.  The exchanges are bound by shared-memory bandwidth (768 KB of
// shared traffic per 128 KB tile either way), so the groups mostly wait for each
// other on the scratch (ncu: 36% barrier stalls) instead of overlapping.
#pragma once

#include "poisson_pow2.cuh"

#ifndef ARENA_YSTREAM
#define ARENA_YSTREAM 0  // 1: y passes use k_ystream (B200 1024^3: 3.75 ms vs 3.52 for k_strided_tma)
#endif

namespace arena_fft {

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <typename T, int N>
struct YsCfg {
  static constexpr int VB = 2 * sizeof(T);
  static constexpr int LH = 64 / VB;  // lines per group: 64-byte half rows (fp64 4, fp32 8)
  static constexpr int L = 2 * LH;    // lines (adjacent k) per tile: 128-byte TMA rows
  static constexpr int E = imin(sizeof(T) == 8 ? 16 : 32, N);
  static constexpr int P = N / E;
  static constexpr int GT = LH * P;  // threads per group
  static constexpr int THREADS = 2 * GT;
  static constexpr int HALF = N * LH;  // elements per half tile (= scratch)
  static constexpr int TILE = 2 * HALF;
  static constexpr int SMEM = (TILE + HALF) * VB + 16;
  static constexpr bool OK = N >= 64 && GT % 32 == 0 && THREADS <= 1024 && SMEM <= 227 * 1024 && num_stages(N, E) >= 2;
};

// Exchange through the shared scratch, taking turns with the other group.
// `first`: group 0's first use in this kernel (nothing to wait for).
template <int N, int E, int LH, int R, int NS, int SW, typename V>
__device__ __forceinline__ void pp_exchange(V (&v)[E], V* scr, int t, int l, int grp, bool& first) {
  constexpr int P = N / E, NB = E / R, GT = LH * P;
  if (grp == 0) {
    if (!first) named_sync(4, 2 * GT);
  } else {
    named_sync(3, 2 * GT);
  }
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int b = t + P * q;
    const int dst = (b & ~(NS - 1)) * R + (b & (NS - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) scr[smem_idx<LH, SW, V>(dst + r * NS, l)] = v[q + NB * r];
  }
  named_sync(1 + grp, GT);
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = scr[smem_idx<LH, SW, V>(t + P * e, l)];
  named_arrive(grp == 0 ? 3 : 4, 2 * GT);
  first = false;
}

template <int N, int E, int LH, int S, int STAGE, typename V, typename TW>
__device__ __forceinline__ void ys_stages(V (&v)[E], V* scr, TW stw, int t, int l, int grp, bool& first) {
  constexpr int NSTAGE = num_stages(N, E);
  if constexpr (STAGE < NSTAGE) {
    constexpr int R = 1 << stage_log2(N, E, STAGE);
    constexpr int NS = stage_ns(N, E, STAGE);
    constexpr int SW = stage_log2(N, E, 0);
    stage_compute<N, E, R, NS, S>(v, t, stw + (STAGE >= 1 ? stage_tw_offset(N, E, STAGE) : 0));
    if constexpr (STAGE + 1 < NSTAGE) pp_exchange<N, E, LH, R, NS, SW>(v, scr, t, l, grp, first);
    ys_stages<N, E, LH, S, STAGE + 1>(v, scr, stw, t, l, grp, first);
  }
}

// PASS 0: y forward, 1: y backward.  Tiles over (il, k-tile) of workspace
// `spec` in Layout g (TMA map `tmap`: 64-byte boxes {2*LH, JB, 1, nj/JB, P});
// results to `out` in Layout gout (rows of pitch ks.kq).
template <typename T, int N, int PASS>
__global__ void __launch_bounds__(YsCfg<T, N>::THREADS, 1)
    k_ystream(const __grid_constant__ CUtensorMap tmap, const vec2_t<T>* __restrict__ stw, Layout g, KSpan ks,
              vec2_t<T>* __restrict__ out, Layout gout) {
  using V = vec2_t<T>;
  using C = YsCfg<T, N>;
  constexpr int E = C::E, P = C::P, LH = C::LH, L = C::L, GT = C::GT;
  constexpr uint32_t HALF_BYTES = C::HALF * sizeof(V);
  constexpr int S = PASS == 0 ? -1 : +1;
  const int KT = (ks.kc + L - 1) / L;
  const int NT = g.ni * KT;
  const size_t kq = size_t(ks.kq);
  V* tile = smem_base<V>();
  V* scr = tile + C::TILE;
  uint64_t* bar = reinterpret_cast<uint64_t*>(scr + C::HALF);
  const int tid = threadIdx.x;
  const int grp = tid / GT, lt = tid % GT;
  const int l = lt % LH, t = lt / LH;
  constexpr int kIssueWarp = GT / 32;  // first warp of group 1 (it reads the tile last)

  auto issue = [&](int gt) {  // both halves of tile gt; a half entirely past kc is skipped
    const int il = gt / KT, k0 = (gt % KT) * L;
    const bool h1 = k0 + LH < ks.kc;
    mbar_arrive_expect_tx(bar, h1 ? 2 * HALF_BYTES : HALF_BYTES);
    tma_load_5d(tile, &tmap, bar, 2 * k0, 0, il, 0, 0);
    if (h1) tma_load_5d(tile + C::HALF, &tmap, bar, 2 * (k0 + LH), 0, il, 0, 0);
  };

  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0 && blockIdx.x < NT) issue(blockIdx.x);
  bool first = true;
  for (int it = 0, gt = blockIdx.x; gt < NT; ++it, gt += gridDim.x) {
    mbar_wait(bar, it & 1);
    V v[E];
    const V* half = tile + grp * C::HALF;
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = half[(t + P * e) * LH + l];
    // Tile consumed: the last group's first warp requests the next one.
    if (tid / 32 == kIssueWarp) {
      named_sync(5, 2 * GT);
      const int gn = gt + gridDim.x;
      if ((tid & 31) == 0 && gn < NT) {
        fence_proxy_async_smem();
        issue(gn);
      }
    } else {
      named_arrive(5, 2 * GT);
    }
    ys_stages<N, E, LH, S, 0>(v, scr, stw, t, l, grp, first);
    const int il = gt / KT;
    const int k = (gt % KT) * L + grp * LH + l;
    if (k < ks.kc) {
#pragma unroll
      for (int e = 0; e < E; ++e) st_out(out + rowB(gout, il, t + P * e) * kq + k, v[e]);
    }
  }
  if (grp == 0 && !first) named_sync(4, 2 * GT);  // pairs with group 1's last "done" arrival
}

}  // namespace arena_fft
