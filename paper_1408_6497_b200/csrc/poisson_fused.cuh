// poisson_fused.cuh — K1+K2 (forward) and K4+K5 (inverse) fused through L2.
//
// One persistent kernel per pair.  Work items are handed out in order by a
// global counter: per plane p the items of the first pass (forward: z-r2c rows,
// inverse: y-backward tiles) and — `lag` planes later — the items of the second
// pass, which spin until the plane's first-pass count is complete.  Items are
// dequeued in order and first-pass items never wait, so every awaited item is
// already resident and running: no deadlock.  With a lag of a few planes the
// awaited plane (8.5 MB at n = 1024) is still in the 126 MB L2, so the pair
// costs one HBM sweep (R + C bytes) instead of two (R + 3C).  The inverse z
// items drop the consumed spectrum rows from L2 (discard.global.L2) so the dead
// intermediate is never written back.
#pragma once

#include "poisson_pow2.cuh"

#ifndef ARENA_FUSED_LAG
#define ARENA_FUSED_LAG 2
#endif


namespace arena_fft {

template <typename T, int N>
struct FusedCfg {
  using TC = TmaCfg<T, N, false>;  // 128-thread tiles (its own y-box TMA map)
  static constexpr int VB = 2 * sizeof(T);
  static constexpr int THREADS = TC::THREADS;
  static constexpr int M = N / 2;
  static constexpr int EZ = imin(32, M);
  static constexpr int PZ = M / EZ;
  static constexpr int RW = imax(1, 32 / PZ);  // z rows per warp
  static constexpr int WARPS = THREADS / 32;
  static constexpr int ZROWS = RW * WARPS;     // rows per z item
  static constexpr int ZSM = (M + 1) * RW;     // shared elements per warp (z items)
  static constexpr int SMEM_ELEMS = imax(TC::TILE, ZSM * WARPS);
  static constexpr int SMEM = SMEM_ELEMS * VB + 32;
  static constexpr bool OK = (THREADS == 128 || THREADS == 256) && PZ <= 32 && (32 % PZ) == 0 &&
                             (N % ZROWS) == 0 && N >= 256;
  static constexpr int MINB = THREADS == 128 ? 2 : 1;  // co-resident CTAs (255 registers per thread)
};

struct FusedItem {
  int first, plane, sub;
};

// Item w of the in-order schedule: rounds r = 0 .. planes-1+lag; round r holds
// the first-pass items of plane r (if r < planes), then the second-pass items of
// plane r-lag (if r >= lag).
__host__ __device__ __forceinline__ FusedItem fused_decode(long long w, int planes, int c1, int c2, int lag) {
  const long long A = (long long)lag * c1;
  if (w < A) return {1, int(w / c1), int(w % c1)};
  w -= A;
  const long long mid = (long long)(planes - lag) * (c1 + c2);
  if (w < mid) {
    const int r = lag + int(w / (c1 + c2));
    const int s = int(w % (c1 + c2));
    return s < c1 ? FusedItem{1, r, s} : FusedItem{0, r - lag, s - c1};
  }
  w -= mid;
  return {0, planes - lag + int(w / c2), int(w % c2)};
}

// DIR -1: forward (z-r2c rows, then y-forward tiles); +1: inverse (y-backward
// tiles, then z-c2r rows).  ctrs[0] = work counter, ctrs[1 + p] = finished
// first-pass items of plane p (zeroed before the launch).
template <typename T, int N, int DIR>
__global__ void __launch_bounds__(FusedCfg<T, N>::THREADS, FusedCfg<T, N>::MINB)
    k_zy_fused(const __grid_constant__ CUtensorMap tmap, const T* __restrict__ f, T* __restrict__ u,
               vec2_t<T>* __restrict__ S, const vec2_t<T>* __restrict__ tw, const vec2_t<T>* __restrict__ stw_z,
               const vec2_t<T>* __restrict__ stw_y, Layout g, int* __restrict__ ctrs, int lag) {
  using V = vec2_t<T>;
  using F = FusedCfg<T, N>;
  using TC = TmaCfg<T, N, false>;  // 128-thread tiles (its own y-box TMA map)
  constexpr int E = TC::E, P = TC::P, L = TC::L, KT = TC::KT;
  constexpr int ncp = spec_pitch(N);
  constexpr uint32_t TILE_BYTES = TC::TILE * sizeof(V);
  constexpr int NZ = N / F::ZROWS, NY = KT;
  constexpr int C1 = DIR < 0 ? NZ : NY, C2 = DIR < 0 ? NY : NZ;
  V* sm = smem_base<V>();
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + F::SMEM_ELEMS);
  int* slot = reinterpret_cast<int*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int planes = g.ni;
  lag = lag < 1 ? 1 : (lag > planes ? planes : lag);
  const long long total = (long long)planes * (NZ + NY);
  int* done = ctrs + 1;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase = 0;
  for (;;) {
    if (tid == 0) *slot = atomicAdd(&ctrs[0], 1);
    __syncthreads();
    const long long w = *slot;
    __syncthreads();  // everyone has read the slot before thread 0 may refill it
    if (w >= total) break;
    const FusedItem it = fused_decode(w, planes, C1, C2, lag);
    if (!it.first) {
      if (tid == 0) {
        while (ld_acquire_gpu(&done[it.plane]) < C1) __nanosleep(128);
      }
      __syncthreads();
    }
    const bool is_z = (DIR < 0) == (it.first != 0);
    if (is_z) {
      const size_t row0 = size_t(it.plane) * N + size_t(it.sub) * F::ZROWS + size_t(warp) * F::RW;
      V* wsm = sm + warp * F::ZSM;
      if constexpr (DIR < 0)
        zfwd_rows<T, N, F::EZ, F::RW, kSyncWarp>(f, S, tw, stw_z, g, row0, wsm, lane);
      else
        zinv_rows<T, N, F::EZ, F::RW, kSyncWarp, true>(S, u, tw, stw_z, g, row0, wsm, lane);
    } else {
      const int l = tid % L, t = tid / L;
      const int il = it.plane, kt = it.sub;
      if (tid == 0) {
        fence_proxy_async_global();  // acquired generic-proxy writes before the TMA read
        fence_proxy_async_smem();    // this CTA's generic shared accesses before the TMA write
        mbar_arrive_expect_tx(bar, TILE_BYTES);
        ytile_half_load(sm, &tmap, bar, g, 1, 2 * kt * L, il, 0, 0, TILE_BYTES);
        ytile_half_load(sm, &tmap, bar, g, 1, 2 * kt * L, il, 0, 1, TILE_BYTES);
      }
      mbar_wait(bar, phase);
      phase ^= 1;
      V v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = sm[(t + P * e) * L + l];
      __syncthreads();
      line_fft<N, E, L, DIR>(v, sm, stw_y, t, l);
      const int k = kt * L + l;
      if (k < TC::NC) {
#pragma unroll
        for (int e = 0; e < E; ++e) S[rowB(g, il, t + P * e) * ncp + k] = v[e];
      }
    }
    if (it.first) __threadfence();  // this thread's results visible GPU-wide before the count
    __syncthreads();
    if (tid == 0 && it.first) atomicAdd(&done[it.plane], 1);
  }
}

}  // namespace arena_fft
