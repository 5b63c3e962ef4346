// poisson_xtmem.cuh — the fused x pass (K3: forward FFT along i * Poisson symbol
// * backward FFT along i, fft_solver.cpp:65-80 first axis + the scale loop
// fft_solver.cpp:66-79) with the next tile staged in tensor memory.
//
// K3 at n = 1024 fp64 holds 32 points per thread (254 registers), so an SM runs
// one 8-warp CTA whose 128 KB tile buffer doubles as the FFT exchange scratch:
// with one buffer the next tile can only be requested after the last exchange
// and its load is partly exposed (r01: 4.4 ms, 59% of the HBM roofline).  Here
// the 128 KB of shared memory stay exchange scratch only, and the next tile
// streams in while the current one is transformed:
//
//   TMA (4 boxes of 256 positions x 8 lines, 32 KB) -> two 32 KB shared staging
//   buffers -> tcgen05.cp.128x256b -> TMEM (256 columns x 128 lanes = 128 KB)
//   -> tcgen05.ld.32x32b into the registers of the thread that owns them.
//
// Thread tid (line l = tid % 8, position group t = tid / 8; positions t + 32 e)
// owns TMEM lane tid % 128, columns 128 (tid / 128) + 4 e .. + 3 (one complex
// double per 4 columns): staging row lambda of piece q holds position
// 16 cb + lambda / 8 + 32 e, line lambda % 8 — rows 16 bytes apart, so every
// tcgen05.cp reads 128 consecutive 16-byte rows (no-swizzle descriptor, SBO 128 B)
// and its second 16-byte unit (e + 1) 4 KB further (LBO).
//
// Thread 0 runs the copy pipeline of the NEXT tile as an 8-step state machine
// (two TMA loads, two copies, two loads, two copies), advanced without blocking
// at every exchange barrier of the current tile's FFTs and finished after the
// stores; the TMEM loads of the next iteration wait on an mbarrier the last
// tcgen05.commit arrives on.
#pragma once

#include "poisson_pow2.cuh"
#include "tmem.cuh"

namespace arena_fft {

#ifndef ARENA_XTMEM_PF
#define ARENA_XTMEM_PF 1  // L2-prefetch pieces 2 and 3 of the next tile when its copy pipeline starts
#endif

struct XTmemCfg {
  static constexpr int N = 1024, E = 32, P = N / E, L = 8, THREADS = L * P;  // 256
  static constexpr int TILE = N * L;                     // complex doubles (128 KB)
  static constexpr int PIECE = 256;                      // positions per TMA box (tma_ib)
  static constexpr int NPIECE = N / PIECE;               // 4
  static constexpr int PIECE_BYTES = PIECE * L * 16;     // 32 KB
  static constexpr int TW = stage_tw_total(N, E);        // staged stage twiddles
  static constexpr int TMEM_COLS = 256;
  static constexpr int SMEM = (TILE + 2 * PIECE * L + TW) * 16 + 8 * 8 + 16;
};

template <typename T, int N>
__global__ void __launch_bounds__(XTmemCfg::THREADS, 1)
    k_xpass_tmem(const __grid_constant__ CUtensorMap tmap, vec2_t<T>* __restrict__ spec,
                 const vec2_t<T>* __restrict__ stw, T scale, T four_pi2) {
  static_assert(sizeof(T) == 8 && N == XTmemCfg::N, "the TMEM-staged x pass is the fp64 1024-point one");
  using V = vec2_t<T>;
  using C = XTmemCfg;
  static_assert(C::TMEM_COLS == (C::THREADS / 128) * 128, "one 128-column block per 128 threads");
  constexpr int E = C::E, P = C::P, L = C::L;
  constexpr Layout g = fixed_layout<N>();
  constexpr KSpan ks{N / 2 + 1, spec_pitch(N), 0};
  constexpr int KT = (ks.kc + L - 1) / L;
  constexpr int NT = g.nj * KT;
  constexpr int jbm = (1 << g.jbs) - 1;
  constexpr size_t kq = size_t(ks.kq);

  V* scratch = smem_base<V>();
  V* stg0 = scratch + C::TILE;
  V* stg1 = stg0 + C::PIECE * L;
  V* tws = stg1 + C::PIECE * L;
  uint64_t* full = reinterpret_cast<uint64_t*>(tws + C::TW);  // [2]: TMA of staging s landed
  uint64_t* cpd = full + 2;                                   // [2]: copies out of staging s done
  uint64_t* tmf = full + 4;                                   // TMEM holds the next tile
  uint32_t* taddr_s = reinterpret_cast<uint32_t*>(full + 5);
  const int tid = threadIdx.x;
  const int l = tid % L, t = tid / L, warp = tid / 32;

  if (tid == 0) {
    for (int b = 0; b < 5; ++b) mbar_init(&full[b], 1);
    fence_mbar_init();
  }
  for (int i = tid; i < C::TW; i += blockDim.x) tws[i] = __ldg(stw + i);
  if (warp == 0) tmem_alloc<C::TMEM_COLS>(taddr_s);
  tmem_fence_before();
  __syncthreads();
  tmem_fence_after();
  const uint32_t taddr = *taddr_s;
  const SmemTable<V> twp{tws};

  // ---- copy pipeline of one tile (thread 0 only)
  int pstep = 8, pgt = 0;
  uint32_t fullc0 = 0, fullc1 = 0, cpdc0 = 0, cpdc1 = 0, wait0 = 0, wait1 = 0;
  auto issue = [&](int gt, int q, int s) {
    const int outer = gt / KT, kt = gt % KT;
    uint64_t* b = &full[s];
    mbar_arrive_expect_tx(b, C::PIECE_BYTES);
    tma_load_5d(s ? stg1 : stg0, &tmap, b, 2 * kt * L, outer & jbm, q * C::PIECE, outer >> g.jbs, 0);
  };
  auto copy = [&](int q, int s) {
    const uint32_t base = smem_u32(s ? stg1 : stg0);
#pragma unroll
    for (int cb = 0; cb < 2; ++cb)
#pragma unroll
      for (int ep = 0; ep < 4; ++ep) {
        const int e = 8 * q + 2 * ep;
        tmem_cp_128x256b(taddr + uint32_t(128 * cb + 4 * e), tmem_sdesc(base + 2048 * cb + 8192 * ep, 4096, 128));
      }
  };
  auto advance = [&](bool block) {
    while (pstep < 8) {
      switch (pstep) {
        case 0:
          issue(pgt, 0, 0);
          if constexpr (ARENA_XTMEM_PF) {  // pieces 2, 3 into L2 now: their TMA loads later hit L2
            const int outer = pgt / KT, kt = pgt % KT;
            tma_prefetch_5d(&tmap, 2 * kt * L, outer & jbm, 2 * C::PIECE, outer >> g.jbs, 0);
            tma_prefetch_5d(&tmap, 2 * kt * L, outer & jbm, 3 * C::PIECE, outer >> g.jbs, 0);
          }
          break;
        case 1: issue(pgt, 1, 1); break;
        case 2:
        case 6:
          if (!block && !mbar_test(&full[0], fullc0 & 1)) return;
          mbar_wait(&full[0], fullc0 & 1);
          ++fullc0;
          tmem_fence_after();
          copy(pstep == 2 ? 0 : 2, 0);
          if (pstep == 2) wait0 = cpdc0;
          ++cpdc0;
          tmem_commit(&cpd[0]);
          break;
        case 3:
        case 7:
          if (!block && !mbar_test(&full[1], fullc1 & 1)) return;
          mbar_wait(&full[1], fullc1 & 1);
          ++fullc1;
          tmem_fence_after();
          copy(pstep == 3 ? 1 : 3, 1);
          if (pstep == 3) wait1 = cpdc1;
          ++cpdc1;
          tmem_commit(&cpd[1]);
          if (pstep == 7) tmem_commit(tmf);
          break;
        case 4:
          if (!block && !mbar_test(&cpd[0], wait0 & 1)) return;
          mbar_wait(&cpd[0], wait0 & 1);
          issue(pgt, 2, 0);
          break;
        case 5:
          if (!block && !mbar_test(&cpd[1], wait1 & 1)) return;
          mbar_wait(&cpd[1], wait1 & 1);
          issue(pgt, 3, 1);
          break;
      }
      ++pstep;
    }
  };

  if (tid == 0 && int(blockIdx.x) < NT) {
    pgt = blockIdx.x;
    pstep = 0;
    advance(true);
  }
  const uint32_t tl = taddr + (uint32_t(32 * (warp % 4)) << 16) + uint32_t(128 * (tid / 128));
  auto hook = [&]() {
    if (tid == 0) advance(false);
  };
  int it = 0;
  for (int gt = blockIdx.x; gt < NT; gt += gridDim.x, ++it) {
    mbar_wait(tmf, it & 1);
    tmem_fence_after();
    V v[E];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint32_t r[32];
      tmem_ld32(tl + uint32_t(32 * j), r);
      tmem_wait_ld();
#pragma unroll
      for (int m = 0; m < 8; ++m)
        v[8 * j + m] = V{__hiloint2double(int(r[4 * m + 1]), int(r[4 * m])),
                         __hiloint2double(int(r[4 * m + 3]), int(r[4 * m + 2]))};
    }
    tmem_fence_before();
    __syncthreads();  // TMEM free for the next tile; the scratch free of the last iteration's reads
    if (tid == 0) {
      const int gn = gt + int(gridDim.x);
      if (gn < NT) {
        tmem_fence_after();
        pgt = gn;
        pstep = 0;
        advance(false);
      }
    }
    const int outer = gt / KT;
    const int k = (gt % KT) * L + l;
    line_fft<N, E, L, -1>(v, scratch, twp, t, l, hook);
    const T kj = T(signed_freq(outer, N));
    const T kk = T(k);
    const T c = kj * kj + kk * kk;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const T ki = T(signed_freq(t + P * e, N));
      const T m = poisson_symbol(ki * ki + c, scale, four_pi2);
      v[e].x *= m;
      v[e].y *= m;
    }
    line_fft<N, E, L, +1>(v, scratch, twp, t, l, hook);
    if (k < ks.kc) {
#pragma unroll
      for (int e = 0; e < E; ++e) st_out(spec + rowC(g, t + P * e, outer) * kq + k, v[e]);
    }
    if (tid == 0) advance(true);
  }
  tmem_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<C::TMEM_COLS>(taddr);
}

}  // namespace arena_fft
