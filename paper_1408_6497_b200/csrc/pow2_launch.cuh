// pow2_launch.cuh — host-side launch sequence of the power-of-two path.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include <cudaTypedefs.h>

#include "launchers.h"
#include "poisson_fused.cuh"
#include "poisson_quad.cuh"
#include "poisson_qpencil.cuh"
#include "poisson_split3.cuh"

namespace arena_fft {

// Raise the dynamic shared-memory limit of a kernel once per device and pick
// the smallest shared-memory carveout that still holds every CTA the register
// file allows (the rest stays L1).  The kernel is a template argument so each
// instantiation has its own flag.
template <auto kernel>
inline cudaError_t ensure_smem(int bytes, int threads) {
  static std::atomic<unsigned long long> done_mask{0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const unsigned long long bit = 1ull << (dev & 63);
  if (done_mask.load(std::memory_order_relaxed) & bit) return cudaSuccess;
  if (bytes > 48 * 1024) {
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
  }
  int blocks = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, threads, bytes);
  if (e != cudaSuccess) return e;
  const int per_block = bytes + 1024;  // + driver-reserved shared memory per CTA
  int pct = (blocks * per_block * 100 + 228 * 1024 - 1) / (228 * 1024);
  pct = pct < 0 ? 0 : (pct > 100 ? 100 : pct);
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  if (e != cudaSuccess) return e;
  done_mask.fetch_or(bit);
  return cudaSuccess;
}

inline PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

#ifndef ARENA_Y_FIXED
#define ARENA_Y_FIXED 0  // single GPU: compile-time geometry for the y passes too (as the x pass)
#endif
#ifndef ARENA_TMA_PROMO
#define ARENA_TMA_PROMO 0  // L2 promotion of the TMA boxes: 0 none, 1 64B, 2 128B, 3 256B
#endif
// TMA descriptor of a workspace in Layout g (5-D, see k_strided_tma).
// ni_count / njb_count (0 = all): a sub-range view for the slab's chunked exchange —
// `spec` already advanced to the sub-range, strides those of the full layout g.
template <typename T, int N>
cudaError_t encode_map(void* out, void* spec, const Layout& g, int nchunks, bool ybox, int kc = N / 2 + 1,
                       int kq = spec_pitch(N), int ly = TmaCfg<T, N, true>::L, bool one_chunk = false,
                       int lx = TmaCfg<T, N, false, x_wide<T, false>()>::L, int ni_count = 0, int njb_count = 0) {
  const int LX = lx;
  const int LY = ly;
  auto enc = tensor_map_encoder();
  if (!enc) return cudaErrorNotSupported;
  const CUtensorMapDataType dt = sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
  const cuuint64_t row = cuuint64_t(kq) * 2 * sizeof(T);
  const int JB = 1 << g.jbs;
  const cuuint64_t dims[5] = {cuuint64_t(2 * kc), cuuint64_t(JB), cuuint64_t(ni_count ? ni_count : g.ni),
                              cuuint64_t(njb_count ? njb_count : g.nj / JB), cuuint64_t(nchunks)};
  const cuuint64_t strides[4] = {row, row * JB, row * JB * g.ni, row * g.ni * g.nj};
  const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  cuuint32_t box[5];
  if (ybox) {  // half a y tile (ytile_split; the kernels fetch a tile as two boxes)
    const int nch = one_chunk ? 1 : nchunks;
    const int sd = ytile_split(g, nch);
    if (sd == 4 && (nch & 1)) return cudaErrorInvalidValue;
    box[0] = 2 * LY; box[1] = JB; box[2] = 1; box[3] = (g.nj / JB) / (sd == 3 ? 2 : 1); box[4] = nch / (sd == 4 ? 2 : 1);
  } else {
    box[0] = 2 * LX; box[1] = 1; box[2] = tma_ib(g.ni); box[3] = 1; box[4] = 1;
  }
  for (int d = 1; d < 5; ++d)
    if (box[d] > 256) return cudaErrorInvalidValue;
  const CUtensorMapL2promotion promo = ARENA_TMA_PROMO == 1   ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                       : ARENA_TMA_PROMO == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                       : ARENA_TMA_PROMO == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                              : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(out), dt, 5, spec, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <typename T>
inline const vec2_t<T>* stw_ptr(const Pow2Args& a, int which, int E) {
  return static_cast<const vec2_t<T>*>(a.stw) + stw_offset(a.n, which, E);
}

template <typename T, int N, int PASS, bool PEER = false, bool FIXED = false, int SPL = 0>
cudaError_t launch_strided_tma(const Pow2Args& a, const CUtensorMap& map, void* spec, const Layout& g, T scale,
                               T four_pi2, KSpan ks = KSpan{N / 2 + 1, spec_pitch(N), 0}, void* out = nullptr,
                               const Layout* gout = nullptr, const PeerOut<vec2_t<T>>* po = nullptr) {
  using C = TmaCfg<T, N, (PASS < 2), PASS == 2 && x_wide<T, (SPL != 0)>()>;
  using V = vec2_t<T>;
  auto kern = k_strided_tma<T, N, PASS, PEER, FIXED, SPL>;
  constexpr int SMEM = PASS == 2 ? C::SMEM_X : C::SMEM_Y;
  cudaError_t e = ensure_smem<k_strided_tma<T, N, PASS, PEER, FIXED, SPL>>(SMEM, C::THREADS);
  if (e) return e;
  PeerOut<V> pov{};
  if (po) pov = *po;
  int per_sm = 1;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, SMEM))) return e;
  const int tiles = (ks.no ? ks.no : (PASS < 2 ? g.ni : g.nj)) * ((ks.kc + C::L - 1) / C::L) * spl_chunks(SPL);
  int grid = a.sm_count * (per_sm > 0 ? per_sm : 1);
  if (grid > tiles) grid = tiles;
  // stage twiddles of N-point lines: table `which` 1 (N = n), 0 (N = n/2: quadrant / split lines)
  kern<<<grid, C::THREADS, SMEM, a.stream>>>(map, static_cast<V*>(spec), stw_ptr<T>(a, N == a.n ? 1 : 0, C::E), scale, four_pi2, g,
                                               a.nchunks, a.j0, ks, static_cast<V*>(out ? out : spec),
                                               gout ? *gout : g, pov);
  return cudaGetLastError();
}

// Peer destinations of a scattering pass: chunk c -> peers[c] (rank c's
// workspace, already advanced to this rank's chunk); chunk_rows = ni * nj.
constexpr int kPeerMinN = 16;
template <typename V>
PeerOut<V> peer_table(void* const* peers, int nchunks, size_t chunk_rows) {
  PeerOut<V> po{};
  for (int c = 0; c < nchunks && c < kMaxPeers; ++c) po.base[c] = static_cast<V*>(peers[c]);
  int sh = 0;
  while ((size_t(1) << sh) < chunk_rows) ++sh;
  po.shift = sh;
  return po;
}

template <typename T, int N, int DIR>
cudaError_t launch_fused(const Pow2Args& a, const CUtensorMap& map, const Layout& g) {
  using F = FusedCfg<T, N>;
  using V = vec2_t<T>;
  auto kern = k_zy_fused<T, N, DIR>;
  cudaError_t e = ensure_smem<k_zy_fused<T, N, DIR>>(F::SMEM, F::THREADS);
  if (e) return e;
  if ((e = cudaMemsetAsync(a.ctrs, 0, sizeof(int) * size_t(g.ni + 1), a.stream))) return e;
  int per_sm = 1;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, F::THREADS, F::SMEM))) return e;
  const long long items = (long long)g.ni * (N / F::ZROWS + TmaCfg<T, N, false>::KT);
  long long grid = (long long)a.sm_count * (per_sm > 0 ? per_sm : 1);
  if (grid > items) grid = items;
  const V* stw_z = static_cast<const V*>(a.stw) + stw_offset(a.n, 0, F::EZ);
  const V* stw_y = static_cast<const V*>(a.stw) + stw_offset(a.n, 1, TmaCfg<T, N, false>::E);
  kern<<<unsigned(grid), F::THREADS, F::SMEM, a.stream>>>(map, static_cast<const T*>(a.f), static_cast<T*>(a.u),
                                                          static_cast<V*>(a.spec), static_cast<const V*>(a.tw),
                                                          stw_z, stw_y, g, a.ctrs, a.lag);
  return cudaGetLastError();
}

inline void mark(const Pow2Args& a, int i) {
  if (a.ev) cudaEventRecord(a.ev[i], a.stream);
}

// Single-GPU quadrant path (poisson_quad.cuh): K1q, then the H-point y / x / y
// TMA passes on the four quadrant chunks, then K5q.
template <typename T, int NR>
cudaError_t launch_quad(const Pow2Args& a) {
  if constexpr (!(QuadZCfg<T, NR>::OK && NR / 2 >= 8)) {
    return cudaErrorNotSupported;
  } else {
    constexpr int H = NR / 2;
    using V = vec2_t<T>;
    using QC = QuadZCfg<T, NR>;
    cudaError_t e;
    if (!a.tma || a.nchunks != 1 || a.specC != a.spec || a.ni != NR || a.nj != NR) return cudaErrorNotSupported;
    if (a.ncp != spec_pitch(NR) || a.nc != NR / 2 + 1) return cudaErrorInvalidValue;
    if ((e = ensure_smem<k_zfwd_quad<T, NR>>(QC::SMEM, QC::THREADS))) return e;
    if ((e = ensure_smem<k_zinv_quad<T, NR>>(QC::SMEM, QC::THREADS))) return e;
    const Layout gq = make_layout(H, H);
    const KSpan ks{NR / 2 + 1, spec_pitch(NR), 0};
    TmaCache* c = a.tma;
    if (c->specB != a.spec || c->specC != a.spec || c->n != NR || c->nchunks != 4 || c->quad != 1) {
      if ((e = encode_map<T, H>(c->maps[0], a.spec, gq, 4, true, ks.kc, ks.kq, TmaCfg<T, H, true>::L, true))) return e;
      if ((e = encode_map<T, H>(c->maps[1], a.spec, gq, 4, false, ks.kc, ks.kq, TmaCfg<T, H, true>::L, false,
                                TmaCfg<T, H, false, x_wide<T, true>()>::L)))
        return e;
      c->specB = c->specC = a.spec;
      c->n = NR;
      c->ni = c->nj = H;
      c->nchunks = 4;
      c->quad = 1;
    }
    const CUtensorMap* my = reinterpret_cast<const CUtensorMap*>(c->maps[0]);
    const CUtensorMap* mx = reinterpret_cast<const CUtensorMap*>(c->maps[1]);
    const T scale = T(1.0 / (double(NR) * NR * NR));  // fft_solver.cpp:67
    const T four_pi2 = T(4.0 * M_PI * M_PI);           // fft_solver.cpp:66
    const V* tw = static_cast<const V*>(a.tw);
    V* S = static_cast<V*>(a.spec);
    const unsigned qgrid = unsigned(H) * H;
    int mk = 0;
    if (a.phases & kPhaseZY) {
      mark(a, mk++);
      k_zfwd_quad<T, NR><<<qgrid, QC::THREADS, QC::SMEM, a.stream>>>(static_cast<const T*>(a.f), S, tw,
                                                                     stw_ptr<T>(a, 0, QC::E), gq);
      mark(a, mk++);
      if ((e = launch_strided_tma<T, H, 0, false, false, 2>(a, *my, a.spec, gq, scale, four_pi2, ks))) return e;
    }
    if (a.phases & kPhaseX) {
      mark(a, mk++);
      // compile-time quadrant geometry for the x pass, as the single-GPU x pass (FIXED)
      if ((e = launch_strided_tma<T, H, 2, false, true, 2>(a, *mx, a.spec, gq, scale, four_pi2, ks))) return e;
    }
    if (a.phases & kPhaseYZ) {
      mark(a, mk++);
      if ((e = launch_strided_tma<T, H, 1, false, false, 2>(a, *my, a.spec, gq, scale, four_pi2, ks))) return e;
      mark(a, mk++);
      k_zinv_quad<T, NR><<<qgrid, QC::THREADS, QC::SMEM, a.stream>>>(S, static_cast<T*>(a.u), tw,
                                                                     stw_ptr<T>(a, 0, QC::E), gq);
      mark(a, mk++);
    }
    return cudaGetLastError();
  }
}

// Radix-3 split path (poisson_split3.cuh): generic z r2c, split, M-point y / x / y
// TMA passes on the nine chunks, merge, generic z c2r.
template <typename T, int R, int M>
cudaError_t launch_split3_m(const Split3Args& s) {
  using V = vec2_t<T>;
  constexpr int CH = R * R;  // chunks
  cudaError_t e;
  const int n = s.n;
  if (n != R * M || !s.tma) return cudaErrorInvalidValue;
  const Layout gq = make_layout(M, M);
  const KSpan ks{s.nc, s.ncp, 0};
  TmaCache* c = s.tma;
  if (c->specB != s.Q || c->n != n || c->nchunks != CH) {
    if ((e = encode_map<T, M>(c->maps[0], s.Q, gq, CH, true, ks.kc, ks.kq, TmaCfg<T, M, true>::L, true))) return e;
    if ((e = encode_map<T, M>(c->maps[1], s.Q, gq, CH, false, ks.kc, ks.kq, TmaCfg<T, M, true>::L, false,
                              TmaCfg<T, M, false, x_wide<T, true>()>::L)))
      return e;
    c->specB = c->specC = s.Q;
    c->n = n;
    c->ni = c->nj = M;
    c->nchunks = CH;
    c->quad = R;
  }
  const CUtensorMap* my = reinterpret_cast<const CUtensorMap*>(c->maps[0]);
  const CUtensorMap* mx = reinterpret_cast<const CUtensorMap*>(c->maps[1]);
  const T scale = T(1.0 / (double(n) * n * n));  // fft_solver.cpp:67
  const T four_pi2 = T(4.0 * M_PI * M_PI);       // fft_solver.cpp:66
  // the strided kernels read the M-point stage tables through a (n' = 2M) plan's offsets
  Pow2Args a{};
  a.stw = s.stw;
  a.n = 2 * M;
  a.stream = s.stream;
  a.sm_count = s.sm_count;
  a.nchunks = 1;
  const GenArgs ga{s.gplan, s.tw, n, s.nc, s.ncp, s.stream, nullptr};
  auto mk = [&](int i) {
    if (s.ev) cudaEventRecord(s.ev[i], s.stream);
  };
  const unsigned grid = unsigned(M) * M;
  constexpr int MH = M / 2;
  using ZC = SplitZCfg<T, R, MH>;
  const long long nrows = (long long)n * n;
  const unsigned zgrid = unsigned((nrows + ZC::L - 1) / ZC::L);
  const V* stwz = static_cast<const V*>(s.stwz) + stw_offset(M, 0, ZC::E);
  if ((e = ensure_smem<k_zfwd_split<T, R, MH>>(ZC::SMEM, ZC::THREADS))) return e;
  if ((e = ensure_smem<k_zinv_split<T, R, MH>>(ZC::SMEM, ZC::THREADS))) return e;
  mk(0);
  if (s.stwz) {
    k_zfwd_split<T, R, MH><<<zgrid, ZC::THREADS, ZC::SMEM, s.stream>>>(static_cast<const T*>(s.f), static_cast<V*>(s.S),
                                                                       static_cast<const V*>(s.tw), stwz, s.ncp, nrows);
  } else if ((e = sizeof(T) == 8 ? gen_z_r2c_f64(ga, s.f, s.S) : gen_z_r2c_f32(ga, s.f, s.S))) {
    return e;
  }
  mk(1);
  k_split3_fwd<T, R><<<grid, 128, 0, s.stream>>>(static_cast<const V*>(s.S), static_cast<V*>(s.Q),
                                               static_cast<const V*>(s.tw), n, M, s.nc, s.ncp, gq);
  mk(2);
  if ((e = launch_strided_tma<T, M, 0, false, false, R>(a, *my, s.Q, gq, scale, four_pi2, ks))) return e;
  mk(3);
  if ((e = launch_strided_tma<T, M, 2, false, false, R>(a, *mx, s.Q, gq, scale, four_pi2, ks))) return e;
  mk(4);
  if ((e = launch_strided_tma<T, M, 1, false, false, R>(a, *my, s.Q, gq, scale, four_pi2, ks))) return e;
  mk(5);
  k_split3_inv<T, R><<<grid, 128, 0, s.stream>>>(static_cast<const V*>(s.Q), static_cast<V*>(s.S),
                                               static_cast<const V*>(s.tw), n, M, s.nc, s.ncp, gq);
  mk(6);
  if (s.stwz) {
    k_zinv_split<T, R, MH><<<zgrid, ZC::THREADS, ZC::SMEM, s.stream>>>(static_cast<const V*>(s.S), static_cast<T*>(s.u),
                                                                       static_cast<const V*>(s.tw), stwz, s.ncp, nrows);
  } else if ((e = sizeof(T) == 8 ? gen_z_c2r_f64(ga, s.S, s.u) : gen_z_c2r_f32(ga, s.S, s.u))) {
    return e;
  }
  mk(7);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_split3(const Split3Args& s) {
  if (s.R == 3) {
    switch (s.M) {
      case 16: return launch_split3_m<T, 3, 16>(s);
      case 32: return launch_split3_m<T, 3, 32>(s);
      case 64: return launch_split3_m<T, 3, 64>(s);
      case 128: return launch_split3_m<T, 3, 128>(s);
      case 256: return launch_split3_m<T, 3, 256>(s);
      case 512: return launch_split3_m<T, 3, 512>(s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (s.R == 5) {
    switch (s.M) {
      case 16: return launch_split3_m<T, 5, 16>(s);
      case 32: return launch_split3_m<T, 5, 32>(s);
      case 64: return launch_split3_m<T, 5, 64>(s);
      case 128: return launch_split3_m<T, 5, 128>(s);
      case 256: return launch_split3_m<T, 5, 256>(s);
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaErrorInvalidValue;
}

template <typename T, int NR>
cudaError_t launch_pow2_n(const Pow2Args& a) {
  if (a.quad == 1) return launch_quad<T, NR>(a);
  using V = vec2_t<T>;
  using CC = ContigCfg<T, NR>;
  using SC = StridedCfg<T, NR, 0>;
  using XC = StridedCfg<T, NR, 1>;
  const V* tw = static_cast<const V*>(a.tw);
  V* S = static_cast<V*>(a.spec);
  cudaError_t e;
  static_assert((size_t(NR) * NR) % CC::L == 0, "rows per CTA must divide n^2");
  if (a.ncp != spec_pitch(NR) || a.nc != NR / 2 + 1) return cudaErrorInvalidValue;
  if (size_t(a.ni) * NR % CC::L) return cudaErrorInvalidValue;
  if ((e = ensure_smem<k_zfwd<T, NR>>(CC::SMEM, CC::THREADS))) return e;
  if ((e = ensure_smem<k_zinv<T, NR>>(CC::SMEM, CC::THREADS))) return e;
  if ((e = ensure_smem<k_zfwd<T, NR, true>>(CC::SMEM, CC::THREADS))) return e;
  if ((e = ensure_smem<k_zinv<T, NR, true>>(CC::SMEM, CC::THREADS))) return e;
  const Layout gB = make_layout(a.ni, NR / a.nchunks);  // (local i, global j) chunks of nj
  const Layout gC = make_layout(NR / a.nchunks, a.nj);  // (global i, local j) chunks of ni
  const unsigned zgrid = unsigned((size_t(a.ni) * NR) / CC::L);
  const T scale = T(1.0 / (double(NR) * NR * NR));  // fft_solver.cpp:67
  const T four_pi2 = T(4.0 * M_PI * M_PI);           // fft_solver.cpp:66
  const bool tma = a.tma != nullptr && NR >= 4;
  if (!tma && a.nchunks != 1) return cudaErrorNotSupported;  // classic kernels are single-GPU only
  if (tma) {
    TmaCache* c = a.tma;
    if (c->specB != a.spec || c->specC != a.specC || c->n != NR || c->ni != a.ni || c->nj != a.nj ||
        c->nchunks != a.nchunks || c->quad) {
      if ((e = encode_map<T, NR>(c->maps[0], a.spec, gB, a.nchunks, true))) return e;
      if ((e = encode_map<T, NR>(c->maps[1], a.specC, gC, a.nchunks, false))) return e;
      if ((e = encode_map<T, NR>(c->maps[2], a.spec, gB, a.nchunks, true, NR / 2 + 1, spec_pitch(NR),
                                 TmaCfg<T, NR, false>::L)))
        return e;
      c->specB = a.spec;
      c->specC = a.specC;
      c->n = NR;
      c->ni = a.ni;
      c->nj = a.nj;
      c->nchunks = a.nchunks;
      c->quad = 0;
    }
  }
  const CUtensorMap* my = tma ? reinterpret_cast<const CUtensorMap*>(a.tma->maps[0]) : nullptr;
  const CUtensorMap* mx = tma ? reinterpret_cast<const CUtensorMap*>(a.tma->maps[1]) : nullptr;
  const CUtensorMap* mf = tma ? reinterpret_cast<const CUtensorMap*>(a.tma->maps[2]) : nullptr;
  const KSpan kfull{NR / 2 + 1, spec_pitch(NR), 0};
  // one GPU, in place: the x kernel's compile-time geometry (FIXED) applies (B200
  // 1024^3: x 4.53 -> 4.32 ms fp64, 2.57 -> 2.20 ms fp32; the y passes measured
  // slower that way, 1.72 -> 2.06 ms fp32, and keep the runtime geometry)
  const bool single = a.nchunks == 1 && a.ni == NR && a.nj == NR && a.specC == a.spec && a.j0 == 0;
  int mk = 0;
  const bool fused = tma && a.ctrs != nullptr && FusedCfg<T, NR>::OK && !a.peer_y;
  // Sub-range launches of the slab's chunked exchange (a.subn > 0, one phase): K1 + K2 on
  // local i planes [sub0, sub0 + subn), or K3 on local j lines [sub0, sub0 + subn) (whole
  // JB blocks).  Rows of layout B are linear in il (rowB(g, il0 + il, j) = rowB(g, il, j) +
  // il0 JB) and rows of layout C in whole j blocks, so a sub-range is the full layout's
  // kernels on advanced bases, with TMA views of the sub-range's extent.
  if (a.subn > 0) {
    if (!tma || fused || a.peer_y || a.peer_x || single) return cudaErrorNotSupported;
    const size_t ncp = size_t(spec_pitch(NR));
    if (a.phases == kPhaseZY) {
      const int JB = 1 << gB.jbs;
      if (a.sub0 < 0 || a.sub0 + a.subn > a.ni) return cudaErrorInvalidValue;
      V* Ssub = S + size_t(a.sub0) * JB * ncp;
      k_zfwd<T, NR><<<unsigned(size_t(a.subn) * NR / CC::L), CC::THREADS, CC::SMEM, a.stream>>>(
          static_cast<const T*>(a.f) + size_t(a.sub0) * NR * NR, Ssub, tw, stw_ptr<T>(a, 0, CC::E), gB);
      alignas(64) CUtensorMap m;
      if ((e = encode_map<T, NR>(&m, Ssub, gB, a.nchunks, true, NR / 2 + 1, spec_pitch(NR), TmaCfg<T, NR, true>::L,
                                 false, TmaCfg<T, NR, false, x_wide<T, false>()>::L, a.subn)))
        return e;
      KSpan ks{NR / 2 + 1, spec_pitch(NR), 0};
      ks.no = a.subn;
      return launch_strided_tma<T, NR, 0>(a, m, Ssub, gB, scale, four_pi2, ks);
    }
    if (a.phases == kPhaseX) {
      const int JB = 1 << gC.jbs;
      if (a.sub0 % JB || a.subn % JB || a.sub0 + a.subn > a.nj) return cudaErrorInvalidValue;
      V* Csub = static_cast<V*>(a.specC) + size_t(a.sub0 / JB) * gC.ni * JB * ncp;
      alignas(64) CUtensorMap m;
      if ((e = encode_map<T, NR>(&m, Csub, gC, a.nchunks, false, NR / 2 + 1, spec_pitch(NR), TmaCfg<T, NR, true>::L,
                                 false, TmaCfg<T, NR, false, x_wide<T, false>()>::L, 0, a.subn / JB)))
        return e;
      Pow2Args a2 = a;
      a2.j0 = a.j0 + a.sub0;  // global j of the sub-range's first line (symbol)
      KSpan ks{NR / 2 + 1, spec_pitch(NR), 0};
      ks.no = a.subn;
      return launch_strided_tma<T, NR, 2>(a2, m, Csub, gC, scale, four_pi2, ks);
    }
    return cudaErrorInvalidValue;
  }
  if (fused && (a.fuse & kFuseFwd) && (a.phases & kPhaseZY)) {
    mark(a, mk++);
    if constexpr (FusedCfg<T, NR>::OK) {
      if ((e = launch_fused<T, NR, -1>(a, *mf, gB))) return e;
    }
  } else if (a.phases & kPhaseZY) {
    mark(a, mk++);
    if (single)
      k_zfwd<T, NR, true><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(static_cast<const T*>(a.f), S, tw,
                                                                     stw_ptr<T>(a, 0, CC::E), gB);
    else
      k_zfwd<T, NR><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(static_cast<const T*>(a.f), S, tw,
                                                                 stw_ptr<T>(a, 0, CC::E), gB);
    mark(a, mk++);
    if (tma && a.peer_y) {
      if constexpr (NR >= kPeerMinN) {
        const PeerOut<V> po = peer_table<V>(a.peer_y, a.nchunks, size_t(a.ni) * a.nj);
        e = launch_strided_tma<T, NR, 0, true>(a, *my, a.spec, gB, scale, four_pi2, kfull, nullptr, nullptr, &po);
      } else {
        e = cudaErrorNotSupported;
      }
      if (e) return e;
    } else if (tma) {
      if (ARENA_Y_FIXED && single) e = launch_strided_tma<T, NR, 0, false, true>(a, *my, a.spec, gB, scale, four_pi2);
      else e = launch_strided_tma<T, NR, 0>(a, *my, a.spec, gB, scale, four_pi2);
      if (e) return e;
    } else {
      if ((e = ensure_smem<k_ypass<T, NR, -1>>(SC::SMEM, SC::THREADS))) return e;
      k_ypass<T, NR, -1><<<dim3((a.nc + SC::L - 1) / SC::L, NR), SC::THREADS, SC::SMEM, a.stream>>>(
          S, stw_ptr<T>(a, 1, SC::E), gB);
    }
  }
  if (a.phases & kPhaseX) {
    mark(a, mk++);
    if (tma && a.peer_x) {
      if constexpr (NR >= kPeerMinN) {
        const PeerOut<V> po = peer_table<V>(a.peer_x, a.nchunks, size_t(a.ni) * a.nj);
        e = launch_strided_tma<T, NR, 2, true>(a, *mx, a.specC, gC, scale, four_pi2, kfull, nullptr, nullptr, &po);
      } else {
        e = cudaErrorNotSupported;
      }
      if (e) return e;
    } else if (tma) {
      if (single) e = launch_strided_tma<T, NR, 2, false, true>(a, *mx, a.specC, gC, scale, four_pi2);
      else e = launch_strided_tma<T, NR, 2>(a, *mx, a.specC, gC, scale, four_pi2);
      if (e) return e;
    } else {
      if ((e = ensure_smem<k_xmid<T, NR>>(XC::SMEM, XC::THREADS))) return e;
      k_xmid<T, NR><<<dim3((a.nc + XC::L - 1) / XC::L, NR), XC::THREADS, XC::SMEM, a.stream>>>(
          S, stw_ptr<T>(a, 1, XC::E), scale, four_pi2, gC);
    }
  }
  if (fused && (a.fuse & kFuseInv) && (a.phases & kPhaseYZ)) {
    mark(a, mk++);
    if constexpr (FusedCfg<T, NR>::OK) {
      if ((e = launch_fused<T, NR, +1>(a, *mf, gB))) return e;
    }
    mark(a, mk++);
  } else if (a.phases & kPhaseYZ) {
    mark(a, mk++);
    if (tma) {
      if (ARENA_Y_FIXED && single) e = launch_strided_tma<T, NR, 1, false, true>(a, *my, a.spec, gB, scale, four_pi2);
      else e = launch_strided_tma<T, NR, 1>(a, *my, a.spec, gB, scale, four_pi2);
      if (e) return e;
    } else {
      if ((e = ensure_smem<k_ypass<T, NR, +1>>(SC::SMEM, SC::THREADS))) return e;
      k_ypass<T, NR, +1><<<dim3((a.nc + SC::L - 1) / SC::L, NR), SC::THREADS, SC::SMEM, a.stream>>>(
          S, stw_ptr<T>(a, 1, SC::E), gB);
    }
    mark(a, mk++);
    if (single)
      k_zinv<T, NR, true><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(S, static_cast<T*>(a.u), tw,
                                                                     stw_ptr<T>(a, 0, CC::E), gB);
    else
      k_zinv<T, NR><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(S, static_cast<T*>(a.u), tw,
                                                                 stw_ptr<T>(a, 0, CC::E), gB);
    mark(a, mk++);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- pencil
template <typename T, int NR>
cudaError_t pencil_phase_n(const PencilArgs& a, int phase) {
  using V = vec2_t<T>;
  using CC = ContigCfg<T, NR>;
  const int ni = NR / a.Pr, nj = NR / a.Pc, nj2 = NR / a.Pr;
  const int nc = NR / 2 + 1;
  const KSpan ks{imin(a.kq, nc - a.c * a.kq), a.kq, a.c * a.kq};
  const bool has_k = ks.kc > 0;
  const Layout gz = make_layout(ni, nj);   // rows of the rank's f block / R chunks
  const Layout gY = make_layout(ni, nj);   // Y: j chunks of n/Pc (Pc chunks)
  const Layout gB2 = make_layout(ni, nj2); // B2: j chunks of n/Pr (Pr chunks)
  const Layout gC = make_layout(ni, nj2);  // C: i chunks of n/Pr, local j n/Pr (Pr chunks)
  const T scale = T(1.0 / (double(NR) * NR * NR));
  const T four_pi2 = T(4.0 * M_PI * M_PI);
  Pow2Args pa{};  // carries the launch context the TMA launcher reads
  pa.n = NR;
  pa.stw = a.stw;
  pa.stream = a.stream;
  pa.sm_count = a.sm_count;
  pa.j0 = a.r * nj2;
  cudaError_t e;
  if (has_k && (a.tma->specB != a.buf2 || a.tma->n != NR || a.tma->ni != ni || a.tma->nj != nj ||
                a.tma->nchunks != a.Pc)) {
    if ((e = encode_map<T, NR>(a.tma->maps[0], a.buf2, gY, a.Pc, true, ks.kc, ks.kq))) return e;
    if ((e = encode_map<T, NR>(a.tma->maps[1], a.buf2, gC, a.Pr, false, ks.kc, ks.kq))) return e;
    if ((e = encode_map<T, NR>(a.tma2->maps[0], a.buf1, gB2, a.Pr, true, ks.kc, ks.kq))) return e;
    if ((e = encode_map<T, NR>(a.tma2->maps[1], a.buf1, gC, a.Pr, false, ks.kc, ks.kq))) return e;
    if ((e = encode_map<T, NR>(a.tma2->maps[2], a.buf2, gB2, a.Pr, true, ks.kc, ks.kq))) return e;
    a.tma->specB = a.buf2;
    a.tma->n = NR;
    a.tma->ni = ni;
    a.tma->nj = nj;
    a.tma->nchunks = a.Pc;
  }
  const CUtensorMap& mY = *reinterpret_cast<const CUtensorMap*>(a.tma->maps[0]);
  const CUtensorMap& mC = *reinterpret_cast<const CUtensorMap*>(a.tma->maps[1]);
  const CUtensorMap& mB2 = *reinterpret_cast<const CUtensorMap*>(a.tma2->maps[0]);
  const CUtensorMap& mC1 = *reinterpret_cast<const CUtensorMap*>(a.tma2->maps[1]);   // peer: C in buf1
  const CUtensorMap& mB2b = *reinterpret_cast<const CUtensorMap*>(a.tma2->maps[2]);  // peer: B2 in buf2
  const bool peer = a.pz != nullptr;
  const size_t rows_row = size_t(ni) * nj, rows_col = size_t(ni) * nj2;  // rows per row / column chunk
  const V* tw = static_cast<const V*>(a.tw);
  const V* stwz = static_cast<const V*>(a.stw) + stw_offset(NR, 0, CC::E);
  const unsigned zgrid = unsigned((size_t(ni) * nj) / CC::L);
  switch (phase) {
    case kPencilZ1:
      if (peer) {
        if ((e = ensure_smem<k_zfwd_pencil<T, NR, true>>(CC::SMEM, CC::THREADS))) return e;
        const PeerOut<V> po = peer_table<V>(a.pz, a.Pc, rows_row);
        k_zfwd_pencil<T, NR, true><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(static_cast<const T*>(a.f), nullptr,
                                                                                tw, stwz, gz, a.kq, po);
        break;
      }
      if ((e = ensure_smem<k_zfwd_pencil<T, NR>>(CC::SMEM, CC::THREADS))) return e;
      k_zfwd_pencil<T, NR><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(static_cast<const T*>(a.f),
                                                                      static_cast<V*>(a.buf1), tw, stwz, gz, a.kq,
                                                                      PeerOut<V>{});
      break;
    case kPencilY1:  // Y (buf2) -> B2 (buf1); peer: -> column peers' C (buf1)
      if (!has_k) break;
      pa.nchunks = a.Pc;
      if (peer) {
        const PeerOut<V> po = peer_table<V>(a.py1, a.Pr, rows_col);
        e = launch_strided_tma<T, NR, 0, true>(pa, mY, a.buf2, gY, scale, four_pi2, ks, nullptr, &gB2, &po);
      } else {
        e = launch_strided_tma<T, NR, 0>(pa, mY, a.buf2, gY, scale, four_pi2, ks, a.buf1, &gB2);
      }
      if (e) return e;
      break;
    case kPencilX:  // C (buf2) in place; peer: C (buf1) -> column peers' B2 (buf2)
      if (!has_k) break;
      pa.nchunks = a.Pr;
      if (peer) {
        const PeerOut<V> po = peer_table<V>(a.px, a.Pr, rows_col);
        e = launch_strided_tma<T, NR, 2, true>(pa, mC1, a.buf1, gC, scale, four_pi2, ks, nullptr, nullptr, &po);
      } else {
        e = launch_strided_tma<T, NR, 2>(pa, mC, a.buf2, gC, scale, four_pi2, ks);
      }
      if (e) return e;
      break;
    case kPencilY2:  // B2 (buf1) -> Y (buf2); peer: B2 (buf2) -> row peers' R (buf1)
      if (!has_k) break;
      pa.nchunks = a.Pr;
      if (peer) {
        const PeerOut<V> po = peer_table<V>(a.py2, a.Pc, rows_row);
        e = launch_strided_tma<T, NR, 1, true>(pa, mB2b, a.buf2, gB2, scale, four_pi2, ks, nullptr, &gY, &po);
      } else {
        e = launch_strided_tma<T, NR, 1>(pa, mB2, a.buf1, gB2, scale, four_pi2, ks, a.buf2, &gY);
      }
      if (e) return e;
      break;
    case kPencilZ2:
      if ((e = ensure_smem<k_zinv_pencil<T, NR>>(CC::SMEM, CC::THREADS))) return e;
      k_zinv_pencil<T, NR><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(static_cast<const V*>(a.buf1),
                                                                      static_cast<T*>(a.u), tw, stwz, gz, a.kq);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// Folded pencil (poisson_qpencil.cuh): K1q / K5q on the rank's folded block, and per
// quadrant q = 2 ci + cj the plain pencil's strided passes of the H = n/2 problem
// (H-point lines, the n grid's k chunks), quadrant q's regions of buf1 / buf2 at q qstride.
template <typename T, int NR>
cudaError_t pencil_fold_phase_n(const PencilArgs& a, int phase) {
  constexpr int H = NR / 2;
  using QC = QuadZCfg<T, NR>;
  if constexpr (!(QC::OK && H >= 32)) {
    return cudaErrorNotSupported;
  } else {
    using V = vec2_t<T>;
    const int ni = H / a.Pr, nj = H / a.Pc, nj2 = H / a.Pr;
    const int nc = NR / 2 + 1;
    KSpan ks{imin(a.kq, nc - a.c * a.kq), a.kq, a.c * a.kq};
    ks.fm = 1;
    const bool has_k = ks.kc > 0;
    const Layout gz = make_layout(ni, nj);
    const Layout gY = make_layout(ni, nj), gB2 = make_layout(ni, nj2), gC = make_layout(ni, nj2);
    const T scale = T(1.0 / (double(NR) * NR * NR));
    const T four_pi2 = T(4.0 * M_PI * M_PI);
    Pow2Args pa{};
    pa.n = NR;  // H-point lines read the n/2 stage tables
    pa.stw = a.stw;
    pa.stream = a.stream;
    pa.sm_count = a.sm_count;
    pa.j0 = a.r * nj2;
    const size_t qs = size_t(ni) * H * a.kq;  // complex per quadrant region
    V* b1 = static_cast<V*>(a.buf1);
    V* b2 = static_cast<V*>(a.buf2);
    const V* tw = static_cast<const V*>(a.tw);
    cudaError_t e;
    if ((e = ensure_smem<k_zfwd_qpencil<T, NR>>(QC::SMEM, QC::THREADS))) return e;
    if ((e = ensure_smem<k_zfwd_qpencil<T, NR, true>>(QC::SMEM, QC::THREADS))) return e;
    if ((e = ensure_smem<k_zinv_qpencil<T, NR>>(QC::SMEM, QC::THREADS))) return e;
    alignas(64) CUtensorMap m;
    // Peer exchange (as the plain pencil: K1 -> row peers' buf2, K2 -> column peers' buf1,
    // K3 -> column peers' buf2, K4 -> row peers' buf1), quadrant q at q qs in every buffer.
    const bool peer = a.pz != nullptr;
    const size_t rows_row = size_t(ni) * nj, rows_col = size_t(ni) * nj2;
    auto qtable = [&](void* const* peers, int np, size_t chunk_rows, int q) {
      void* adv[kMaxPeers] = {};
      for (int c = 0; c < np && c < kMaxPeers; ++c) adv[c] = static_cast<V*>(peers[c]) + q * qs;
      return peer_table<V>(adv, np, chunk_rows);
    };
    switch (phase) {
      case kPencilZ1:
        if (peer) {
          k_zfwd_qpencil<T, NR, true><<<unsigned(ni) * nj, QC::THREADS, QC::SMEM, a.stream>>>(
              static_cast<const T*>(a.f), nullptr, tw, stw_ptr<T>(pa, 0, QC::E), gz, a.r * ni, a.c * nj, a.kq, qs,
              qtable(a.pz, a.Pc, rows_row, 0));
        } else {
          k_zfwd_qpencil<T, NR><<<unsigned(ni) * nj, QC::THREADS, QC::SMEM, a.stream>>>(
              static_cast<const T*>(a.f), b1, tw, stw_ptr<T>(pa, 0, QC::E), gz, a.r * ni, a.c * nj, a.kq, qs,
              PeerOut<V>{});
        }
        break;
      case kPencilY1:  // Y (buf2) -> B2 (buf1); peer: -> column peers' C (buf1), per quadrant
        if (!has_k) break;
        pa.nchunks = a.Pc;
        for (int q = 0; q < 4; ++q) {
          ks.fci = q >> 1;
          ks.fcj = q & 1;
          if ((e = encode_map<T, H>(&m, b2 + q * qs, gY, a.Pc, true, ks.kc, ks.kq))) return e;
          if (peer) {
            const PeerOut<V> po = qtable(a.py1, a.Pr, rows_col, q);
            e = launch_strided_tma<T, H, 0, true>(pa, m, b2 + q * qs, gY, scale, four_pi2, ks, nullptr, &gB2, &po);
          } else {
            e = launch_strided_tma<T, H, 0>(pa, m, b2 + q * qs, gY, scale, four_pi2, ks, b1 + q * qs, &gB2);
          }
          if (e) return e;
        }
        break;
      case kPencilX:  // C (buf2) in place; peer: C (buf1) -> column peers' B2 (buf2), per quadrant
        if (!has_k) break;
        pa.nchunks = a.Pr;
        for (int q = 0; q < 4; ++q) {
          ks.fci = q >> 1;
          ks.fcj = q & 1;
          V* cq = (peer ? b1 : b2) + q * qs;
          if ((e = encode_map<T, H>(&m, cq, gC, a.Pr, false, ks.kc, ks.kq))) return e;
          if (peer) {
            const PeerOut<V> po = qtable(a.px, a.Pr, rows_col, q);
            e = launch_strided_tma<T, H, 2, true>(pa, m, cq, gC, scale, four_pi2, ks, nullptr, nullptr, &po);
          } else {
            e = launch_strided_tma<T, H, 2>(pa, m, cq, gC, scale, four_pi2, ks);
          }
          if (e) return e;
        }
        break;
      case kPencilY2:  // B2 (buf1) -> Y (buf2); peer: B2 (buf2) -> row peers' R (buf1), per quadrant
        if (!has_k) break;
        pa.nchunks = a.Pr;
        for (int q = 0; q < 4; ++q) {
          ks.fci = q >> 1;
          ks.fcj = q & 1;
          V* bq = (peer ? b2 : b1) + q * qs;
          if ((e = encode_map<T, H>(&m, bq, gB2, a.Pr, true, ks.kc, ks.kq))) return e;
          if (peer) {
            const PeerOut<V> po = qtable(a.py2, a.Pc, rows_row, q);
            e = launch_strided_tma<T, H, 1, true>(pa, m, bq, gB2, scale, four_pi2, ks, nullptr, &gY, &po);
          } else {
            e = launch_strided_tma<T, H, 1>(pa, m, bq, gB2, scale, four_pi2, ks, b2 + q * qs, &gY);
          }
          if (e) return e;
        }
        break;
      case kPencilZ2:
        k_zinv_qpencil<T, NR><<<unsigned(ni) * nj, QC::THREADS, QC::SMEM, a.stream>>>(
            b1, static_cast<T*>(a.u), tw, stw_ptr<T>(pa, 0, QC::E), gz, a.r * ni, a.c * nj, a.kq, qs);
        break;
      default:
        return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
  }
}

template <typename T>
cudaError_t pencil_phase(const PencilArgs& a, int phase) {
  if (a.fold) {
    switch (a.n) {
      case 64: return pencil_fold_phase_n<T, 64>(a, phase);
      case 128: return pencil_fold_phase_n<T, 128>(a, phase);
      case 256: return pencil_fold_phase_n<T, 256>(a, phase);
      case 512: return pencil_fold_phase_n<T, 512>(a, phase);
      case 1024: return pencil_fold_phase_n<T, 1024>(a, phase);
      case 2048: return pencil_fold_phase_n<T, 2048>(a, phase);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.n) {
    case 64: return pencil_phase_n<T, 64>(a, phase);
    case 128: return pencil_phase_n<T, 128>(a, phase);
    case 256: return pencil_phase_n<T, 256>(a, phase);
    case 512: return pencil_phase_n<T, 512>(a, phase);
    case 1024: return pencil_phase_n<T, 1024>(a, phase);
    case 2048: return pencil_phase_n<T, 2048>(a, phase);
    default: return cudaErrorInvalidValue;
  }
}

// Tile geometry of each kernel (exported for the CPU index-model tests).
template <typename T, int NR>
void pow2_config_n(KernelGeom* g) {
  using CC = ContigCfg<T, NR>;
  using SC = StridedCfg<T, NR, 0>;
  using XC = StridedCfg<T, NR, 1>;
  g[0] = {CC::M, CC::E, CC::L, CC::THREADS, CC::SMEM};  // zfwd: M-point lines
  g[1] = {NR, SC::E, SC::L, SC::THREADS, SC::SMEM};     // ypass
  g[2] = {NR, XC::E, XC::L, XC::THREADS, XC::SMEM};     // xmid
}

template <typename T>
bool pow2_config(int n, KernelGeom* g) {
  switch (n) {
    case 2: pow2_config_n<T, 2>(g); return true;
    case 4: pow2_config_n<T, 4>(g); return true;
    case 8: pow2_config_n<T, 8>(g); return true;
    case 16: pow2_config_n<T, 16>(g); return true;
    case 32: pow2_config_n<T, 32>(g); return true;
    case 64: pow2_config_n<T, 64>(g); return true;
    case 128: pow2_config_n<T, 128>(g); return true;
    case 256: pow2_config_n<T, 256>(g); return true;
    case 512: pow2_config_n<T, 512>(g); return true;
    case 1024: pow2_config_n<T, 1024>(g); return true;
    case 2048: pow2_config_n<T, 2048>(g); return true;
    default: return false;
  }
}

template <typename T>
cudaError_t launch_pow2(const Pow2Args& a) {
  switch (a.n) {
    case 2: return launch_pow2_n<T, 2>(a);
    case 4: return launch_pow2_n<T, 4>(a);
    case 8: return launch_pow2_n<T, 8>(a);
    case 16: return launch_pow2_n<T, 16>(a);
    case 32: return launch_pow2_n<T, 32>(a);
    case 64: return launch_pow2_n<T, 64>(a);
    case 128: return launch_pow2_n<T, 128>(a);
    case 256: return launch_pow2_n<T, 256>(a);
    case 512: return launch_pow2_n<T, 512>(a);
    case 1024: return launch_pow2_n<T, 1024>(a);
    case 2048: return launch_pow2_n<T, 2048>(a);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace arena_fft
