// poisson_pow2.cuh — sm_100a kernels of the power-of-two spectral Poisson
// solve (the hot path of /root/reference/proj/src/fft_solver.cpp:51-87).
//
// Device layout of the half spectrum (internal; the boundary layout is the
// GridField one): S[(i*n + j)*ncp + k], k in [0, nc), nc = n/2 + 1, row pitch
// ncp = round_up(nc, 8) complex so every (i, j) row starts 128-byte aligned.
// This is the r2c layout FFTW produces at fft_solver.cpp:60-61 (index
// (i*n+j)*nc+k, fft_solver.cpp:74) with a padded row.
//
// Five kernels, one HBM sweep each:
//   K1 zfwd : f rows (k axis, contiguous)  -> S      real->half complex (r2c)
//   K2 yfwd : S lines along j (stride ncp) in place  c2c forward
//   K3 xmid : S lines along i (stride n*ncp) in place  c2c forward, Poisson
//             scale (fft_solver.cpp:66-79), c2c backward — one round trip
//   K4 yinv : as K2, backward
//   K5 zinv : S rows -> u rows              half complex->real (c2r)
// The r2c/c2r along the contiguous axis run an n/2-point complex FFT on the
// packed even/odd pairs (a double2 load of two reals) plus an O(n) split.
#pragma once

#include "async_copy.cuh"
#include "fft_engine.cuh"
#include "launchers.h"

namespace arena_fft {

__host__ __device__ constexpr int imin(int a, int b) { return a < b ? a : b; }
__host__ __device__ constexpr int imax(int a, int b) { return a > b ? a : b; }
__host__ __device__ constexpr int pow2_floor(int x) { return x <= 1 ? 1 : 2 * pow2_floor(x / 2); }

// Row pitch (complex elements) of the half spectrum for an n-point grid; the
// plan allocates with the same formula (plan.cu).
// spec_pitch(n): launchers.h (shared with the plan's allocation)

// Tuning knobs (compile-time; variants are built side by side for A/B runs).
#ifndef ARENA_STRIDED_MINB
#define ARENA_STRIDED_MINB 2  // min CTAs/SM hint for the strided (y, x) kernels
#endif
#ifndef ARENA_CONTIG_MINB
#define ARENA_CONTIG_MINB 8  // min CTAs/SM hint for the contiguous (z) kernels
#endif
#ifndef ARENA_STRIDED_E
#define ARENA_STRIDED_E 16  // points per thread, y / x kernels
#endif
#ifndef ARENA_CONTIG_LARGE_N
#define ARENA_CONTIG_LARGE_N 2048
#endif
#ifndef ARENA_CONTIG_LARGE_E
#define ARENA_CONTIG_LARGE_E 32  // points per thread of the z kernels for n >= ARENA_CONTIG_LARGE_N: 64-thread
                                 // CTAs, 4 per SM, 255 registers (B200 2048^3 plain path: z 27.5 -> 24.7 ms;
                                 // 16 points at 128 registers was the earlier choice)
#endif
#ifndef ARENA_CONTIG_SMALL_N
#define ARENA_CONTIG_SMALL_N 512  // B200: 512^3 z passes 0.50 -> 0.39 ms, 256^3 0.10 -> 0.07 ms
#endif
#ifndef ARENA_CONTIG_E
#define ARENA_CONTIG_E 32  // points per thread, z kernels
#endif
#ifndef ARENA_CONTIG_ROWS
#define ARENA_CONTIG_ROWS 2  // rows per z CTA: with E = 32 and n = 1024 one warp per CTA, so the
                             // exchanges' barrier spans a single warp (B200 A/B: 3.2 ms vs 6.6 ms
                             // for 8 rows x 16 points per thread)
#endif
#ifndef ARENA_Y_SMEM
#define ARENA_Y_SMEM (64 * 1024)  // shared-memory budget per y tile (sets its width L)
#endif
#ifndef ARENA_X_SMEM
#define ARENA_X_SMEM (64 * 1024)  // shared-memory budget per x tile
#endif
#ifndef ARENA_Z_PF
#define ARENA_Z_PF 1  // z passes: each CTA prefetches into L2 (one bulk request) the rows of the
                      // CTA this many waves of resident CTAs ahead, so that CTA's loads hit L2
                      // (B200 A/B, 1024^3 fp64: K1 3.40 -> 3.05 ms; 0: off)
#endif
#ifndef ARENA_SMS
#define ARENA_SMS 148  // B200 SM count (sets the prefetch distance of the z passes)
#endif


// ------------------------------------------------------------ configuration
// E: points per thread; L: lines per CTA.  Shared memory per CTA is
// N*L*sizeof(V) (<= 64 KB so two or more CTAs fit per SM).
template <typename T, int N, int PASS = 0>
struct StridedCfg {  // y (PASS 0) / x (PASS 1) passes: lines along a strided axis, L adjacent k
  static constexpr int E = imin(ARENA_STRIDED_E, N);
  static constexpr int VB = 2 * sizeof(T);
  static constexpr int BUDGET = PASS == 0 ? ARENA_Y_SMEM : ARENA_X_SMEM;
  static constexpr int L = pow2_floor(imax(1, imin(8, BUDGET / (N * VB))));
  static constexpr int P = N / E;
  static constexpr int THREADS = L * P;
  static constexpr int SMEM_X = N * L * VB;                   // exchange buffer bytes
  static constexpr int SMEM = SMEM_X;
};

template <typename T, int NR>
struct ContigCfg {  // z passes: rows of NR reals = M = NR/2 complex
  static constexpr int M = NR / 2;
  // Short rows (n <= ARENA_CONTIG_SMALL_N): 16 points per thread and twice the
  // resident warps (B200, 256^3: z passes 0.10 -> 0.07 ms; at n = 1024 E = 16
  // with 16 CTAs/SM spills).
  static constexpr bool SMALL = NR <= ARENA_CONTIG_SMALL_N;
  // n >= ARENA_CONTIG_LARGE_N (2048: M = 1024): half the CTAs per SM, so E = 32
  // (ARENA_CONTIG_LARGE_E) has 255 registers and does not spill.
  static constexpr bool LARGE = NR >= ARENA_CONTIG_LARGE_N;
  static constexpr int E = imin(SMALL ? 16 : LARGE ? ARENA_CONTIG_LARGE_E : ARENA_CONTIG_E, M);
  static constexpr int MINB = SMALL ? 2 * ARENA_CONTIG_MINB : (LARGE ? ARENA_CONTIG_MINB / 2 : ARENA_CONTIG_MINB);
  static constexpr int P = M / E;
  static constexpr int VB = 2 * sizeof(T);
  // rows per CTA (a power of two, so it divides the n^2 rows): aim for 256
  // threads and at least 8 rows, at most ~96 KB of shared memory.
  static constexpr int L0 = imax(ARENA_CONTIG_ROWS, 32 / P);  // at least one full warp
  static constexpr int L1 = imin(L0, imax(1, (96 * 1024) / ((M + 1) * VB)));
  static constexpr int L = pow2_floor(imin(L1, NR * NR));
  static constexpr int THREADS = L * P;
  static constexpr int SMEM_X = (M * L + L) * VB;
  static constexpr int SMEM = SMEM_X;
  static constexpr int PF = ARENA_Z_PF * ARENA_SMS * MINB;  // L2 prefetch distance (CTAs)
};

__device__ __forceinline__ int signed_freq(int k, int n) { return k <= n / 2 ? k : k - n; }  // fft_solver.hpp:19

// Half-spectrum layout, shared by the single-GPU and the slab (multi-GPU)
// paths.  A workspace holds P chunks of ni x nj rows of ncp complex; inside a
// chunk rows are blocked by JB = min(ARENA_JBLOCK, nj) in j:
//   row(c, il, jl) = c*ni*nj + ((jl / JB)*ni + il)*JB + jl % JB.
// Single GPU: P = 1, ni = nj = n, so row(i, j) = ((j/JB)*n + i)*JB + j%JB — a y
// tile (fixed i) reads n/JB contiguous JB-row chunks and an x tile (fixed j)
// reads rows JB*ncp apart; with plain row-major rows the x pass touched n
// different 2 MB pages per tile and its access pattern alone capped at 3.1 TB/s
// on B200 (tools/pattern_bw.cu; 6.2-6.4 TB/s with JB = 8).  Larger blocks trade
// a little x for more y (JB = 64: y 3.41 -> 3.19 ms, x 4.13 -> 4.23 ms at 1024^3).
// Slab over P ranks (ni = nj = n/P): layout B (K1/K2/K4/K5 on a rank's i-slab)
// puts j in chunk c = j / nj, so the block for peer c is contiguous; layout C
// (K3 on a j-slab) puts i in chunk c = i / ni — exactly what arrives from rank c.
struct Layout {
  int ni, nj;       // rows per chunk: il in [0, ni), jl in [0, nj)
  int nis, njs;     // log2 ni, log2 nj
  int jbs;          // log2 JB
};

__host__ __device__ __forceinline__ size_t lrow(const Layout& g, int c, int il, int jl) {
  return (size_t(c) << (g.nis + g.njs)) + ((size_t(jl >> g.jbs) * g.ni + il) << g.jbs) + (jl & ((1 << g.jbs) - 1));
}
// Layout B: (local i, global j).  Layout C: (global i, local j).
__host__ __device__ __forceinline__ size_t rowB(const Layout& g, int il, int j) {
  return lrow(g, j >> g.njs, il, j & (g.nj - 1));
}
__host__ __device__ __forceinline__ size_t rowC(const Layout& g, int i, int jl) {
  return lrow(g, i >> g.nis, i & (g.ni - 1), jl);
}

inline int ilog2_host(int x) {
  int r = 0;
  while ((1 << r) < x) ++r;
  return r;
}
inline Layout make_layout(int ni, int nj) {
  Layout g;
  g.ni = ni;
  g.nj = nj;
  g.nis = ilog2_host(ni);
  g.njs = ilog2_host(nj);
  g.jbs = ilog2_host(nj < ARENA_JBLOCK ? nj : ARENA_JBLOCK);
  return g;
}

// The single-GPU geometry (one chunk of n x n rows, full k range, in
// place) as compile-time constants, so every row / address computation folds
// into constant strides (kernels with FIXED = true ignore their runtime geometry).
__host__ __device__ constexpr int ilog2_c(int x) { return x <= 1 ? 0 : 1 + ilog2_c(x >> 1); }
template <int N>
__host__ __device__ constexpr Layout fixed_layout() {
  return Layout{N, N, ilog2_c(N), ilog2_c(N), ilog2_c(N < ARENA_JBLOCK ? N : ARENA_JBLOCK)};
}

// The Poisson symbol of fft_solver.cpp:66-79, k2 == 0 ? 0 : scale / (four_pi2 * k2),
// with the division done as a hardware reciprocal estimate refined by Newton
// steps (no slow path / divergence); within 2 ulp of the IEEE quotient.
#ifndef ARENA_RCP_NEWTON
#define ARENA_RCP_NEWTON 2
#endif
__device__ __forceinline__ double poisson_symbol(double k2, double scale, double four_pi2) {
  const double d = four_pi2 * k2;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  // MUFU.RCP64H is good to ~2^-20; each Newton step squares the relative error.
#pragma unroll
  for (int it = 0; it < ARENA_RCP_NEWTON; ++it) {
    const double e = fma(-d, r, 1.0);
    r = fma(r, e, r);
  }
  return k2 == 0.0 ? 0.0 : scale * r;
}
// Lean fp64 symbol of the x passes: m = 1 / (k2 * (four_pi2 / scale)), the scale folded
// into the divisor (exact for the power-of-two path, scale = 2^-3 log2 n), the MUFU
// estimate refined by one cubic step r (1 + e + e^2) (~2^-66 from its ~2^-22), and no
// k2 == 0 select — the caller zeroes the one k = 0 mode (ARENA_LEAN_SYMBOL).
#ifndef ARENA_LEAN_SYMBOL
#define ARENA_LEAN_SYMBOL 1
#endif
__device__ __forceinline__ double poisson_symbol_lean(double k2, double cinv) {
  const double d = k2 * cinv;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  const double e = fma(-d, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ float poisson_symbol(float k2, float scale, float four_pi2) {
  const float d = four_pi2 * k2;
  float r;
  // MUFU.RCP (<= 1 ulp): the IEEE __frcp_rn is a subroutine call per element, and the
  // fp32 tolerance (1e-5) is far above an ulp
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(d));
  return k2 == 0.0f ? 0.0f : scale * r;
}

template <typename V>
__device__ __forceinline__ V* smem_base() {
  extern __shared__ __align__(16) unsigned char arena_smem_raw[];
  return reinterpret_cast<V*>(arena_smem_raw);
}


// W_n^k, k = t + P e, for the r2c / c2r split of an n = 2 P E point row: the thread's
// W_n^t times the compile-time root W_{2E}^e (e is constant once the caller's loop is
// unrolled) — one complex product instead of a table load per element, off the
// L1TEX pipe the z kernels are bound by (ncu: l1tex 88%).  ARENA_Z_TWREC = 0: loads.
#ifndef ARENA_Z_PAIRS
#define ARENA_Z_PAIRS 1  // r2c split: both outputs of a pair (k, M - k) from one thread
#endif
#ifndef ARENA_Z_TWREC
#define ARENA_Z_TWREC 1
#endif
// W_64^m = exp(-2 pi i m / 64) in the constant cache: split_twiddle's index is warp-uniform
// (the unrolled loop's e), so each read is one broadcast LDC, not an L1TEX request.
#define ARENA_W64(m) {cos64(m), -sin64(m)}
static __constant__ double2 kW64d[64] = {
    ARENA_W64(0), ARENA_W64(1), ARENA_W64(2), ARENA_W64(3), ARENA_W64(4), ARENA_W64(5), ARENA_W64(6), ARENA_W64(7),
    ARENA_W64(8), ARENA_W64(9), ARENA_W64(10), ARENA_W64(11), ARENA_W64(12), ARENA_W64(13), ARENA_W64(14), ARENA_W64(15),
    ARENA_W64(16), ARENA_W64(17), ARENA_W64(18), ARENA_W64(19), ARENA_W64(20), ARENA_W64(21), ARENA_W64(22), ARENA_W64(23),
    ARENA_W64(24), ARENA_W64(25), ARENA_W64(26), ARENA_W64(27), ARENA_W64(28), ARENA_W64(29), ARENA_W64(30), ARENA_W64(31),
    ARENA_W64(32), ARENA_W64(33), ARENA_W64(34), ARENA_W64(35), ARENA_W64(36), ARENA_W64(37), ARENA_W64(38), ARENA_W64(39),
    ARENA_W64(40), ARENA_W64(41), ARENA_W64(42), ARENA_W64(43), ARENA_W64(44), ARENA_W64(45), ARENA_W64(46), ARENA_W64(47),
    ARENA_W64(48), ARENA_W64(49), ARENA_W64(50), ARENA_W64(51), ARENA_W64(52), ARENA_W64(53), ARENA_W64(54), ARENA_W64(55),
    ARENA_W64(56), ARENA_W64(57), ARENA_W64(58), ARENA_W64(59), ARENA_W64(60), ARENA_W64(61), ARENA_W64(62), ARENA_W64(63)};
static __constant__ float2 kW64f[64] = {
    ARENA_W64(0), ARENA_W64(1), ARENA_W64(2), ARENA_W64(3), ARENA_W64(4), ARENA_W64(5), ARENA_W64(6), ARENA_W64(7),
    ARENA_W64(8), ARENA_W64(9), ARENA_W64(10), ARENA_W64(11), ARENA_W64(12), ARENA_W64(13), ARENA_W64(14), ARENA_W64(15),
    ARENA_W64(16), ARENA_W64(17), ARENA_W64(18), ARENA_W64(19), ARENA_W64(20), ARENA_W64(21), ARENA_W64(22), ARENA_W64(23),
    ARENA_W64(24), ARENA_W64(25), ARENA_W64(26), ARENA_W64(27), ARENA_W64(28), ARENA_W64(29), ARENA_W64(30), ARENA_W64(31),
    ARENA_W64(32), ARENA_W64(33), ARENA_W64(34), ARENA_W64(35), ARENA_W64(36), ARENA_W64(37), ARENA_W64(38), ARENA_W64(39),
    ARENA_W64(40), ARENA_W64(41), ARENA_W64(42), ARENA_W64(43), ARENA_W64(44), ARENA_W64(45), ARENA_W64(46), ARENA_W64(47),
    ARENA_W64(48), ARENA_W64(49), ARENA_W64(50), ARENA_W64(51), ARENA_W64(52), ARENA_W64(53), ARENA_W64(54), ARENA_W64(55),
    ARENA_W64(56), ARENA_W64(57), ARENA_W64(58), ARENA_W64(59), ARENA_W64(60), ARENA_W64(61), ARENA_W64(62), ARENA_W64(63)};
#undef ARENA_W64
__device__ __forceinline__ double2 w64(int m, double) { return kW64d[m]; }
__device__ __forceinline__ float2 w64(int m, float) { return kW64f[m]; }

template <int E, typename V>
__device__ __forceinline__ V split_twiddle(const V* __restrict__ tw, V wt, int k, int e) {
  if constexpr (ARENA_Z_TWREC && E <= 32) {
    using T = decltype(wt.x);
    const V r = w64((e * (32 / E)) & 63, T(0));  // W_{2E}^e = W_64^{e 32 / E}
    return cmul(wt, r);
  } else {
    return tw_load(tw, k);
  }
}

// ------------------------------------------------------------------- K1 zfwd
// Rows of NR reals: z[m] = f[2m] + i f[2m+1] (one vector load), M-point FFT,
// then X[k] = 1/2 (A + B) - 1/2 i W_n^k (A - B), A = Z[k], B = conj(Z[M-k]),
// for k in [0, M]; X[M] = Re Z0 - Im Z0.
// One group of L*P threads (index gt) transforms slab rows row0 .. row0+L-1
// (row = il*n + j) using `sm` ((M+1)*L elements); SYNC is the group barrier.
template <typename T, int NR, int E, int L, int SYNC>
__device__ __forceinline__ void zfwd_rows(const T* __restrict__ f, vec2_t<T>* __restrict__ S,
                                          const vec2_t<T>* __restrict__ tw, const vec2_t<T>* __restrict__ stw,
                                          const Layout& g, size_t row0, vec2_t<T>* sm, int gt) {
  using V = vec2_t<T>;
  constexpr int M = NR / 2, P = M / E;
  constexpr int ncp = spec_pitch(NR);
  constexpr int SW = engine_swizzle<M, E>();
  const int l = gt % L, t = gt / L;
  const size_t row = row0 + l;
  const V* src = reinterpret_cast<const V*>(f + row * NR);
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  line_fft<M, E, L, -1, SYNC>(v, sm, stw, t, l);
  constexpr bool PAIRS = ARENA_Z_PAIRS && E >= 2 && (E % 2) == 0 && ARENA_Z_TWREC && E <= 32;
  // staging for the mirror reads: the paired split only reads positions > M/2 (and Z[0] from its owner)
#pragma unroll
  for (int e = PAIRS ? E / 2 : 0; e < E; ++e) sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  xbarrier<SYNC>();
  V* dst = S + rowB(g, int(row / NR), int(row % NR)) * ncp;
  const V wt = tw_load(tw, t);  // W_n^t (split_twiddle)
  if constexpr (PAIRS) {
    // Both members of a pair from one thread: with A = Z[k], B = conj(Z[M-k]), S = (A + B)/2 and
    // U = (i/2) W_n^k (A - B),  X[k] = S - U  and  X[M-k] = conj(S + U)  (W_n^{M-k} = -conj W_n^k),
    // so the difference and its product with the twiddle are formed once per pair: 8 fp64
    // operations per output instead of 16, and half the mirror reads.  k = t + P e, e < E/2,
    // covers [0, M/2); k = 0 pairs with the Nyquist output X[M]; X[M/2] = conj(Z[M/2]).
    const V wh{T(-0.5) * wt.y, T(0.5) * wt.x};  // (i/2) W_n^t
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int k = t + P * e;
      const V A = v[e];
      const V Bc = k == 0 ? A : sm[smem_idx<L, SW, V>(M - k, l)];
      const V B{Bc.x, -Bc.y};
      const V Wh = split_twiddle<E>(tw, wh, k, e);  // (i/2) W_n^k
      const V U = cmul(Wh, csub(A, B));
      const V Sm = cadd(A, B);
      dst[k] = V{fma(T(0.5), Sm.x, -U.x), fma(T(0.5), Sm.y, -U.y)};
      V Xm{fma(T(0.5), Sm.x, U.x), -fma(T(0.5), Sm.y, U.y)};
      if (k == 0) Xm.y = T(0);  // X[M] = Re Z0 - Im Z0, real
      dst[M - k] = Xm;
    }
    if (t == 0) dst[M / 2] = V{v[E / 2].x, -v[E / 2].y};
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = t + P * e;
      const V A = v[e];
      const V Bc = sm[smem_idx<L, SW, V>((M - k) & (M - 1), l)];
      const V B{Bc.x, -Bc.y};
      const V W = split_twiddle<E>(tw, wt, k, e);  // W_n^k
      const V WD = cmul(W, csub(A, B));
      dst[k] = V{T(0.5) * (A.x + B.x + WD.y), T(0.5) * (A.y + B.y - WD.x)};
      if (k == 0) dst[M] = V{A.x - A.y, T(0)};
    }
  }
}

template <typename T, int NR, bool FIXED = false>
__global__ void __launch_bounds__(ContigCfg<T, NR>::THREADS, ContigCfg<T, NR>::MINB)
    k_zfwd(const T* __restrict__ f, vec2_t<T>* __restrict__ S, const vec2_t<T>* __restrict__ tw,
           const vec2_t<T>* __restrict__ stw, Layout g_) {
  using C = ContigCfg<T, NR>;
  const Layout g = FIXED ? fixed_layout<NR>() : g_;
  if constexpr (ARENA_Z_PF > 0) {
    const unsigned b = blockIdx.x + C::PF;
    if (threadIdx.x == 0 && b < gridDim.x) bulk_prefetch_l2(f + size_t(b) * C::L * NR, C::L * NR * sizeof(T));
  }
  zfwd_rows<T, NR, C::E, C::L, kSyncCta>(f, S, tw, stw, g, size_t(blockIdx.x) * C::L, smem_base<vec2_t<T>>(),
                                         threadIdx.x);
}

// Evict-without-writeback (PTX discard.global.L2) of one 128-byte line.
__device__ __forceinline__ void l2_discard(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

// ------------------------------------------------------------------- K5 zinv
// Inverse of K1 with FFTW c2r semantics (imaginary parts of X[0] and X[M]
// ignored): Z[k] = (A + B) + i (A - B) conj(W_n^k), A = X[k], B = conj(X[M-k]),
// M-point backward FFT, u[2m] = Re z[m], u[2m+1] = Im z[m].  DISCARD drops the
// consumed half-spectrum rows from L2 without writing them back (fused path:
// they were produced in L2 by the y pass and are dead after this read).
template <typename T, int NR, int E, int L, int SYNC, bool DISCARD>
__device__ __forceinline__ void zinv_rows(const vec2_t<T>* __restrict__ S, T* __restrict__ u,
                                          const vec2_t<T>* __restrict__ tw, const vec2_t<T>* __restrict__ stw,
                                          const Layout& g, size_t row0, vec2_t<T>* sm, int gt) {
  using V = vec2_t<T>;
  constexpr int M = NR / 2, P = M / E;
  constexpr int ncp = spec_pitch(NR);
  constexpr int SW = engine_swizzle<M, E>();
  V* xm = sm + M * L;  // X[M] per line
  const int l = gt % L, t = gt / L;
  const size_t row = row0 + l;
  const V* src = S + rowB(g, int(row / NR), int(row % NR)) * ncp;
  V v[E];
  auto ld = [&](int k) { return DISCARD ? __ldcg(src + k) : __ldcs(src + k); };
  if constexpr (ARENA_Z_PAIRS && E >= 2 && (E % 2) == 0 && ARENA_Z_TWREC && E <= 32) {
    // Both members of a pair from one thread (the mirror of zfwd_rows' split): with A = X[k],
    // B = conj(X[M-k]), Ep = A + B and Op = i conj(W_n^k) (A - B),  Z[k] = Ep + Op  and
    // Z[M-k] = conj(Ep - Op).  The thread loads X[k] and X[M-k] itself (k = t + P e, e < E/2;
    // k = 0 pairs X[0] with X[M], imaginary parts ignored as FFTW's c2r does), keeps Z[k]
    // and hands Z[M-k] to its owner through shared memory: half the staging traffic and
    // 8 instead of 14 fp64 operations per element.  Z[M/2] = 2 conj(X[M/2]).
    const V wt = tw_load(tw, t);
    const V wi{wt.y, wt.x};  // i conj(W_n^t)
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int k = t + P * e;
      V A = ld(k);
      V C = ld(M - k);
      if (k == 0) {
        A.y = T(0);
        C.y = T(0);
      }
      const V B{C.x, -C.y};
      const V Wi = cmulc(wi, w64((e * (32 / E)) & 63, T(0)));  // i conj(W_n^k), W_n^{P e} = W_64^{e 32 / E}
      const V Ep = cadd(A, B);
      const V Op = cmul(csub(A, B), Wi);
      v[e] = cadd(Ep, Op);
      if (k != 0) sm[smem_idx<L, SW, V>(M - k, l)] = V{Ep.x - Op.x, Op.y - Ep.y};
    }
    if (t == 0) {
      const V h = ld(M / 2);
      sm[smem_idx<L, SW, V>(M / 2, l)] = V{T(2) * h.x, T(-2) * h.y};
    }
    xbarrier<SYNC>();
    if constexpr (DISCARD) {
      constexpr int LINES = ncp * int(sizeof(V)) / 128;
      for (int q = t; q < LINES; q += P) l2_discard(reinterpret_cast<const char*>(src) + size_t(q) * 128);
    }
#pragma unroll
    for (int e = E / 2; e < E; ++e) v[e] = sm[smem_idx<L, SW, V>(t + P * e, l)];
    xbarrier<SYNC>();
    line_fft<M, E, L, +1, SYNC>(v, sm, stw, t, l);
    V* dstp = reinterpret_cast<V*>(u + row * NR);
#pragma unroll
    for (int e = 0; e < E; ++e) st_out(dstp + t + P * e, v[e]);
  } else {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    v[e] = ld(t + P * e);
    sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  }
  if (t == 0) xm[l] = ld(M);
  xbarrier<SYNC>();
  if constexpr (DISCARD) {
    constexpr int LINES = ncp * int(sizeof(V)) / 128;
    for (int q = t; q < LINES; q += P) l2_discard(reinterpret_cast<const char*>(src) + size_t(q) * 128);
  }
  const V wt = tw_load(tw, t);  // W_n^t (split_twiddle)
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    V A = v[e];
    V Bs = (k == 0) ? xm[l] : sm[smem_idx<L, SW, V>(M - k, l)];
    if (k == 0) {
      A.y = T(0);
      Bs.y = T(0);
    }
    const V B{Bs.x, -Bs.y};
    const V W = split_twiddle<E>(tw, wt, k, e);
    const V Ep = cadd(A, B);
    const V Op = cmulc(csub(A, B), W);
    v[e] = V{Ep.x - Op.y, Ep.y + Op.x};
  }
  xbarrier<SYNC>();
  line_fft<M, E, L, +1, SYNC>(v, sm, stw, t, l);
  V* dst = reinterpret_cast<V*>(u + row * NR);
#pragma unroll
  for (int e = 0; e < E; ++e) st_out(dst + t + P * e, v[e]);
  }
}

template <typename T, int NR, bool FIXED = false>
__global__ void __launch_bounds__(ContigCfg<T, NR>::THREADS, ContigCfg<T, NR>::MINB)
    k_zinv(const vec2_t<T>* __restrict__ S, T* __restrict__ u, const vec2_t<T>* __restrict__ tw,
           const vec2_t<T>* __restrict__ stw, Layout g_) {
  using C = ContigCfg<T, NR>;
  const Layout g = FIXED ? fixed_layout<NR>() : g_;
  if constexpr (ARENA_Z_PF > 0) {
    const unsigned b = blockIdx.x + C::PF;
    if (threadIdx.x < C::L && b < gridDim.x) {
      const size_t row = size_t(b) * C::L + threadIdx.x;
      constexpr int ncp = spec_pitch(NR);
      bulk_prefetch_l2(S + rowB(g, int(row / NR), int(row % NR)) * ncp, ncp * sizeof(vec2_t<T>));
    }
  }
  zinv_rows<T, NR, C::E, C::L, kSyncCta, false>(S, u, tw, stw, g, size_t(blockIdx.x) * C::L, smem_base<vec2_t<T>>(),
                                                threadIdx.x);
}

// --------------------------------------------------------------- K2/K4 ypass
template <typename T, int N, int S>
__global__ void __launch_bounds__(StridedCfg<T, N, 0>::THREADS, ARENA_STRIDED_MINB)
    k_ypass(vec2_t<T>* __restrict__ spec, const vec2_t<T>* __restrict__ stw, Layout g) {
  using V = vec2_t<T>;
  using C = StridedCfg<T, N, 0>;
  constexpr int E = C::E, P = C::P, L = C::L;
  constexpr int ncp = spec_pitch(N), nc = N / 2 + 1;
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int k = blockIdx.x * L + l;
  const bool valid = k < nc;
  V* base = spec + k;
  const int i = blockIdx.y;
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = valid ? __ldcs(base + rowB(g, i, t + P * e) * ncp) : V{T(0), T(0)};
  line_fft<N, E, L, S>(v, sm, stw, t, l);
  if (valid) {
#pragma unroll
    for (int e = 0; e < E; ++e) st_out(base + rowB(g, i, t + P * e) * ncp, v[e]);
  }
}

// -------------------------------------------------------------- K3 xmid
// Forward FFT along i, multiply by the Poisson symbol of fft_solver.cpp:66-79
// (same expression: k2 == 0 ? 0 : scale / (four_pi2 * k2), k2 summed in T from
// exact integer squares), backward FFT along i.  The data never leaves
// registers between the two transforms.
template <typename T, int N>
__global__ void __launch_bounds__(StridedCfg<T, N, 1>::THREADS, ARENA_STRIDED_MINB)
    k_xmid(vec2_t<T>* __restrict__ spec, const vec2_t<T>* __restrict__ stw, T scale, T four_pi2, Layout g) {
  using V = vec2_t<T>;
  using C = StridedCfg<T, N, 1>;
  constexpr int E = C::E, P = C::P, L = C::L;
  constexpr int ncp = spec_pitch(N), nc = N / 2 + 1;
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int k = blockIdx.x * L + l;
  const int j = blockIdx.y;
  const bool valid = k < nc;
  const size_t istride = (rowC(g, 1, j) - rowC(g, 0, j)) * ncp;  // JB * ncp (single GPU)
  V* base = spec + rowC(g, 0, j) * ncp + k;
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = valid ? __ldcs(base + size_t(t + P * e) * istride) : V{T(0), T(0)};
  line_fft<N, E, L, -1>(v, sm, stw, t, l);
  const T kj = T(signed_freq(j, N)), kk = T(k);
  const T c = kj * kj + kk * kk;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const T ki = T(signed_freq(t + P * e, N));
    const T k2 = ki * ki + c;
    const T m = poisson_symbol(k2, scale, four_pi2);
    v[e].x *= m;
    v[e].y *= m;
  }
  line_fft<N, E, L, +1>(v, sm, stw, t, l);
  if (valid) {
#pragma unroll
    for (int e = 0; e < E; ++e) st_out(base + size_t(t + P * e) * istride, v[e]);
  }
}

}  // namespace arena_fft

// ===================================================================== TMA path
// Persistent, software-pipelined versions of the strided passes: one CTA per
// SM walks the tiles; while it transforms tile g (registers + the tile's own
// shared buffer as exchange scratch), the tensor-memory accelerator streams
// tile g + gridDim.x into the other buffer.  Loads therefore never stall the
// FFT and need no per-thread address arithmetic; stores go straight from
// registers.
#include "async_copy.cuh"

namespace arena_fft {

// B200 A/B at 1024^3 fp64 (tools/ab.sh): one tile buffer per CTA with two
// co-resident CTAs per SM (x pass 5.4 ms) beat a double-buffered single CTA
// (6.3 ms); three buffers were slower still (the carveout starves L1, which
// holds the twiddle tables).
#ifndef ARENA_TMA_E
#define ARENA_TMA_E 32  // points per thread in the TMA strided kernels
#endif
#ifndef ARENA_TMA_MINB
#define ARENA_TMA_MINB 2  // co-resident CTAs per SM
#endif
#ifndef ARENA_TMA_NBUF
#define ARENA_TMA_NBUF 1  // tile buffers per CTA (prefetch distance NBUF-1)
#endif
#ifndef ARENA_TMA_TWSMEM_X
#define ARENA_TMA_TWSMEM_X 1  // x pass: stage-twiddle table staged in shared memory once per CTA
#endif                        // (B200 A/B: x 5.76 -> 5.04 ms)
#ifndef ARENA_TMA_TWSMEM_Y
#define ARENA_TMA_TWSMEM_Y 0  // same for the y passes
#endif
#ifndef ARENA_TMA_L2PF
#define ARENA_TMA_L2PF 0  // also prefetch the tile this many iterations ahead into L2 (0: off; B200
                          // 1024^3: x 4.3 -> 6.1 ms at 1, and the same with per-thread
                          // prefetch.global.L2 of the next tile's rows — the strided passes lose
                          // to any early L2 traffic, unlike the z passes, ARENA_Z_PF)
#endif

// y passes (B200 A/B, 1024^3): 8-line tiles (128-byte TMA rows), one CTA per SM,
// next tile requested right after the last exchange: 3.71 ms vs 4.15 ms for the
// x-pass configuration (4-line tiles, two CTAs per SM).
#ifndef ARENA_TMA_Y_TILE
#define ARENA_TMA_Y_TILE (128 * 1024)  // y-pass tile budget (bytes): sets the y tile width L
#endif
#ifndef ARENA_TMA_MINB_Y
#define ARENA_TMA_MINB_Y 1
#endif
#ifndef ARENA_TMA_E_Y
#define ARENA_TMA_E_Y 16  // y passes: 16 points/thread, 512 threads per 8-line tile (3.51 vs 3.71 ms)
#endif
#ifndef ARENA_TMA_X_TILE
#define ARENA_TMA_X_TILE (64 * 1024)  // x-pass tile budget (bytes)
#endif
#ifndef ARENA_TMA_E_XS
#define ARENA_TMA_E_XS 32  // fp64 x pass on lines of N <= 512 points (quadrant / split lines)
#endif
#ifndef ARENA_TMA_NBUF_Y
#define ARENA_TMA_NBUF_Y ARENA_TMA_NBUF
#endif
#ifndef ARENA_TMA_E2S_X
#define ARENA_TMA_E2S_X 1  // x pass: last exchange shifted into spare shared memory, first half of the next
#endif                     // tile requested before it
#ifndef ARENA_TMA_E2S_Y
#define ARENA_TMA_E2S_Y 0  // y passes: same (B200 1024^3 fp64: y 3.06 -> 3.21 ms — they run at ~90% of their access
                           // pattern's bandwidth cap and wait on DRAM, not on a late request)
#endif
#ifndef ARENA_TMA_EARLY_Y
#define ARENA_TMA_EARLY_Y 1  // y passes: request the next tile right after the last exchange
#endif

// fp32 variants (a complex float is 8 bytes, so 128-byte TMA rows need 16 lines).
#ifndef ARENA_TMA_LROW
#define ARENA_TMA_LROW 128  // bytes of a tile row (L adjacent k) at most
#endif
#ifndef ARENA_TMA_Y_TINY
#define ARENA_TMA_Y_TINY 0  // tile bytes up to which the y passes run four CTAs per SM (0: never)
#endif
#ifndef ARENA_TMA_Y_SMALL
#define ARENA_TMA_Y_SMALL 65536  // tile bytes up to which the y passes run two CTAs per SM (512^3: y 0.53 -> 0.46 ms)
#endif
#ifndef ARENA_TMA_E32
#define ARENA_TMA_E32 32
#endif
#ifndef ARENA_TMA_E_Y32
#define ARENA_TMA_E_Y32 16  // fp32 y: 16-line tiles (128-byte rows), 1024 threads (B200: 1.73 vs 2.02 ms at E = 32)
#endif
#ifndef ARENA_TMA_X_TILE32
#define ARENA_TMA_X_TILE32 ARENA_TMA_X_TILE
#endif
#ifndef ARENA_TMA_Y_TILE32
#define ARENA_TMA_Y_TILE32 ARENA_TMA_Y_TILE
#endif
#ifndef ARENA_TMA_MINB32
#define ARENA_TMA_MINB32 ARENA_TMA_MINB
#endif
#ifndef ARENA_TMA_MINB_Y32
#define ARENA_TMA_MINB_Y32 ARENA_TMA_MINB_Y
#endif

// YP: configuration of the y passes (PASS 0/1) vs the x pass.  XW: the x pass
// takes the wide (two-budget, one CTA per SM) tile regardless of its row width.
#ifndef ARENA_QUAD_XW
#define ARENA_QUAD_XW 1  // quadrant x pass: 128-byte rows (B200 2048^3: 64-byte rows re-read 1.7x in L2)
#endif
#ifndef ARENA_X_WIDE64
#define ARENA_X_WIDE64 1  // fp64 x pass: 128-byte rows too (1024^3: one 8-warp CTA per SM, 4.35 -> 4.30 ms;
                          // fp32 measured slower that way, 2.31 -> 2.50 ms)
#endif
#ifndef ARENA_X_WIDE32
#define ARENA_X_WIDE32 0  // fp32 x pass: 16-line tiles (128-byte rows), one 512-thread CTA per SM
#endif
template <typename T, int N, bool YP = false, bool XW = false>
struct TmaCfg;
// XW of the x pass (TmaCfg<T, N, false, x_wide<T, QUAD>()>)
template <typename T, bool QUAD>
constexpr bool x_wide() {
  return QUAD ? bool(ARENA_QUAD_XW) : (sizeof(T) == 8 ? bool(ARENA_X_WIDE64) : bool(ARENA_X_WIDE32));
}
template <typename T, int N, bool YP, bool XW>
struct TmaCfg {
  static constexpr bool F64 = sizeof(T) == 8;
  static constexpr int VB = 2 * sizeof(T);
  static constexpr int E = imin(YP ? (F64 ? ARENA_TMA_E_Y : ARENA_TMA_E_Y32)
                                   : (F64 ? (N <= 512 ? ARENA_TMA_E_XS : ARENA_TMA_E) : ARENA_TMA_E32),
                                N);
  static constexpr int P = N / E;
  static constexpr int BUDGET0 = YP ? (F64 ? ARENA_TMA_Y_TILE : ARENA_TMA_Y_TILE32)
                                    : (F64 ? ARENA_TMA_X_TILE : ARENA_TMA_X_TILE32);
  // Long x lines (n >= 2048 fp64): a 64 KB tile would leave rows of 32 bytes, so the x
  // pass takes a tile twice as wide (one CTA per SM) — B200 2048^3: x 98.8 -> 51.1 ms.
  static constexpr int ROWB = imax(1, BUDGET0 / (N * VB)) * VB;  // tile row bytes at the base budget
  static constexpr bool WIDEX = !YP && ((XW && ROWB < 128) || ROWB < 64);
  static constexpr int BUDGET = WIDEX ? 2 * BUDGET0 : BUDGET0;
  static constexpr int L = pow2_floor(imax(2, imin(ARENA_TMA_LROW / VB, BUDGET / (N * VB))));
  static constexpr int MINB0 = WIDEX ? 1
                               : YP ? (F64 ? ARENA_TMA_MINB_Y : ARENA_TMA_MINB_Y32) : (F64 ? ARENA_TMA_MINB : ARENA_TMA_MINB32);
  // y passes with tiles of <= 64 KB (n <= 512): two CTAs per SM
  static constexpr int MINB = (YP && N * L * VB <= ARENA_TMA_Y_TINY)    ? imax(MINB0, 4)
                              : (YP && N * L * VB <= ARENA_TMA_Y_SMALL) ? imax(MINB0, 2)
                                                                        : MINB0;
  static constexpr int THREADS = L * P;
  static constexpr int NC = N / 2 + 1;
  static constexpr int KT = (NC + L - 1) / L;  // k tiles per line set
  static constexpr int TILE = N * L;          // elements per tile
  static constexpr int NB0 = YP ? ARENA_TMA_NBUF_Y : ARENA_TMA_NBUF;
  static constexpr int NBUF = (NB0 * TILE * VB <= 200 * 1024) ? NB0 : imin(2, NB0);
  static constexpr int TW = stage_tw_total(N, E);  // staged twiddle entries (x pass)
  // Shifted last exchange (E2S): half a tile of spare shared memory behind the tile buffer.
  // The pass's last exchange runs in [TILE/2, 3 TILE/2) instead of [0, TILE), so the first
  // half of the next tile is requested before it (right after the previous exchange, or
  // after the tile read when there is none) and only the second half has to wait for it:
  // the strided passes spent 9% (x) / 13% (y) of their time waiting for the tile (ncu).
  static constexpr int E2SW = YP ? ARENA_TMA_E2S_Y : ARENA_TMA_E2S_X;
  static constexpr bool E2S = E2SW != 0 && NBUF == 1 && num_stages(N, E) > 1 && N >= 4 &&
                              MINB * (TILE * VB * 3 / 2 + ((YP ? ARENA_TMA_TWSMEM_Y : ARENA_TMA_TWSMEM_X) ? TW * VB : 0) + 1024 + 64) <= 228 * 1024;
  static constexpr int SMEM = NBUF * TILE * VB + 16 * NBUF + (E2S ? TILE * VB / 2 : 0);
  static constexpr int SMEM_X = SMEM + (ARENA_TMA_TWSMEM_X ? TW * VB : 0);
  static constexpr int SMEM_Y = SMEM + (ARENA_TMA_TWSMEM_Y ? TW * VB : 0);
};

// TMA view of a workspace in Layout g: a 5-D tensor of reals
//   {2*nc (re/im of k), JB (jl % JB), ni (il), nj/JB (jl / JB), P (chunk)}.
// y tile (fixed il): box {2L, JB, 1, nj/JB, P}  -> all j in natural order.
// x tile (fixed jl): boxes {2L, 1, IB, 1, 1} over il blocks and chunks -> all i.
__host__ __device__ constexpr int tma_ib(int ni) { return ni < 256 ? ni : 256; }

// A y tile is fetched as two half boxes (so the first half can be requested ahead of the
// second, E2S): split over the chunks (dimension 4) when it spans several, else over the
// j blocks (dimension 3) when there are at least two, else one whole box (returns 0).
// nch = chunks a y tile spans (1 for the chunked single-GPU layouts).  encode_map builds
// the box by the same rule.
__host__ __device__ __forceinline__ int ytile_split(const Layout& g, int nch) {
  return nch >= 2 ? 4 : ((g.nj >> g.jbs) >= 2 ? 3 : 0);
}
// Half h (0 / 1) of y tile (k offset c0 reals, line `outer`, chunk qd) into dst_tile; with an
// unsplit box, half 1 is the whole tile and half 0 empty (half 0 may be requested while the
// upper half of the tile buffer is still exchange scratch).  The caller posts the bytes
// (ytile_half_bytes) on `bar` first.
__host__ __device__ __forceinline__ uint32_t ytile_half_bytes(const Layout& g, int nch, int h, uint32_t tile_bytes) {
  return ytile_split(g, nch) ? tile_bytes / 2 : (h ? tile_bytes : 0u);
}
template <typename V>
__device__ __forceinline__ void ytile_half_load(V* dst_tile, const CUtensorMap* tmap, uint64_t* bar, const Layout& g,
                                                int nch, int c0, int outer, int qd, int h, uint32_t tile_bytes) {
  const int sd = ytile_split(g, nch);
  if (sd == 0) {
    if (h == 1) tma_load_5d(dst_tile, tmap, bar, c0, 0, outer, 0, qd);
  } else {
    const int c3 = sd == 3 ? h * ((g.nj >> g.jbs) / 2) : 0;
    const int c4 = sd == 4 ? h * (nch / 2) : qd;
    tma_load_5d(reinterpret_cast<char*>(dst_tile) + size_t(h) * (tile_bytes / 2), tmap, bar, c0, 0, outer, c3, c4);
  }
}

// The k range a workspace holds: local k in [0, kc), row pitch kq complex,
// global k = k0 + local k.  One GPU and slab: {nc, ncp, 0}; pencil: the rank's
// k chunk.
struct KSpan {
  int kc, kq, k0;
  int no = 0;  // lines (outer index) to transform, 0 = all of the layout's (sub-range launches of the
               // slab's chunked exchange pass a shifted base and the sub-range's count)
  // Folded pencil (poisson_qpencil.cuh): N-point lines of quadrant (fci, fcj) of a 2N grid,
  // frequencies ki = 2 i'' + fci, kj = 2 (j0 + j'') + fcj (x pass symbol).
  int fm = 0, fci = 0, fcj = 0;
};

// Chunked ("split") layouts of the single-GPU path, selected by the SPL template
// argument of the strided kernels: SPL = R > 0 splits both i and j by R (R*R
// chunks of (n/R)^2 rows: the quadrant formulation R = 2, poisson_quad.cuh; the
// radix-3/5 splits, poisson_split3.cuh).
__host__ __device__ constexpr int spl_chunks(int spl) { return spl > 0 ? spl * spl : 1; }
// Compile-time geometry of a FIXED (single-GPU) strided pass on N-point lines.
template <int N, int SPL, int PASS>
__host__ __device__ constexpr Layout fixed_geom() {
  return fixed_layout<N>();
}
template <int N, int SPL, int PASS>
__host__ __device__ constexpr KSpan fixed_kspan() {
  // the n of the grid the N-point lines belong to
  constexpr int NG = SPL > 0 ? SPL * N : N;
  return KSpan{NG / 2 + 1, spec_pitch(NG), 0};
}

// PASS 0: y forward, 1: y backward (layout B, tiles over (il, k-tile)); the y
// passes may write to another buffer / layout (`out`, `gout`; the pencil path
// re-chunks j between its two exchanges).
// PASS 2: x forward * Poisson symbol * x backward (layout C, tiles over (jl, k-tile)).
// j0: global j of this rank's first local j (x pass symbol; 0 on one GPU).
// Results of a pass scattered straight into other ranks' workspaces (slab
// decomposition with peer-mapped buffers): output row `row`
// of chunk c = row >> shift goes to base[c] + (row & (2^shift - 1)) * kq, where
// base[c] is rank c's workspace advanced to this rank's chunk.  The all-to-all
// is then the pass's own stores (over NVLink), overlapping the transform tile
// by tile.
template <typename V>
struct PeerOut {
  V* base[kMaxPeers];
  int shift;
};

// SPL = 2: the quadrant layout of an n = 2N grid (poisson_quad.cuh): four chunks
// of N x N rows, one per (i parity, j parity) of the frequency; SPL = 3: nine
// chunks of an n = 3N grid (poisson_split3.cuh).  Lines stay inside a chunk,
// tile index gt = (chunk * lines + outer) * KT + k-tile, and the symbol reads
// ki = SPL i' + ci, kj = SPL j' + cj of the n-point transform (chunk = SPL ci + cj).
template <typename T, int N, int PASS, bool PEER = false, bool FIXED = false, int SPL = 0>
__global__ void __launch_bounds__(TmaCfg<T, N, (PASS < 2), PASS == 2 && x_wide<T, (SPL != 0)>()>::THREADS,
                                  TmaCfg<T, N, (PASS < 2), PASS == 2 && x_wide<T, (SPL != 0)>()>::MINB)
    k_strided_tma(const __grid_constant__ CUtensorMap tmap, vec2_t<T>* __restrict__ spec,
                  const vec2_t<T>* __restrict__ stw, T scale, T four_pi2, Layout g_, int nchunks_, int j0_, KSpan ks_,
                  vec2_t<T>* __restrict__ out_, Layout gout_, const __grid_constant__ PeerOut<vec2_t<T>> po) {
  static_assert(!(FIXED && PEER), "the fixed geometry is the single-GPU one");
  constexpr bool QUAD = SPL != 0;  // chunked split layout (i and j split by SPL)
  constexpr int NCH = spl_chunks(SPL);
  static_assert(!(QUAD && PEER), "the quadrant layout is single-GPU");
  const Layout g = FIXED ? fixed_geom<N, SPL, PASS>() : g_;
  const Layout gout = FIXED ? fixed_geom<N, SPL, PASS>() : gout_;
  const int nchunks = FIXED ? 1 : nchunks_;
  const int j0 = FIXED ? 0 : j0_;
  // FIXED: the single-GPU geometry (QUAD: a chunk of the 2N grid's quadrant layout)
  const KSpan ks = FIXED ? fixed_kspan<N, SPL, PASS>() : ks_;
  vec2_t<T>* __restrict__ out = FIXED ? spec : out_;
  using V = vec2_t<T>;
  using C = TmaCfg<T, N, (PASS < 2), PASS == 2 && x_wide<T, (SPL != 0)>()>;
  constexpr int E = C::E, P = C::P, L = C::L, TILE = C::TILE;
  constexpr uint32_t TILE_BYTES = TILE * sizeof(V);
  constexpr int NBUF = C::NBUF;
  const int KT = (ks.kc + L - 1) / L;
  const size_t kq = size_t(ks.kq);
  const int NL = (ks.no ? ks.no : (PASS < 2 ? g.ni : g.nj)) * KT;  // tiles per chunk (QUAD) / in all
  const int NT = NL * NCH;
  constexpr bool TWS = PASS == 2 ? bool(ARENA_TMA_TWSMEM_X) : bool(ARENA_TMA_TWSMEM_Y);
  constexpr bool E2S = C::E2S;
  constexpr int NST = num_stages(N, E);
  V* bufs = smem_base<V>();
  V* tws = bufs + NBUF * TILE + (E2S ? TILE / 2 : 0);  // E2S: half a tile of spare behind the tile buffer
  uint64_t* bar = reinterpret_cast<uint64_t*>(tws + (TWS ? C::TW : 0));
  const int tid = threadIdx.x;
  const int l = tid % L, t = tid / L;

  if (tid == 0) {
#pragma unroll
    for (int b = 0; b < NBUF + (E2S ? 1 : 0); ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  if constexpr (TWS) {
    for (int i = tid; i < C::TW; i += blockDim.x) tws[i] = __ldg(stw + i);
  }
  __syncthreads();
  // x pass: LDS from the staged table; y passes: the L1 path
  auto twp = [&]() {
    if constexpr (TWS) return SmemTable<V>{tws};
    else return stw;
  }();

  auto issue = [&](int gt, V* dst, uint64_t* b) {
    const int qd = QUAD ? gt / NL : 0;
    if constexpr (QUAD) gt -= qd * NL;
    const int outer = gt / KT, kt = gt % KT;
    mbar_arrive_expect_tx(b, TILE_BYTES);
    if constexpr (PASS < 2) {  // y tile: fixed il = outer, all j (QUAD: of chunk qd), two half boxes
      ytile_half_load(dst, &tmap, b, g, QUAD ? 1 : nchunks, 2 * kt * L, outer, qd, 0, TILE_BYTES);
      ytile_half_load(dst, &tmap, b, g, QUAD ? 1 : nchunks, 2 * kt * L, outer, qd, 1, TILE_BYTES);
    } else {  // x tile: fixed jl = outer, all i (chunk c, il blocks of IB)
      const int IB = tma_ib(g.ni);
      const int jb = (1 << g.jbs) - 1;
      for (int c = qd; c < (QUAD ? qd + 1 : nchunks); ++c)
        for (int q = 0; q < g.ni; q += IB)
          tma_load_5d(dst + (size_t(c - qd) * g.ni + q) * L, &tmap, b, 2 * kt * L, outer & jb, q, outer >> g.jbs, c);
    }
  };
  // E2S (x pass): half h of a tile = boxes [h NBX/2, (h + 1) NBX/2) of its NBX = chunks * ni/IB
  // boxes, completing bar[h]; with an odd box count (one box) the whole tile is half 1.
  auto issue_half = [&](int gt, int h) {
    const int qd = QUAD ? gt / NL : 0;
    if constexpr (QUAD) gt -= qd * NL;
    const int outer = gt / KT, kt = gt % KT;
    if constexpr (PASS < 2) {
      mbar_arrive_expect_tx(&bar[h], ytile_half_bytes(g, QUAD ? 1 : nchunks, h, TILE_BYTES));
      ytile_half_load(bufs, &tmap, &bar[h], g, QUAD ? 1 : nchunks, 2 * kt * L, outer, qd, h, TILE_BYTES);
      return;
    }
    const int IB = tma_ib(g.ni);
    const int jb = (1 << g.jbs) - 1;
    const int nbq = g.ni / IB, nbx = (QUAD ? 1 : nchunks) * nbq;
    const bool split = (nbx & 1) == 0;
    const int lo = split ? h * (nbx / 2) : (h ? 0 : nbx), hi = split ? lo + nbx / 2 : nbx;
    mbar_arrive_expect_tx(&bar[h], uint32_t(hi - lo) * uint32_t(IB * L * sizeof(V)));
    for (int bx = lo; bx < hi; ++bx) {
      const int c = bx / nbq, q = (bx - c * nbq) * IB;
      tma_load_5d(bufs + (size_t(c) * g.ni + q) * L, &tmap, &bar[h], 2 * kt * L, outer & jb, q, outer >> g.jbs, qd + c);
    }
  };
  auto prefetch = [&](int gt) {  // same boxes, into L2 only
    const int outer = gt / KT, kt = gt % KT;
    if constexpr (PASS < 2) {
      tma_prefetch_5d(&tmap, 2 * kt * L, 0, outer, 0, 0);
    } else {
      const int IB = tma_ib(g.ni);
      const int jb = (1 << g.jbs) - 1;
      for (int c = 0; c < nchunks; ++c)
        for (int q = 0; q < g.ni; q += IB) tma_prefetch_5d(&tmap, 2 * kt * L, outer & jb, q, outer >> g.jbs, c);
    }
  };

  // Prologue: tiles 0 .. NBUF-2 of this CTA in flight (and the next ones queued in L2).
  if (tid == 0) {
    for (int p = 1; p < ARENA_TMA_L2PF; ++p) {
      const int gp = blockIdx.x + p * gridDim.x;
      if (gp < NT) prefetch(gp);
    }
#pragma unroll
    for (int p = 0; p < NBUF - 1; ++p) {
      const int gp = blockIdx.x + p * gridDim.x;
      if (gp < NT) issue(gp, bufs + p * TILE, &bar[p]);
    }
  }
  int gt = blockIdx.x;
  // x pass, NBUF == 1: the first tile is requested here; every later one by the
  // previous iteration as soon as its last exchange has released the buffer, so
  // the load overlaps that iteration's last FFT stage and stores (B200: x 4.95
  // -> 4.32 ms).  The y passes measured 40% slower that way and request their
  // tile at the top of each iteration instead.
  constexpr bool EARLY = NBUF == 1 && (PASS == 2 || ARENA_TMA_EARLY_Y || E2S);
  if constexpr (E2S) {
    if (tid == 0 && gt < NT) {
      issue_half(gt, 0);
      issue_half(gt, 1);
    }
  } else if constexpr (EARLY) {
    if (tid == 0 && gt < NT) issue(gt, bufs, &bar[0]);
  }
  for (int it = 0; gt < NT; ++it, gt += gridDim.x) {
    const int b = it % NBUF;
    V* cur = bufs + b * TILE;
    if constexpr (ARENA_TMA_L2PF > 0) {
      const int gp = gt + ARENA_TMA_L2PF * gridDim.x;
      if (tid == 0 && gp < NT) prefetch(gp);
    }
    if constexpr (NBUF > 1) {
      const int gn = gt + (NBUF - 1) * gridDim.x;
      if (tid == 0 && gn < NT) {  // refill the buffer iteration it-1 used
        const int bn = (it + NBUF - 1) % NBUF;
        fence_proxy_async_smem();
        issue(gn, bufs + bn * TILE, &bar[bn]);
      }
    } else if constexpr (!EARLY) {
      if (tid == 0) {
        fence_proxy_async_smem();
        issue(gt, bufs, &bar[0]);
      }
    }
    mbar_wait(&bar[b], (it / NBUF) & 1);
    if constexpr (E2S) mbar_wait(&bar[1], it & 1);
    V v[E];
#pragma unroll
    for (int e = 0; e < E; ++e) v[e] = cur[(t + P * e) * L + l];
    __syncthreads();  // the tile buffer becomes exchange scratch
    const int qd = QUAD ? gt / NL : 0;
    const int gl = QUAD ? gt - qd * NL : gt;
    const int outer = gl / KT;
    const int k = (gl % KT) * L + l;
    auto release_half = [&](int h) {  // E2S: the half's region is free
      const int gn = gt + gridDim.x;
      if (tid == 0 && gn < NT) {
        fence_proxy_async_smem();
        issue_half(gn, h);
      }
    };
    auto release = [&]() {  // buffer free (all exchange reads done): request the next tile
      if constexpr (EARLY && !E2S) {
        const int gn = gt + gridDim.x;
        if (tid == 0 && gn < NT) {
          fence_proxy_async_smem();
          issue(gn, bufs, &bar[0]);
        }
      }
    };
    if constexpr (PASS < 2 && E2S) {
      // every exchange but the last in the tile buffer, then the first half of the next tile is
      // requested; the last exchange in the upper half + the spare half tile, then the second half
      constexpr int SG = PASS == 0 ? -1 : +1;
      V* sm2 = cur + TILE / 2;
      if constexpr (NST > 2) fft_stages<N, E, L, SG, kSyncCta, 0, V, decltype(twp), NST - 2>(v, cur, twp, t, l);
      release_half(0);
      fft_stages<N, E, L, SG, kSyncCta, NST - 2, V, decltype(twp), NST - 1>(v, sm2, twp, t, l);
      release_half(1);
      fft_stages<N, E, L, SG, kSyncCta, NST - 1, V, decltype(twp), NST>(v, sm2, twp, t, l);
    } else if constexpr (PASS == 0) {
      line_fft_head<N, E, L, -1>(v, cur, twp, t, l);
      release();
      line_fft_tail<N, E, L, -1>(v, cur, twp, t, l);
    } else if constexpr (PASS == 1) {
      line_fft_head<N, E, L, +1>(v, cur, twp, t, l);
      release();
      line_fft_tail<N, E, L, +1>(v, cur, twp, t, l);
    } else {
      if constexpr (E2S && NST == 2) {  // the forward exchange is the last use of the whole tile buffer
        fft_stages<N, E, L, -1, kSyncCta, 0, V, decltype(twp), 1>(v, cur, twp, t, l);
        release_half(0);
        fft_stages<N, E, L, -1, kSyncCta, 1, V, decltype(twp), 2>(v, cur, twp, t, l);
      } else {
        line_fft<N, E, L, -1>(v, cur, twp, t, l);
      }
      // full-grid frequencies: SPL > 0: (ki, kj) = (SPL i'' + ci, SPL j'' + cj), chunk SPL ci + cj
      constexpr int NG = SPL > 0 ? SPL * N : N;
      const T kj = SPL > 0 ? T(signed_freq(SPL * outer + qd % imax(SPL, 1), NG))
                   : ks.fm ? T(signed_freq(2 * (j0 + outer) + ks.fcj, 2 * N))
                           : T(signed_freq(j0 + outer, NG));
      const T kk = T(ks.k0 + k);
      const T c = kj * kj + kk * kk;
      auto kiof = [&](int e) {
        return SPL > 0 ? T(signed_freq(SPL * (t + P * e) + qd / imax(SPL, 1), NG))
               : ks.fm ? T(signed_freq(2 * (t + P * e) + ks.fci, 2 * N))
                       : T(signed_freq(t + P * e, NG));
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
      if constexpr (E2S) {
        V* sm2 = cur + TILE / 2;  // last exchange: upper half of the tile buffer + the spare half tile
        if constexpr (NST > 2) {
          fft_stages<N, E, L, +1, kSyncCta, 0, V, decltype(twp), NST - 2>(v, cur, twp, t, l);
          release_half(0);
        }
        fft_stages<N, E, L, +1, kSyncCta, NST - 2, V, decltype(twp), NST - 1>(v, sm2, twp, t, l);
        release_half(1);
        fft_stages<N, E, L, +1, kSyncCta, NST - 1, V, decltype(twp), NST>(v, sm2, twp, t, l);
      } else {
        line_fft_head<N, E, L, +1>(v, cur, twp, t, l);
        if constexpr (num_stages(N, E) == 1) __syncthreads();  // no exchange: make the buffer reads complete
        release();
        line_fft_tail<N, E, L, +1>(v, cur, twp, t, l);
      }
    }
    if (k < ks.kc) {
      auto dst = [&](V* base, size_t row) -> V* {
        if constexpr (PEER) {
          return po.base[row >> po.shift] + (row & ((size_t(1) << po.shift) - 1)) * kq + k;
        } else {
          return base + row * kq + k;
        }
      };
      if constexpr (PASS < 2) {
#pragma unroll
        for (int e = 0; e < E; ++e)
          st_out(dst(out, QUAD ? lrow(gout, qd, outer, t + P * e) : rowB(gout, outer, t + P * e)), v[e]);
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e)
          st_out(dst(spec, QUAD ? lrow(g, qd, t + P * e, outer) : rowC(g, t + P * e, outer)), v[e]);
      }
    }
    // No barrier needed here: every thread's last access to `cur` (the tile
    // read, or the last exchange read) is followed by a __syncthreads, so
    // thread 0 only refills it next iteration after all threads are done.
  }
  if constexpr (PEER) __threadfence_system();  // peer stores performed before the ranks' barrier
}

}  // namespace arena_fft

// ============================================================ pencil z passes
// Pencil decomposition: a rank owns the f / u block
// (ni = n/Pr planes) x (nj = n/Pc rows of j) x n, rows (il, jl) contiguous.  K1
// writes each row's half spectrum split into Pc k-chunks of kq complex — chunk
// c is the block sent to column c of the rank's row group — and K5 gathers them
// back.  Inside a chunk rows are in Layout(ni, nj) order.
namespace arena_fft {

// PEER: k-chunk c goes straight to po.base[c] (row peer c's Y buffer, advanced
// to this rank's chunk) instead of chunk c of R — the row all-to-all fused into K1.
template <typename T, int NR, bool PEER = false>
__global__ void __launch_bounds__(ContigCfg<T, NR>::THREADS, ContigCfg<T, NR>::MINB)
    k_zfwd_pencil(const T* __restrict__ f, vec2_t<T>* __restrict__ R, const vec2_t<T>* __restrict__ tw,
                  const vec2_t<T>* __restrict__ stw, Layout gz, int kq, const __grid_constant__ PeerOut<vec2_t<T>> po) {
  using V = vec2_t<T>;
  using C = ContigCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L;
  constexpr int SW = engine_swizzle<M, E>();
  V* sm = smem_base<V>();
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  if constexpr (ARENA_Z_PF > 0) {  // as k_zfwd: the rows one resident wave ahead into L2
    const unsigned b = blockIdx.x + C::PF;
    if (threadIdx.x == 0 && b < gridDim.x) bulk_prefetch_l2(f + size_t(b) * C::L * NR, C::L * NR * sizeof(T));
  }
  const size_t row = size_t(blockIdx.x) * L + l;  // il * nj + jl
  const V* src = reinterpret_cast<const V*>(f + row * NR);
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  line_fft<M, E, L, -1>(v, sm, stw, t, l);
  constexpr bool PAIRS = ARENA_Z_PAIRS && E >= 2 && (E % 2) == 0 && ARENA_Z_TWREC && E <= 32;
#pragma unroll
  for (int e = PAIRS ? E / 2 : 0; e < E; ++e) sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  __syncthreads();
  const size_t rin = lrow(gz, 0, int(row >> gz.njs), int(row & (gz.nj - 1)));
  const size_t chunk = size_t(gz.ni) * gz.nj;
  auto put = [&](int k, V x) {
    const int c = k / kq;
    if constexpr (PEER) {
      po.base[c][rin * kq + (k - c * kq)] = x;
    } else {
      R[(size_t(c) * chunk + rin) * kq + (k - c * kq)] = x;
    }
  };
  const V wt = tw_load(tw, t);  // W_n^t (split_twiddle)
  if constexpr (PAIRS) {  // Hermitian pairs (k, M - k) from one thread, as zfwd_rows
    const V wh{T(-0.5) * wt.y, T(0.5) * wt.x};  // (i/2) W_n^t
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int k = t + P * e;
      const V A = v[e];
      const V Bc = k == 0 ? A : sm[smem_idx<L, SW, V>(M - k, l)];
      const V B{Bc.x, -Bc.y};
      const V Wh = split_twiddle<E>(tw, wh, k, e);  // (i/2) W_n^k
      const V U = cmul(Wh, csub(A, B));
      const V Sm = cadd(A, B);
      put(k, V{fma(T(0.5), Sm.x, -U.x), fma(T(0.5), Sm.y, -U.y)});
      V Xm{fma(T(0.5), Sm.x, U.x), -fma(T(0.5), Sm.y, U.y)};
      if (k == 0) Xm.y = T(0);
      put(M - k, Xm);
    }
    if (t == 0) put(M / 2, V{v[E / 2].x, -v[E / 2].y});
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int k = t + P * e;
      const V A = v[e];
      const V Bc = sm[smem_idx<L, SW, V>((M - k) & (M - 1), l)];
      const V B{Bc.x, -Bc.y};
      const V W = split_twiddle<E>(tw, wt, k, e);
      const V WD = cmul(W, csub(A, B));
      put(k, V{T(0.5) * (A.x + B.x + WD.y), T(0.5) * (A.y + B.y - WD.x)});
      if (k == 0) put(M, V{A.x - A.y, T(0)});
    }
  }
  if constexpr (PEER) __threadfence_system();
}

template <typename T, int NR>
__global__ void __launch_bounds__(ContigCfg<T, NR>::THREADS, ContigCfg<T, NR>::MINB)
    k_zinv_pencil(const vec2_t<T>* __restrict__ R, T* __restrict__ u, const vec2_t<T>* __restrict__ tw,
                  const vec2_t<T>* __restrict__ stw, Layout gz, int kq) {
  using V = vec2_t<T>;
  using C = ContigCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L;
  constexpr int SW = engine_swizzle<M, E>();
  V* sm = smem_base<V>();
  V* xm = sm + M * L;
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const size_t row = size_t(blockIdx.x) * L + l;
  const size_t rin = lrow(gz, 0, int(row >> gz.njs), int(row & (gz.nj - 1)));
  const size_t chunk = size_t(gz.ni) * gz.nj;
  if constexpr (ARENA_Z_PF > 0) {  // the k-chunks of the rows one resident wave ahead into L2
    const unsigned b = blockIdx.x + C::PF;
    const int nch = (M + 1 + kq - 1) / kq;
    if (b < gridDim.x && threadIdx.x < L * nch) {
      const size_t rb = size_t(b) * L + threadIdx.x % L;
      const int c = threadIdx.x / L;
      const size_t rinb = lrow(gz, 0, int(rb >> gz.njs), int(rb & (gz.nj - 1)));
      bulk_prefetch_l2(R + (size_t(c) * chunk + rinb) * kq, kq * sizeof(V));
    }
  }
  auto get = [&](int k) {
    const int c = k / kq;
    return __ldcs(R + (size_t(c) * chunk + rin) * kq + (k - c * kq));
  };
  V v[E];
  constexpr bool PAIRS = ARENA_Z_PAIRS && E >= 2 && (E % 2) == 0 && ARENA_Z_TWREC && E <= 32;
  if constexpr (PAIRS) {  // Hermitian pairs (k, M - k) from one thread, as zinv_rows
    const V wt = tw_load(tw, t);
    const V wi{wt.y, wt.x};  // i conj(W_n^t)
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int k = t + P * e;
      V A = get(k);
      V C = get(M - k);
      if (k == 0) {
        A.y = T(0);
        C.y = T(0);
      }
      const V B{C.x, -C.y};
      const V Wi = cmulc(wi, w64((e * (32 / E)) & 63, T(0)));  // i conj(W_n^k)
      const V Ep = cadd(A, B);
      const V Op = cmul(csub(A, B), Wi);
      v[e] = cadd(Ep, Op);
      if (k != 0) sm[smem_idx<L, SW, V>(M - k, l)] = V{Ep.x - Op.x, Op.y - Ep.y};
    }
    if (t == 0) {
      const V h = get(M / 2);
      sm[smem_idx<L, SW, V>(M / 2, l)] = V{T(2) * h.x, T(-2) * h.y};
    }
    __syncthreads();
#pragma unroll
    for (int e = E / 2; e < E; ++e) v[e] = sm[smem_idx<L, SW, V>(t + P * e, l)];
  } else {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    v[e] = get(t + P * e);
    sm[smem_idx<L, SW, V>(t + P * e, l)] = v[e];
  }
  if (t == 0) xm[l] = get(M);
  __syncthreads();
  const V wt = tw_load(tw, t);  // W_n^t (split_twiddle)
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    V A = v[e];
    V Bs = (k == 0) ? xm[l] : sm[smem_idx<L, SW, V>(M - k, l)];
    if (k == 0) {
      A.y = T(0);
      Bs.y = T(0);
    }
    const V B{Bs.x, -Bs.y};
    const V W = split_twiddle<E>(tw, wt, k, e);
    const V Ep = cadd(A, B);
    const V Op = cmulc(csub(A, B), W);
    v[e] = V{Ep.x - Op.y, Ep.y + Op.x};
  }
  }
  __syncthreads();
  line_fft<M, E, L, +1>(v, sm, stw, t, l);
  V* dst = reinterpret_cast<V*>(u + row * NR);
#pragma unroll
  for (int e = 0; e < E; ++e) st_out(dst + t + P * e, v[e]);
}

}  // namespace arena_fft
