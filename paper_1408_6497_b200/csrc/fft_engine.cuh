// fft_engine.cuh — register/shared-memory FFT line engine for sm_100a.
//
// Replaces the FFTW codelets the reference calls at
// /root/reference/proj/src/fft_solver.cpp:65 (r2c execute) and :80 (c2r
// execute).  Same DFT conventions (FFTW's published definitions): forward is
// exp(-2 pi i k x / n), unnormalised; backward exp(+...), unnormalised.
//
// Formulation: Stockham autosort, radix-2^k stages (Govindaraju et al. 2008).
// One "tile" = L independent lines of length N, processed by L*P threads
// (P = N/E threads per line, each thread holding E points in registers).
// Thread (l, t) — l fastest in threadIdx.x — always holds line-l elements
// t + P*e, e in [0, E), both before the first stage and after the last stage,
// so global loads and stores use the same (coalesced) pattern, and a forward
// transform can feed an inverse one without leaving registers (the fused
// x-pass).  Between stages the tile is exchanged through shared memory laid
// out [position][line] so that the 8 lanes of a 16-byte shared-memory phase
// hit 8 distinct bank groups.
#pragma once

#include <cuda_runtime.h>


#include <stdint.h>

namespace arena_fft {

// ---------------------------------------------------------------- complex ops
template <typename T>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};
template <typename T>
using vec2_t = typename Vec2<T>::type;

template <typename V>
__device__ __forceinline__ V cadd(V a, V b) {
  return V{a.x + b.x, a.y + b.y};
}
template <typename V>
__device__ __forceinline__ V csub(V a, V b) {
  return V{a.x - b.x, a.y - b.y};
}
// a * w
template <typename V>
__device__ __forceinline__ V cmul(V a, V w) {
  return V{fma(a.x, w.x, -a.y * w.y), fma(a.x, w.y, a.y * w.x)};
}
// a * conj(w)
template <typename V>
__device__ __forceinline__ V cmulc(V a, V w) {
  return V{fma(a.x, w.x, a.y * w.y), fma(a.y, w.x, -a.x * w.y)};
}
// a * (S * i), S = +-1
template <int S, typename V>
__device__ __forceinline__ V cmul_si(V a) {
  return S > 0 ? V{-a.y, a.x} : V{a.y, -a.x};
}

// fp32: the same operations on packed pairs (sm_100 FADD2 / FMUL2 / FFMA2: one
// instruction for both components; the fp32 passes are issue-bound).
#ifndef ARENA_F32X2
#define ARENA_F32X2 2  // 0: off, 1: sums, 2: sums and products
#endif
#if ARENA_F32X2
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return __ffma2_rn(b, make_float2(-1.f, -1.f), a); }
#endif
#if ARENA_F32X2 >= 2  // products too (the operand broadcasts cost MOVs)
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
  return __ffma2_rn(make_float2(a.x, a.x), w, __fmul2_rn(make_float2(a.y, a.y), make_float2(-w.y, w.x)));
}
__device__ __forceinline__ float2 cmulc(float2 a, float2 w) {
  return __ffma2_rn(make_float2(a.x, a.x), make_float2(w.x, -w.y), __fmul2_rn(make_float2(a.y, a.y), make_float2(w.y, w.x)));
}
#endif

// cos(2 pi m / 64), m = 0..16 (first quadrant), double-rounded.
constexpr double kCos64[17] = {1.0,
                               0.9951847266721969,
                               0.9807852804032304,
                               0.9569403357322088,
                               0.9238795325112867,
                               0.881921264348355,
                               0.8314696123025452,
                               0.773010453362737,
                               0.7071067811865476,
                               0.6343932841636455,
                               0.5555702330196022,
                               0.47139673682599764,
                               0.3826834323650898,
                               0.2902846772544624,
                               0.19509032201612828,
                               0.0980171403295606,
                               0.0};

constexpr double cos64(int m) {
  m = ((m % 64) + 64) % 64;
  const int q = m / 16, r = m % 16;
  return q == 0 ? kCos64[r] : q == 1 ? -kCos64[16 - r] : q == 2 ? -kCos64[r] : kCos64[16 - r];
}
constexpr double sin64(int m) { return cos64(m - 16); }

// a * exp(S * 2 pi i * E / R), R | 64, all compile-time.
template <int R, int E, int S, typename V>
__device__ __forceinline__ V cmul_const(V a) {
  constexpr int m = ((E * (64 / R)) % 64 + 64) % 64;
  if constexpr (m == 0) {
    return a;
  } else if constexpr (m == 16) {
    return cmul_si<S>(a);
  } else if constexpr (m == 32) {
    return V{-a.x, -a.y};
  } else if constexpr (m == 48) {
    return cmul_si<-S>(a);
  } else {
    using T = decltype(a.x);
    constexpr T c = T(cos64(m));
    constexpr T s = T(S * sin64(m));
#if ARENA_F32X2 >= 2
    if constexpr (sizeof(T) == 4) {
      return __ffma2_rn(make_float2(a.x, a.x), make_float2(c, s), __fmul2_rn(make_float2(a.y, a.y), make_float2(-s, c)));
    }
#endif
    return V{fma(a.x, c, -a.y * s), fma(a.x, s, a.y * c)};
  }
}

// ---------------------------------------------------------- in-register DFTs
// In-place DFT of x[0..R) with sign S (-1 forward, +1 backward), natural order
// in and out.  R = 1, 2, 4 directly; larger powers of two by one radix-4 (or
// radix-2) decimation-in-time step over recursive sub-DFTs, all indices and
// twiddles compile-time so everything stays in registers.
// FMA: the twiddled radix-4 steps in FMA form (bfly4_tw below) — on for the 32-point
// butterflies of the fp64 x pass and z passes; the 16- / 8-point stages of the y passes
// (128-register kernels) measured 1.5% slower with it (a 32-byte spill).
template <int R, int S, bool FMA = (R >= 32)>
struct Dft;

template <int S, bool FMA>
struct Dft<1, S, FMA> {
  template <typename V>
  __device__ __forceinline__ static void run(V*) {}
};

template <int S, bool FMA>
struct Dft<2, S, FMA> {
  template <typename V>
  __device__ __forceinline__ static void run(V* x) {
    const V t = x[1];
    x[1] = csub(x[0], t);
    x[0] = cadd(x[0], t);
  }
};

template <int S, bool FMA>
struct Dft<4, S, FMA> {
  template <typename V>
  __device__ __forceinline__ static void run(V* x) {
    const V s02 = cadd(x[0], x[2]), d02 = csub(x[0], x[2]);
    const V s13 = cadd(x[1], x[3]), d13 = cmul_si<S>(csub(x[1], x[3]));
    x[0] = cadd(s02, s13);
    x[2] = csub(s02, s13);
    x[1] = cadd(d02, d13);
    x[3] = csub(d02, d13);
  }
};

// FMA form of the twiddled radix-4 step (Linzer & Feig style): a constant twiddle is
// written W = rho * C * (1 + i T) with rho in {1, S i}, |T| <= 1 (the angle reduced to
// (-pi/4, pi/4] by quarter turns, a half turn folded into the sign of C), so W a = C a'
// with a' = rho (a.x - T a.y, a.y + T a.x) — two FMAs instead of the four operations of a
// complex product — and the scale C rides on the butterfly's additions, which become FMAs:
//   s02 = a0 + C2 a2', d02 = a0 - C2 a2', u = a1' + (C3/C1) a3', v = a1' - (C3/C1) a3',
//   x0 = s02 + C1 u, x2 = s02 - C1 u, x1 = d02 + C1 (S i) v, x3 = d02 - C1 (S i) v.
// A 32-point DFT takes 376 fp64 instructions instead of 436 (FFTW's n1_32 codelet: 372).
#ifndef ARENA_DFT_FMA
#define ARENA_DFT_FMA 1  // 0: separate complex products (cmul_const) and additions
#endif
template <int R, int EX, int S>
struct CTw {  // exp(S 2 pi i EX / R)
  static constexpr int M = ((EX * (64 / R)) % 64 + 64) % 64;
  static constexpr int QT = (M + 7) / 16;         // quarter turns taken out (0..4)
  static constexpr int RM = M - 16 * QT;          // residual angle in 64ths of a turn, [-7, 8]
  static constexpr bool ROT = (QT & 1) != 0;      // rho = S i (else 1)
  static constexpr double C = ((QT & 2) ? -1.0 : 1.0) * cos64(RM);
  static constexpr double T = S * sin64(RM) / cos64(RM);
};
// a' = rho (1 + i T) a
template <typename W, int S, typename V>
__device__ __forceinline__ V tw_rot(V a) {
  using T = decltype(a.x);
  V r;
  if constexpr (W::RM == 0) {
    r = a;
  } else if constexpr (W::RM == 8) {  // T = S
    r = S > 0 ? V{a.x - a.y, a.y + a.x} : V{a.x + a.y, a.y - a.x};
  } else {
    constexpr T tau = T(W::T);
    r = V{fma(-tau, a.y, a.x), fma(tau, a.x, a.y)};
  }
  if constexpr (W::ROT) return cmul_si<S>(r);
  else return r;
}
#ifndef ARENA_DFT_FMA32
#define ARENA_DFT_FMA32 1  // the FMA form for fp32 too, on packed pairs (FFMA2)
#endif
#ifndef ARENA_DFT_FMA32_ALL
#define ARENA_DFT_FMA32_ALL 0  // fp32: also the 16- / 8-point stages (y passes)
#endif
#if ARENA_F32X2 >= 2
// fp32: a' = a + (-T, T) (a.y, a.x), one packed FFMA2 on the swapped pair
template <typename W, int S>
__device__ __forceinline__ float2 tw_rot(float2 a) {
  float2 r;
  if constexpr (W::RM == 0) {
    r = a;
  } else {
    constexpr float tau = W::RM == 8 ? float(S) : float(W::T);
    r = __ffma2_rn(make_float2(-tau, tau), make_float2(a.y, a.x), a);
  }
  if constexpr (W::ROT) return cmul_si<S>(r);
  else return r;
}
__device__ __forceinline__ void axpy_pm(double c, float2 x, float2 y, float2& plus, float2& minus) {
  if (c == 1.0) {
    plus = cadd(y, x);
    minus = csub(y, x);
  } else if (c == -1.0) {
    plus = csub(y, x);
    minus = cadd(y, x);
  } else {
    const float cc = float(c);
    plus = __ffma2_rn(make_float2(cc, cc), x, y);
    minus = __ffma2_rn(make_float2(-cc, -cc), x, y);
  }
}
#endif
// y + c x, y - c x with a compile-time real c (plain sums when c = +-1)
template <typename V>
__device__ __forceinline__ void axpy_pm(double c, V x, V y, V& plus, V& minus) {
  using T = decltype(x.x);
  if (c == 1.0) {
    plus = cadd(y, x);
    minus = csub(y, x);
  } else if (c == -1.0) {
    plus = csub(y, x);
    minus = cadd(y, x);
  } else {
    const T cc = T(c);
    plus = V{fma(cc, x.x, y.x), fma(cc, x.y, y.y)};
    minus = V{fma(-cc, x.x, y.x), fma(-cc, x.y, y.y)};
  }
}
// Radix-4 butterfly over inputs a0, W^{K1} a1, W^{2 K1} a2, W^{3 K1} a3 (W = exp(S 2 pi i / R)).
template <int R, int K1, int S, typename V>
__device__ __forceinline__ void bfly4_tw(V a0, V a1, V a2, V a3, V& x0, V& x1, V& x2, V& x3) {
  using W1 = CTw<R, K1, S>;
  using W2 = CTw<R, 2 * K1, S>;
  using W3 = CTw<R, 3 * K1, S>;
  const V p1 = tw_rot<W1, S>(a1), p2 = tw_rot<W2, S>(a2), p3 = tw_rot<W3, S>(a3);
  V s02, d02, u, v;
  axpy_pm(W2::C, p2, a0, s02, d02);
  axpy_pm(W3::C / W1::C, p3, p1, u, v);
  axpy_pm(W1::C, u, s02, x0, x2);
  axpy_pm(W1::C, cmul_si<S>(v), d02, x1, x3);
}
template <int R, int S, int K1, typename V, int Q>
__device__ __forceinline__ void bfly4_all(V (&a)[4][Q], V* x) {
  if constexpr (K1 < Q) {
    V b0, b1, b2, b3;
    bfly4_tw<R, K1, S>(a[0][K1], a[1][K1], a[2][K1], a[3][K1], b0, b1, b2, b3);
    x[K1] = b0;
    x[K1 + Q] = b1;
    x[K1 + 2 * Q] = b2;
    x[K1 + 3 * Q] = b3;
    bfly4_all<R, S, K1 + 1>(a, x);
  }
}

template <int R, int S, bool FMA>
struct Dft {
  static_assert(R % 4 == 0 && R <= 64, "power-of-two radix <= 64");
  template <typename V>
  __device__ __forceinline__ static void run(V* x) {
    constexpr int Q = R / 4;
    V a[4][Q];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1)
#pragma unroll
      for (int n2 = 0; n2 < Q; ++n2) a[n1][n2] = x[4 * n2 + n1];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) Dft<Q, S, FMA>::run(a[n1]);
    constexpr bool F32 = sizeof(x[0].x) == 4;
    constexpr bool kFmaForm = ARENA_DFT_FMA && (F32 ? (ARENA_DFT_FMA32 && ARENA_F32X2 >= 2 && (FMA || ARENA_DFT_FMA32_ALL)) : FMA);
    if constexpr (kFmaForm) {
      bfly4_all<R, S, 0>(a, x);
    } else {
      twiddle_all<1, 0>(a);
#pragma unroll
      for (int k1 = 0; k1 < Q; ++k1) {
        V b[4] = {a[0][k1], a[1][k1], a[2][k1], a[3][k1]};
        Dft<4, S, false>::run(b);
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) x[k1 + Q * k2] = b[k2];
      }
    }
  }
  // compile-time loop applying W_R^{S n1 k1}
  template <int N1, int K1, typename V, int Q>
  __device__ __forceinline__ static void twiddle_all(V (&a)[4][Q]) {
    if constexpr (N1 < 4) {
      if constexpr (K1 < Q) {
        a[N1][K1] = cmul_const<R, N1 * K1, S>(a[N1][K1]);
        twiddle_all<N1, K1 + 1>(a);
      } else {
        twiddle_all<N1 + 1, 0>(a);
      }
    }
  }
};

// ------------------------------------------------------------- stage plans
constexpr int ilog2(int x) { return x <= 1 ? 0 : 1 + ilog2(x / 2); }
constexpr int cdiv(int a, int b) { return (a + b - 1) / b; }

// Number of Stockham stages for an N-point line with E points per thread,
// and the radix (log2) of stage s: bits split as evenly as possible, larger
// radices first.
constexpr int num_stages(int N, int E) { return N <= 1 ? 0 : cdiv(ilog2(N), ilog2(E)); }
constexpr int stage_log2(int N, int E, int s) {
  const int ns = num_stages(N, E), b = ilog2(N);
  return b / ns + (s < b % ns ? 1 : 0);
}
constexpr int stage_ns(int N, int E, int s) {  // product of radices before stage s
  return s == 0 ? 1 : stage_ns(N, E, s - 1) << stage_log2(N, E, s - 1);
}

// Shared-memory element index of (position, line).  A 128-byte shared-memory
// phase covers G = 128/sizeof(V)/L positions; when G > 1 XOR-swizzle the low
// bits of the position with bits above the first-stage radix so both the
// natural-order reads and the first stage's stride-R writes are conflict-free.
template <int L, int SW, typename V>
__device__ __forceinline__ int smem_idx(int pos, int l) {
  constexpr int G = int(128 / sizeof(V)) / L;  // positions per shared-memory phase
  if constexpr (G <= 1 || SW == 0) {
    return pos * L + l;
  } else {
    return (pos ^ ((pos >> SW) & (G - 1))) * L + l;
  }
}

// Twiddle table reads through the read-only (L1) path.  (Staging the stage
// tables in shared memory measured no faster on B200, and a plain generic
// load made the classic x kernel 30% slower.)
#ifndef ARENA_TW_LD
#define ARENA_TW_LD 0  // 0: ld.global.nc, 1: ld.global.nc.L1::evict_last (B200 A/B: evict_last saved 0.3 ms
                       // per 1024^3 solve with 8-row j blocks; with 64-row blocks plain loads win:
                       // 16.38 -> 16.24 ms, y passes 3.20 -> 3.10 ms; 2048^3 +0.5%)
#endif
#ifndef ARENA_ST_MODE
#define ARENA_ST_MODE 2  // data stores: 0 st.global.cs, 1 st.global, 2 st.global.L1::no_allocate
#endif
__device__ __forceinline__ double2 ldg_keep(const double2* p) {
  double2 v;
  asm("ld.global.nc.L1::evict_last.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ float2 ldg_keep(const float2* p) {
  float2 v;
  asm("ld.global.nc.L1::evict_last.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
template <typename V>
__device__ __forceinline__ V tw_load(const V* __restrict__ tw, int idx) {
  if constexpr (ARENA_TW_LD == 1) return ldg_keep(tw + idx);
  else return __ldg(tw + idx);
}
// Streaming store of a result element (write-once data: keep it out of L1).
__device__ __forceinline__ void st_na(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void st_na(float2* p, float2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v.x), "f"(v.y) : "memory");
}
template <typename V>
__device__ __forceinline__ void st_out(V* p, V v) {
  if constexpr (ARENA_ST_MODE == 0) __stcs(p, v);
  else if constexpr (ARENA_ST_MODE == 1) *p = v;
  else st_na(p, v);
}
// A twiddle table staged in shared memory (plain loads -> LDS).
template <typename V>
struct SmemTable {
  const V* p;
  __device__ __forceinline__ SmemTable operator+(int o) const { return SmemTable{p + o}; }
};
template <typename V>
__device__ __forceinline__ V tw_load(SmemTable<V> tw, int idx) {
  return tw.p[idx];
}

// Multiply by a table twiddle (forward sign) or its conjugate (backward).
template <int S, typename V, typename TW>
__device__ __forceinline__ V tw_apply(V a, TW tw, int idx) {
  const V w = tw_load(tw, idx);
  return S < 0 ? cmul(a, w) : cmulc(a, w);
}

// Per-stage twiddle tables.  Stage s >= 1 (radix R, NS = product of the
// earlier radices) multiplies input r of butterfly j by W_{NS*R}^{(j mod NS) r};
// they are stored as tab_s[r*NS + (j mod NS)], so the lanes of a warp (adjacent
// j) read adjacent entries — one 128-byte wavefront instead of one per lane
// group.  Tables for consecutive stages are concatenated (stage_tw_offset).
constexpr int stage_tw_size(int N, int E, int s) { return (1 << stage_log2(N, E, s)) * stage_ns(N, E, s); }
constexpr int stage_tw_offset(int N, int E, int s) {  // offset of stage s (>= 1) in the (N, E) table
  return s <= 1 ? 0 : stage_tw_offset(N, E, s - 1) + stage_tw_size(N, E, s - 1);
}
constexpr int stage_tw_total(int N, int E) { return num_stages(N, E) <= 1 ? 0 : stage_tw_offset(N, E, num_stages(N, E)); }

// One Stockham stage on registers (no exchange).  Thread holds elements
// t + P*e; butterfly q uses v[q + NB*r], r < R.
template <int N, int E, int R, int NS, int S, typename V, typename TW>
__device__ __forceinline__ void stage_compute(V (&v)[E], int t, TW stw) {
  constexpr int P = N / E, NB = E / R;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    V a[R];
#pragma unroll
    for (int r = 0; r < R; ++r) a[r] = v[q + NB * r];
    if constexpr (NS > 1) {
      const int jj = (t + P * q) & (NS - 1);
#pragma unroll
      for (int r = 1; r < R; ++r) a[r] = tw_apply<S>(a[r], stw, r * NS + jj);
    }
    Dft<R, S>::run(a);
#pragma unroll
    for (int r = 0; r < R; ++r) v[q + NB * r] = a[r];
  }
}

// Barrier scope of the exchanges: the whole CTA, or one warp when a warp owns
// its lines and their shared-memory region exclusively.
enum { kSyncCta = 0, kSyncWarp = 1 };
template <int SYNC>
__device__ __forceinline__ void xbarrier() {
  if constexpr (SYNC == kSyncWarp) {
    __syncwarp();
  } else {
    __syncthreads();
  }
}

// Called after every exchange barrier (a caller's producer thread can advance its
// asynchronous copies there without a barrier of its own); no-op by default.
struct NoHook {
  __device__ __forceinline__ void operator()() const {}
};

// Write stage outputs to shared memory at their Stockham destinations and
// read back the natural-order inputs of the next stage.
template <int N, int E, int L, int R, int NS, int SW, int SYNC, typename V, typename HK = NoHook>
__device__ __forceinline__ void stage_exchange(V (&v)[E], V* sm, int t, int l, const HK& hook = HK{}) {
  constexpr int P = N / E, NB = E / R;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    const int b = t + P * q;
    const int dst = (b & ~(NS - 1)) * R + (b & (NS - 1));
#pragma unroll
    for (int r = 0; r < R; ++r) sm[smem_idx<L, SW, V>(dst + r * NS, l)] = v[q + NB * r];
  }
  xbarrier<SYNC>();
  hook();
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = sm[smem_idx<L, SW, V>(t + P * e, l)];
  xbarrier<SYNC>();
  hook();
}

// Stages STAGE .. STOP-1 of the N-point transform, each followed by its exchange through
// `sm` unless it is the transform's last stage.
template <int N, int E, int L, int S, int SYNC, int STAGE, typename V, typename TW, int STOP = num_stages(N, E),
          typename HK = NoHook>
__device__ __forceinline__ void fft_stages(V (&v)[E], V* sm, TW stw, int t, int l, const HK& hook = HK{}) {
  constexpr int NSTAGE = num_stages(N, E);
  if constexpr (STAGE < STOP) {
    constexpr int R = 1 << stage_log2(N, E, STAGE);
    constexpr int NS = stage_ns(N, E, STAGE);
    constexpr int SW = stage_log2(N, E, 0);
    stage_compute<N, E, R, NS, S>(v, t, stw + (STAGE >= 1 ? stage_tw_offset(N, E, STAGE) : 0));
    if constexpr (STAGE + 1 < NSTAGE) stage_exchange<N, E, L, R, NS, SW, SYNC>(v, sm, t, l, hook);
    fft_stages<N, E, L, S, SYNC, STAGE + 1, V, TW, STOP>(v, sm, stw, t, l, hook);
  }
}

// Full N-point line FFT of the tile.  On entry and exit thread (l, t) holds
// line-l elements t + P*e (natural order).  `sm` must hold N*L elements and
// be free (all threads past their last access) on entry; on exit it is free.
// `stw` is the (N, E) stage-twiddle table (stage_tw_total(N, E) entries).
template <int N, int E, int L, int S, int SYNC = kSyncCta, typename V, typename TW, typename HK = NoHook>
__device__ __forceinline__ void line_fft(V (&v)[E], V* sm, TW stw, int t, int l, const HK& hook = HK{}) {
  fft_stages<N, E, L, S, SYNC, 0, V, TW, num_stages(N, E), HK>(v, sm, stw, t, l, hook);
}

// The same transform split in two: `head` runs every stage but the last
// (with all exchanges, so `sm` is free on return), `tail` the last stage,
// in registers only.  Lets a caller refill `sm` while the tail computes.
template <int N, int E, int L, int S, int SYNC = kSyncCta, typename V, typename TW, typename HK = NoHook>
__device__ __forceinline__ void line_fft_head(V (&v)[E], V* sm, TW stw, int t, int l, const HK& hook = HK{}) {
  constexpr int NST = num_stages(N, E);
  if constexpr (NST > 1) fft_stages<N, E, L, S, SYNC, 0, V, TW, NST - 1, HK>(v, sm, stw, t, l, hook);
}
template <int N, int E, int L, int S, int SYNC = kSyncCta, typename V, typename TW>
__device__ __forceinline__ void line_fft_tail(V (&v)[E], V* sm, TW stw, int t, int l) {
  constexpr int NST = num_stages(N, E);
  if constexpr (NST > 0) fft_stages<N, E, L, S, SYNC, NST - 1, V, TW, NST>(v, sm, stw, t, l);
}

// Swizzle parameter callers must use when they stage data in `sm` in the
// engine's layout (natural position order).
template <int N, int E>
constexpr int engine_swizzle() {
  return N <= 1 ? 0 : stage_log2(N, E, 0);
}

}  // namespace arena_fft
