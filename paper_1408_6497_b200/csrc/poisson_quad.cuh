// poisson_quad.cuh — the quadrant formulation of the single-GPU power-of-two
// solve for long lines (n >= 2048 by default).
//
// At n = 2048 a strided tile of 8 fp64 lines (128-byte rows, the DRAM-friendly
// width) is 256 KB, more than an SM's shared memory, so the y / x passes ran
// 4- and 2-line tiles (64- and 32-byte rows) at 55-65% of the 1024^3 passes'
// bandwidth.  Here the first radix-2 step of the i and j transforms moves into
// the z passes, which hold whole rows anyway:
//
//   for n = 2H, a row quad (i', j'), (i', j'+H), (i'+H, j'), (i'+H, j'+H):
//   Y_{ci,cj}[i', j', k] = W_n^{ci i' + cj j'} sum_{a,b} (-1)^{a ci + b cj} X_{a,b}[i', j', k]
//
// (X = the row's r2c half spectrum), after which X[2 i'' + ci, 2 j'' + cj, k] is
// the H x H two-dimensional DFT of Y_{ci,cj} over (i', j') — four independent
// quadrant problems whose y and x lines are H points long, run by the H-point
// TMA kernels (k_strided_tma<..., QUAD>) with 128-byte rows.  The inverse z pass
// undoes it: x_{a,b} = sum_{ci,cj} (-1)^{a ci + b cj} W_n^{-(ci i' + cj j')} Y'_{ci,cj}.
// The symbol uses the full-grid frequencies ki = 2 i'' + ci, kj = 2 j'' + cj, so
// the result is the same DFT as fft_solver.cpp:60-80 computes, in another order.
//
// Workspace: Layout(H, H) with four chunks, chunk q = 2 ci + cj; the 2x2
// butterfly runs in registers on columns k of the quad staged in shared memory.
#pragma once

#include "poisson_pow2.cuh"

namespace arena_fft {

template <typename T, int NR>
struct QuadZCfg {
  static constexpr int M = NR / 2;  // complex points of a packed row
  static constexpr int H = NR / 2;  // quadrant extent in i and j
  // 32 points per thread for long rows: one exchange in the row FFT (the z passes
  // are bound by shared-memory traffic at n = 2048); two 128-thread CTAs per SM.
#ifndef ARENA_QUAD_E
#define ARENA_QUAD_E 32
#endif
  static constexpr int E = NR >= 1024 ? imin(ARENA_QUAD_E, M) : ContigCfg<T, NR>::E;
  static constexpr int P = M / E;
  static constexpr int L = 4;  // the four rows of a quad, one CTA
  static constexpr int THREADS = L * P;
  // Row FFTs run in groups of RW rows (row index fastest inside a group): a warp
  // owns whole rows when P <= 32, so their exchanges need only __syncwarp.
  static constexpr int RW = P >= 32 ? 1 : imin(4, 32 / P);
  static constexpr int SYNC = (THREADS <= 32 || P > 32) ? kSyncCta : kSyncWarp;
  static constexpr int SMEM = (M * L + L) * 2 * int(sizeof(T));
  static constexpr bool OK = NR >= 16 && THREADS <= 1024 && M % THREADS == 0;
};

// 2x2 Hadamard on registers: x[l], l = 2a + b, -> y[q], q = 2 ci + cj,
// y = sum (-1)^{a ci + b cj} x.
template <typename V>
__device__ __forceinline__ void quad_hadamard(V (&x)[4]) {
  const V s0 = cadd(x[0], x[1]), d0 = csub(x[0], x[1]);  // along b, a = 0
  const V s1 = cadd(x[2], x[3]), d1 = csub(x[2], x[3]);  // along b, a = 1
  x[0] = cadd(s0, s1);
  x[2] = csub(s0, s1);
  x[1] = cadd(d0, d1);
  x[3] = csub(d0, d1);
}

// K1 (quad): r2c of the quad's four rows (the FFT as zfwd_rows), then, with the
// four rows' spectra staged row-major in shared memory, every thread takes
// whole columns k: the Hermitian split of all four rows, the 2x2 step of the
// i / j transforms and its twiddle, stores into the four chunks.
template <typename T, int NR>
__global__ void __launch_bounds__(QuadZCfg<T, NR>::THREADS, 2)
    k_zfwd_quad(const T* __restrict__ f, vec2_t<T>* __restrict__ S, const vec2_t<T>* __restrict__ tw,
                const vec2_t<T>* __restrict__ stw, Layout gq) {
  using V = vec2_t<T>;
  using C = QuadZCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, H = C::H, TH = C::THREADS, RW = C::RW;
  constexpr int ncp = spec_pitch(NR);
  V* sm = smem_base<V>();
  const int grp = threadIdx.x / (RW * P), gi = threadIdx.x % (RW * P);
  const int l = grp * RW + gi % RW, t = gi / RW;  // row of the quad, position thread
  V* gsm = sm + grp * RW * M;                      // the group's rows
  const int ip = blockIdx.x / H, jp = blockIdx.x % H;
  auto frow = [&](int r) { return size_t(ip + (r >> 1) * H) * NR + (jp + (r & 1) * H); };
  if constexpr (ARENA_Z_PF > 0) {  // the quad one resident wave ahead, into L2
    const unsigned b = blockIdx.x + ARENA_Z_PF * ARENA_SMS * 2;
    if (threadIdx.x < 4 && b < gridDim.x) {
      const int r = threadIdx.x, ib = b / H, jb = b % H;
      bulk_prefetch_l2(f + (size_t(ib + (r >> 1) * H) * NR + (jb + (r & 1) * H)) * NR, NR * sizeof(T));
    }
  }
  const V* src = reinterpret_cast<const V*>(f + frow(l) * NR);
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  line_fft<M, E, RW, -1, C::SYNC>(v, gsm, stw, t, gi % RW);  // ends with the group's scratch free
#pragma unroll
  for (int e = 0; e < E; ++e) sm[l * M + t + P * e] = v[e];  // row-major: columns read conflict-free
  __syncthreads();
  V wq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) wq[q] = tw_load(tw, (q >> 1) * ip + (q & 1) * jp);  // W_n^{ci i' + cj j'} (< n)
  V* dst[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) dst[q] = S + lrow(gq, q, ip, jp) * ncp;
  constexpr int NM = M / TH;
  if constexpr (ARENA_Z_PAIRS && NM >= 2 && NM % 2 == 0) {
    // columns in Hermitian pairs (k, M - k), as zfwd_rows: S = (A + B)/2, U = (i/2) W_n^k (A - B),
    // X[k] = S - U, X[M-k] = conj(S + U); column 0 pairs with the Nyquist column M
#pragma unroll
    for (int m = 0; m < NM / 2; ++m) {
      const int k = threadIdx.x + TH * m;
      const V Wt = tw_load(tw, k);
      const V Wh{T(-0.5) * Wt.y, T(0.5) * Wt.x};  // (i/2) W_n^k
      V x[4], xr[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const V A = sm[r * M + k];
        const V Bc = sm[r * M + ((M - k) & (M - 1))];
        const V B{Bc.x, -Bc.y};
        const V U = cmul(Wh, csub(A, B));
        const V Sm = cadd(A, B);
        x[r] = V{fma(T(0.5), Sm.x, -U.x), fma(T(0.5), Sm.y, -U.y)};
        xr[r] = V{fma(T(0.5), Sm.x, U.x), -fma(T(0.5), Sm.y, U.y)};
        if (k == 0) xr[r].y = T(0);
      }
      quad_hadamard(x);
      quad_hadamard(xr);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        st_out(dst[q] + k, cmul(x[q], wq[q]));
        st_out(dst[q] + (M - k), cmul(xr[q], wq[q]));
      }
    }
    if (threadIdx.x == 0) {  // X[M/2] = conj(Z[M/2]) of each row
      V x[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const V z = sm[r * M + M / 2];
        x[r] = V{z.x, -z.y};
      }
      quad_hadamard(x);
#pragma unroll
      for (int q = 0; q < 4; ++q) st_out(dst[q] + M / 2, cmul(x[q], wq[q]));
    }
  } else {
#pragma unroll
  for (int m = 0; m < M / TH; ++m) {
    const int k = threadIdx.x + TH * m;
    const V W = tw_load(tw, k);  // W_n^k
    V x[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const V A = sm[r * M + k];
      const V Bc = sm[r * M + ((M - k) & (M - 1))];
      const V B{Bc.x, -Bc.y};
      const V WD = cmul(W, csub(A, B));
      x[r] = V{T(0.5) * (A.x + B.x + WD.y), T(0.5) * (A.y + B.y - WD.x)};
    }
    quad_hadamard(x);
#pragma unroll
    for (int q = 0; q < 4; ++q) st_out(dst[q] + k, cmul(x[q], wq[q]));
  }
  if (threadIdx.x == 0) {  // X[M] = Re Z0 - Im Z0 of each row
    V x[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const V z = sm[r * M];
      x[r] = V{z.x - z.y, T(0)};
    }
    quad_hadamard(x);
#pragma unroll
    for (int q = 0; q < 4; ++q) st_out(dst[q] + M, cmul(x[q], wq[q]));
  }
  }
}

// K5 (quad): every thread takes whole columns k of the quad's four chunk rows —
// the conjugate twiddle and the inverse 2x2 step — into shared memory row-major;
// then each row's Hermitian split and c2r as zinv_rows.
template <typename T, int NR>
__global__ void __launch_bounds__(QuadZCfg<T, NR>::THREADS, 2)
    k_zinv_quad(const vec2_t<T>* __restrict__ S, T* __restrict__ u, const vec2_t<T>* __restrict__ tw,
                const vec2_t<T>* __restrict__ stw, Layout gq) {
  using V = vec2_t<T>;
  using C = QuadZCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L, H = C::H, TH = C::THREADS, RW = C::RW;
  constexpr int ncp = spec_pitch(NR);
  V* sm = smem_base<V>();
  V* xm = sm + M * L;
  const int grp = threadIdx.x / (RW * P), gi = threadIdx.x % (RW * P);
  const int l = grp * RW + gi % RW, t = gi / RW;
  V* gsm = sm + grp * RW * M;
  const int ip = blockIdx.x / H, jp = blockIdx.x % H;
  if constexpr (ARENA_Z_PF > 0) {
    const unsigned b = blockIdx.x + ARENA_Z_PF * ARENA_SMS * 2;
    if (threadIdx.x < 4 && b < gridDim.x)
      bulk_prefetch_l2(S + lrow(gq, threadIdx.x, b / H, b % H) * ncp, ncp * sizeof(V));
  }
  const V* src[4];
  V wq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    src[q] = S + lrow(gq, q, ip, jp) * ncp;
    wq[q] = tw_load(tw, (q >> 1) * ip + (q & 1) * jp);
  }
  // all column loads first (E per thread, as zinv_rows keeps E loads in flight)
  constexpr int NM = M / TH;
  V y[NM][4];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q) y[m][q] = __ldcs(src[q] + threadIdx.x + TH * m);
  V ym[4];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) ym[q] = __ldcs(src[q] + M);
  }
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int k = threadIdx.x + TH * m;
#pragma unroll
    for (int q = 0; q < 4; ++q) y[m][q] = cmulc(y[m][q], wq[q]);
    quad_hadamard(y[m]);
#pragma unroll
    for (int r = 0; r < 4; ++r) sm[r * M + k] = y[m][r];
  }
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) ym[q] = cmulc(ym[q], wq[q]);
    quad_hadamard(ym);
#pragma unroll
    for (int r = 0; r < 4; ++r) xm[r] = ym[r];
  }
  __syncthreads();
  V v[E];
  if constexpr (ARENA_Z_PAIRS && E >= 2 && E % 2 == 0) {
    // Hermitian pairs (k, M - k) as zinv_rows: Ep = A + B, Op = i conj(W_n^k) (A - B),
    // Z[k] = Ep + Op stays in the thread, Z[M-k] = conj(Ep - Op) goes back to its slot
    // (only this thread reads X[k] / X[M-k]) for its owner to pick up
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int k = t + P * e;
      V A = sm[l * M + k];
      V C = (k == 0) ? xm[l] : sm[l * M + M - k];
      if (k == 0) {
        A.y = T(0);
        C.y = T(0);
      }
      const V B{C.x, -C.y};
      const V W = tw_load(tw, k);
      const V Wi{W.y, W.x};  // i conj(W_n^k)
      const V Ep = cadd(A, B);
      const V Op = cmul(csub(A, B), Wi);
      v[e] = cadd(Ep, Op);
      if (k != 0) sm[l * M + M - k] = V{Ep.x - Op.x, Op.y - Ep.y};
    }
    if (t == 0) {
      const V h = sm[l * M + M / 2];
      sm[l * M + M / 2] = V{T(2) * h.x, T(-2) * h.y};
    }
    xbarrier<C::SYNC>();
#pragma unroll
    for (int e = E / 2; e < E; ++e) v[e] = sm[l * M + t + P * e];
  } else {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int k = t + P * e;
    V A = sm[l * M + k];
    V Bs = (k == 0) ? xm[l] : sm[l * M + M - k];
    if (k == 0) {
      A.y = T(0);
      Bs.y = T(0);
    }
    const V B{Bs.x, -Bs.y};
    const V W = tw_load(tw, k);
    const V Ep = cadd(A, B);
    const V Op = cmulc(csub(A, B), W);
    v[e] = V{Ep.x - Op.y, Ep.y + Op.x};
  }
  }
  xbarrier<C::SYNC>();  // the group's split reads done: its rows become FFT scratch
  line_fft<M, E, RW, +1, C::SYNC>(v, gsm, stw, t, gi % RW);
  const size_t row = size_t(ip + (l >> 1) * H) * NR + (jp + (l & 1) * H);
  V* dst = reinterpret_cast<V*>(u + row * NR);
#pragma unroll
  for (int e = 0; e < E; ++e) st_out(dst + t + P * e, v[e]);
}

}  // namespace arena_fft
