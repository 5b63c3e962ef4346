// poisson_qpencil.cuh — z passes of the FOLDED pencil decomposition (config 5:
// 2048^3 at 2 x 2 / 2 x 4 ranks; PAPER.md:69-71,79-81 for the pencil scheme).
//
// The plain pencil runs n-point y / x lines per rank; at n = 2048 an 8-line fp64
// tile (128-byte TMA rows) is 256 KB, more than an SM's shared memory, so those
// passes fall back to 64- / 32-byte rows (55-65% of the 1024^3 passes' bandwidth,
// DESIGN §4.1).  The single-GPU quadrant formulation (poisson_quad.cuh) avoids it
// by moving the first radix-2 step of the i and j transforms into the z passes;
// it needs the four rows (i', j'), (i'+H, j'), (i', j'+H), (i'+H, j'+H) (H = n/2)
// in one CTA.  The FOLDED distribution makes that local: rank (r, c) owns
//   i in I_r U (I_r + H),  j in J_c U (J_c + H),   I_r = [r H/Pr, (r+1) H/Pr), J_c likewise,
// as a (2 ni) x (2 nj) x n block (ni = H/Pr, nj = H/Pc; local i il < ni is i = r ni + il,
// il >= ni is i = H + r ni + il - ni; j alike).  After K1q every quadrant
// q = 2 ci + cj is an H x H problem (full k range of the n grid) distributed as an
// ordinary pencil — rank (r, c) owns its I_r x J_c block — so the exchanges and
// the strided passes are the plain pencil's, on H-point lines with 128-byte rows,
// once per quadrant; the symbol reads ki = 2 i'' + ci, kj = 2 j'' + cj (KSpan fm).
//
// Buffer R (K1q output) holds the four quadrants one after another, each exactly
// the plain pencil's R of the H problem: Pc k-chunks of ni x nj rows (Layout
// (ni, nj)) of kq complex.
#pragma once

#include "poisson_quad.cuh"

namespace arena_fft {

// K1q (folded pencil): r2c of the quad's four rows of the rank's block, the 2x2
// step with the GLOBAL twiddle W_n^{ci i' + cj j'}, k-split stores into quadrant q's R.
// PEER: k-chunk c of quadrant q goes straight to row peer c's Y buffer (po.base[c], advanced
// to this rank's chunk) at quadrant offset q qstride — the row all-to-all fused into K1q.
template <typename T, int NR, bool PEER = false>
__global__ void __launch_bounds__(QuadZCfg<T, NR>::THREADS, 2)
    k_zfwd_qpencil(const T* __restrict__ f, vec2_t<T>* __restrict__ R, const vec2_t<T>* __restrict__ tw,
                   const vec2_t<T>* __restrict__ stw, Layout gz, int i0, int j0, int kq, size_t qstride,
                   const __grid_constant__ PeerOut<vec2_t<T>> po) {
  using V = vec2_t<T>;
  using C = QuadZCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, TH = C::THREADS, RW = C::RW;
  V* sm = smem_base<V>();
  const int ni = gz.ni, nj = gz.nj;
  const int grp = threadIdx.x / (RW * P), gi = threadIdx.x % (RW * P);
  const int l = grp * RW + gi % RW, t = gi / RW;  // row of the quad, position thread
  V* gsm = sm + grp * RW * M;
  const int il = blockIdx.x / nj, jl = blockIdx.x % nj;
  // local rows of the block (2 ni) x (2 nj): quad member l = 2a + b at (il + a ni, jl + b nj)
  auto frow = [&](int r) { return size_t(il + (r >> 1) * ni) * (2 * nj) + (jl + (r & 1) * nj); };
  const V* src = reinterpret_cast<const V*>(f + frow(l) * NR);
  V v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(src + t + P * e);
  line_fft<M, E, RW, -1, C::SYNC>(v, gsm, stw, t, gi % RW);
#pragma unroll
  for (int e = 0; e < E; ++e) sm[l * M + t + P * e] = v[e];
  __syncthreads();
  const int ig = i0 + il, jg = j0 + jl;  // global i', j' in [0, H)
  V wq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) wq[q] = tw_load(tw, (q >> 1) * ig + (q & 1) * jg);  // W_n^{ci i' + cj j'}
  const size_t rin = lrow(gz, 0, il, jl);
  const size_t chunk = size_t(ni) * nj;
  auto put = [&](int q, int k, V x) {
    const int c = k / kq;
    if constexpr (PEER) {
      po.base[c][q * qstride + rin * kq + (k - c * kq)] = x;
    } else {
      st_out(R + q * qstride + (size_t(c) * chunk + rin) * kq + (k - c * kq), x);
    }
  };
  constexpr int NM = M / TH;
  if constexpr (ARENA_Z_PAIRS && NM >= 2 && NM % 2 == 0) {
    // columns in Hermitian pairs (k, M - k), as k_zfwd_quad; column 0 pairs with the Nyquist column M
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
        put(q, k, cmul(x[q], wq[q]));
        put(q, M - k, cmul(xr[q], wq[q]));
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
      for (int q = 0; q < 4; ++q) put(q, M / 2, cmul(x[q], wq[q]));
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
      for (int q = 0; q < 4; ++q) put(q, k, cmul(x[q], wq[q]));
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
      for (int q = 0; q < 4; ++q) put(q, M, cmul(x[q], wq[q]));
    }
  }
  if constexpr (PEER) __threadfence_system();  // peer stores performed before the ranks' barrier
}

// K5q (folded pencil): gather the four quadrants' k-chunked rows, the conjugate
// twiddle and the inverse 2x2 step, then each row's Hermitian split and c2r.
template <typename T, int NR>
__global__ void __launch_bounds__(QuadZCfg<T, NR>::THREADS, 2)
    k_zinv_qpencil(const vec2_t<T>* __restrict__ R, T* __restrict__ u, const vec2_t<T>* __restrict__ tw,
                   const vec2_t<T>* __restrict__ stw, Layout gz, int i0, int j0, int kq, size_t qstride) {
  using V = vec2_t<T>;
  using C = QuadZCfg<T, NR>;
  constexpr int M = C::M, E = C::E, P = C::P, L = C::L, TH = C::THREADS, RW = C::RW;
  V* sm = smem_base<V>();
  V* xm = sm + M * L;
  const int ni = gz.ni, nj = gz.nj;
  const int grp = threadIdx.x / (RW * P), gi = threadIdx.x % (RW * P);
  const int l = grp * RW + gi % RW, t = gi / RW;
  V* gsm = sm + grp * RW * M;
  const int il = blockIdx.x / nj, jl = blockIdx.x % nj;
  const int ig = i0 + il, jg = j0 + jl;
  const size_t rin = lrow(gz, 0, il, jl);
  const size_t chunk = size_t(ni) * nj;
  auto get = [&](int q, int k) {
    const int c = k / kq;
    return __ldcs(R + q * qstride + (size_t(c) * chunk + rin) * kq + (k - c * kq));
  };
  V wq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) wq[q] = tw_load(tw, (q >> 1) * ig + (q & 1) * jg);
  constexpr int NM = M / TH;
  V y[NM][4];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int q = 0; q < 4; ++q) y[m][q] = get(q, threadIdx.x + TH * m);
  V ym[4];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) ym[q] = get(q, M);
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
  if constexpr (ARENA_Z_PAIRS && E >= 2 && E % 2 == 0) {  // Hermitian pairs, as k_zinv_quad
#pragma unroll
    for (int e = 0; e < E / 2; ++e) {
      const int k = t + P * e;
      V A = sm[l * M + k];
      V C = (k == 0) ? xm[l] : sm[l * M + M - k];
      if (k == 0) {  // FFTW c2r: imaginary parts of X[0] and X[M] ignored
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
  }
  xbarrier<C::SYNC>();
  line_fft<M, E, RW, +1, C::SYNC>(v, gsm, stw, t, gi % RW);
  const size_t row = size_t(il + (l >> 1) * ni) * (2 * nj) + (jl + (l & 1) * nj);
  V* dst = reinterpret_cast<V*>(u + row * NR);
#pragma unroll
  for (int e = 0; e < E; ++e) st_out(dst + t + P * e, v[e]);
}

}  // namespace arena_fft
