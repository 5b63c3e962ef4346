// pattern_bw.cu — microbenchmark: HBM bandwidth of the spectral passes' access
// patterns with no FFT work, and the fp64 FMA issue rate.  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pattern_bw tools/pattern_bw.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

// In-place read+write of lines along a strided axis, tile of L adjacent k,
// thread (l, t) touching rows t + P*e (E per thread) — the k_ypass/k_xmid pattern.
template <int N, int E, int L>
__global__ void __launch_bounds__(L * N / E) strided_rw(double2* __restrict__ a, long long row_stride, long long tile_stride_y,
                                                        int ncp, int nc) {
  constexpr int P = N / E;
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int k = blockIdx.x * L + l;
  if (k >= nc) return;
  double2* base = a + (long long)blockIdx.y * tile_stride_y + k;
  double2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) v[e] = __ldcs(base + (long long)(t + P * e) * row_stride);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    v[e].x *= 1.0000001;
    v[e].y *= 0.9999999;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) __stcs(base + (long long)(t + P * e) * row_stride, v[e]);
}

// Two-level addressing: tile base(y) = (y / By) * oy + (y % By) * iy,
// row r at (r / Br) * orr + (r % Br) * ir (elements).
template <int N, int E, int L>
__global__ void __launch_bounds__(L * N / E) strided2_rw(double2* __restrict__ a, int By, long long oy, long long iy,
                                                         int Br, long long orr, long long ir, int nc) {
  constexpr int P = N / E;
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const int k = blockIdx.x * L + l;
  if (k >= nc) return;
  const int y = blockIdx.y;
  double2* base = a + (long long)(y / By) * oy + (long long)(y % By) * iy + k;
  double2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int r = t + P * e;
    v[e] = __ldcs(base + (long long)(r / Br) * orr + (long long)(r % Br) * ir);
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    v[e].x *= 1.0000001;
    v[e].y *= 0.9999999;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int r = t + P * e;
    __stcs(base + (long long)(r / Br) * orr + (long long)(r % Br) * ir, v[e]);
  }
}

// Blocked spectrum layout S[jb][i][jin][k], jb = j / B.
template <int L, int E>
void run_blocked(double2* a, int n, int ncp, int nc, double bytes, int B) {
  constexpr int N = 1024;
  const int H = 1 << 30;
  dim3 grid((nc + L - 1) / L, n);
  const long long nB = (long long)n * B * ncp;
  float ty = time_ms([&] { strided2_rw<N, E, L><<<grid, L * N / E>>>(a, H, 0, (long long)B * ncp, B, nB, ncp, nc); });
  float tx = time_ms([&] { strided2_rw<N, E, L><<<grid, L * N / E>>>(a, B, nB, ncp, H, 0, (long long)B * ncp, nc); });
  printf("blocked B=%3d L=%d E=%d  y %7.1f GB/s   x %7.1f GB/s\n", B, L, E, bytes / ty / 1e6, bytes / tx / 1e6);
}

// k-tiled layout S[kt][i][j][8 k] (the k axis split in 128-byte tiles, outermost):
// a y tile (kt, i) is one contiguous 128 KB block, an x tile (kt, j) reads 128 B
// at a 128 KB stride; blockIdx.x = the line (fastest), blockIdx.y = kt.
template <int N, int E, int L, bool XPAT>
__global__ void __launch_bounds__(L * N / E) ktiled_rw(double2* __restrict__ a) {
  constexpr int P = N / E;
  const int l = threadIdx.x % L, t = threadIdx.x / L;
  const long long kt = blockIdx.y, line = blockIdx.x;
  double2* base = a + kt * (long long)N * N * L + l;
  double2 v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long r = t + P * e;
    v[e] = __ldcs(base + (XPAT ? (r * N + line) : (line * N + r)) * L);
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    v[e].x *= 1.0000001;
    v[e].y *= 0.9999999;
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const long long r = t + P * e;
    __stcs(base + (XPAT ? (r * N + line) : (line * N + r)) * L, v[e]);
  }
}

__global__ void copy_rw(double2* __restrict__ a, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double2 v = __ldcs(a + i);
    v.x *= 1.0000001;
    __stcs(a + i, v);
  }
}

__global__ void dfma_rate(double* out, int iters) {
  double a0 = threadIdx.x * 1e-9, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

template <typename F>
float time_ms(F f, int reps = 5) {
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(s);
  for (int r = 0; r < reps; ++r) f();
  cudaEventRecord(e);
  CK(cudaEventSynchronize(e));
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  return ms / reps;
}

template <int L, int E>
void run_strided(double2* a, int n, int ncp, int nc, double bytes) {
  constexpr int N = 1024;
  dim3 grid((nc + L - 1) / L, n);
  // y pattern: row stride ncp, tile stride (per i) n*ncp
  float ty = time_ms([&] { strided_rw<N, E, L><<<grid, L * N / E>>>(a, ncp, (long long)n * ncp, ncp, nc); });
  // x pattern: row stride n*ncp, tile stride (per j) ncp
  float tx = time_ms([&] { strided_rw<N, E, L><<<grid, L * N / E>>>(a, (long long)n * ncp, ncp, ncp, nc); });
  printf("L=%2d E=%2d  y-pattern %7.1f GB/s   x-pattern %7.1f GB/s\n", L, E, bytes / ty / 1e6, bytes / tx / 1e6);
}

int main() {
  const int n = 1024, nc = n / 2 + 1, ncp = 520;
  const long long elems = (long long)n * n * ncp;
  double2* a;
  CK(cudaMalloc(&a, elems * sizeof(double2)));
  CK(cudaMemset(a, 0, elems * sizeof(double2)));
  const double bytes = 2.0 * n * n * (double)nc * sizeof(double2);
  float tc = time_ms([&] { copy_rw<<<148 * 8, 256>>>(a, elems); });
  printf("contiguous rw          %7.1f GB/s\n", 2.0 * elems * sizeof(double2) / tc / 1e6);
  run_strided<1, 16>(a, n, ncp, nc, bytes);
  run_strided<2, 16>(a, n, ncp, nc, bytes);
  run_strided<4, 16>(a, n, ncp, nc, bytes);
  run_strided<8, 16>(a, n, ncp, nc, bytes);
  run_strided<4, 8>(a, n, ncp, nc, bytes);
  run_strided<8, 8>(a, n, ncp, nc, bytes);
  run_strided<16, 16>(a, n, ncp, nc, bytes);
  {
    dim3 grid(n, ncp / 8);
    float ty = time_ms([&] { ktiled_rw<1024, 16, 8, false><<<grid, 8 * 1024 / 16>>>(a); });
    float tx = time_ms([&] { ktiled_rw<1024, 16, 8, true><<<grid, 8 * 1024 / 16>>>(a); });
    printf("k-tiled L=8 E=16  y %7.1f GB/s   x %7.1f GB/s\n", bytes / ty / 1e6, bytes / tx / 1e6);
  }
  for (int B : {1, 2, 4, 8, 16, 32, 64, 128}) {
    run_blocked<4, 16>(a, n, ncp, nc, bytes, B);
    run_blocked<8, 16>(a, n, ncp, nc, bytes, B);
  }
  double* out;
  CK(cudaMalloc(&out, 148 * 8 * 256 * sizeof(double)));
  const int iters = 4096;
  float tf = time_ms([&] { dfma_rate<<<148 * 8, 256>>>(out, iters); });
  const double fmas = 148.0 * 8 * 256 * iters * 8;
  printf("DFMA rate %.2f TFMA/s = %.1f lanes/clk/SM at 1.965 GHz\n", fmas / tf / 1e9, fmas / (tf / 1e3) / 148 / 1.965e9);
  return 0;
}
