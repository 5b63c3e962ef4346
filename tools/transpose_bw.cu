// transpose_bw.cu — microbenchmark: contiguous-line reads + 128-byte-segment
// transposed writes (the pattern of a transpose-fused FFT pass).  Not product code.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                       \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) {                                                                        \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);              \
      exit(1);                                                                                      \
    }                                                                                               \
  } while (0)

// Source: lines of N complex, line index (a, b, c) -> ((a*B + b)*C + c)*N (contiguous lines).
// A CTA of W warps takes W lines with consecutive c (c0..c0+W-1) at fixed (a, b), and writes
// element e of line w to dst[(a, e, b, c0+w)] with dst index ((a*N + e)*B + b)*C + c  (i.e. the
// line axis moves to the middle and c becomes the contiguous axis: segments of W*16 bytes).
template <int N, int W>
__global__ void __launch_bounds__(32 * W) tcopy(const double2* __restrict__ src, double2* __restrict__ dst, int A,
                                                 int B, int C, long long sa, long long sb, long long sc, long long de,
                                                 long long db, long long dc, long long da) {
  extern __shared__ double2 sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int ct = C / W;
  long long blk = blockIdx.x;
  const int c0 = int(blk % ct) * W;
  blk /= ct;
  const int b = int(blk % B), a = int(blk / B);
  const double2* s = src + a * sa + b * sb + (c0 + warp) * sc;
  double2 v[N / 32];
#pragma unroll
  for (int e = 0; e < N / 32; ++e) v[e] = __ldcs(s + lane + 32 * e);
#pragma unroll
  for (int e = 0; e < N / 32; ++e) { const int r = lane + 32 * e; sm[r * W + (warp ^ (r & (W - 1)))] = v[e]; }
  __syncthreads();
  double2* d = dst + a * da + b * db + c0 * dc;
  // each warp writes rows e = warp, warp + W, ... ; lane covers (e_sub, w) pairs
  constexpr int PER = 32 / W;  // rows per warp instruction
  for (int e0 = warp * PER; e0 < N; e0 += W * PER) {
    const int e = e0 + lane / W, w = lane % W;
    __stcs(d + e * de + w * dc, sm[e * W + (w ^ (e & (W - 1)))]);
  }
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

int main() {
  const int n = 1024, nc = 520;  // nc padded to a multiple of 8
  const long long elems = (long long)n * n * n;
  double2 *a, *b;
  CK(cudaMalloc(&a, elems * sizeof(double2)));
  CK(cudaMalloc(&b, elems * sizeof(double2)));
  CK(cudaMemset(a, 0, elems * sizeof(double2)));
  const double bytes = 2.0 * elems * sizeof(double2);
  constexpr int W = 8;
  const int smem = 1024 * W * 16;
  CK(cudaFuncSetAttribute(tcopy<1024, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  // y->x like transition: src lines [i][k][j] (line = (i,k)); CTA: 8 consecutive i at fixed k ->
  // dst [k][j][i]: a = k? Use generic: (a,b,c) = (0, k, i), src index ((0*nc + k)... emulate strides:
  //   src line (i, k): offset (i*nc + k)*n  => a=0, b=k (B=nc), c=i (C=n): sb = n, sc = nc*n
  //   dst (k, j, i) : offset (k*n + j)*n + i => db = n*n, de = n, dc = 1
  {
    long long nb = (long long)nc * (n / W);
    float t = time_ms([&] {
      tcopy<1024, W><<<nb, 32 * W, smem>>>(a, b, 1, nc, n, 0, n, (long long)nc * n, n, (long long)n * n, 1, 0);
    });
    printf("y->x transpose  [i][k][j] -> [k][j][i]   %7.1f GB/s\n", bytes / t / 1e6);
  }
  //   z->y: src rows (i, j) over k (length n complex here for the test), dst [i][k][j]
  //   line (i, j): a = i, c = j: sa = n*n, sc = n ; dst (i, k, j): da = nc*n... use k<n rows
  {
    long long nb = (long long)n * (n / W);
    float t = time_ms([&] {
      tcopy<1024, W><<<nb, 32 * W, smem>>>(a, b, n, 1, n, (long long)n * n, 0, n, n, 0, 1, (long long)n * n);
    });
    printf("z->y transpose  [i][j][k] -> [i][k][j]   %7.1f GB/s (rows of n)\n", 2.0 * n * n * n * 16 / t / 1e6);
  }
  //   x->y (i-blocked by 8): src lines (k, j) over i: [k][j][i]; dst [ib][k][ii][j] ; CTA: 8 j at fixed k
  //   src line (k, j): sb = n*n (b = k), sc = n (c = j). dst element e = i: (i/8)*(nc*8*n) + (i%8)*n  -> not affine;
  //   emulate with de = 8*n (worst case i-stride inside a block) for the page pattern estimate.
  {
    long long nb = (long long)nc * (n / W);
    float t = time_ms([&] {
      tcopy<1024, W><<<nb, 32 * W, smem>>>(a, b, 1, nc, n, 0, (long long)n * n, n, (long long)8 * n, (long long)8 * n * n / 8, 1, 0);
    });
    printf("x->y (approx)   [k][j][i] -> [.][k][.][j] %7.1f GB/s\n", bytes / t / 1e6);
  }
  {
    long long nb = (long long)nc * (n / W);
    float t = time_ms([&] {
      tcopy<1024, W><<<nb, 32 * W, smem>>>(a, b, 1, nc, n, 0, (long long)n * n, n, (long long)nc * n, n, 1, 0);
    });
    printf("x->y unblocked  [k][j][i] -> [i][k][j]   %7.1f GB/s\n", bytes / t / 1e6);
  }
  return 0;
}
