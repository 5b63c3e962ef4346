// verify.cu — device-side verification reductions:
// GridField::mean / max_abs (grid.cpp:9-19) and the gauge-aligned error of
// linf_rel_error (problems.cpp:88-106), over n^3-point device fields, so that
// 1024^3 and 2048^3 results are checked without copying 8.6-69 GB to the host.
//
// Sums are accumulated per thread with Neumaier compensation in fp64, combined
// per block in fp64 (warp shuffles), and the per-block partials are added on
// the host in long double: the mean of 2^30 values keeps ~1e-16 relative error.
// Fields are `count` contiguous values (n^3 for a GridField, a rank's block for
// a decomposed one).
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "../../include/arena_fft.h"

namespace arena_fft {
arena_status set_error(arena_status s, const std::string& msg);
}

namespace {

constexpr int kThreads = 256;

struct Neu {  // Neumaier-compensated sum
  double s = 0.0, c = 0.0;
  __device__ void add(double x) {
    const double t = s + x;
    c += fabs(s) >= fabs(x) ? (s - t) + x : (x - t) + s;
    s = t;
  }
  __device__ double value() const { return s + c; }
};

template <typename T>
__device__ __forceinline__ double ld(const T* p, size_t i) {
  return double(__ldcs(p + i));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block reduction of NS sums and NM maxima; thread 0 writes them to out[blockIdx.x * (NS + NM) + ...].
template <int NS, int NM>
__device__ void block_out(const double (&sums)[NS], const double (&maxs)[NM], double* out) {
  __shared__ double red[kThreads / 32][NS + NM];
  const int w = threadIdx.x / 32, lane = threadIdx.x % 32;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    const double v = warp_sum(sums[q]);
    if (lane == 0) red[w][q] = v;
  }
#pragma unroll
  for (int q = 0; q < NM; ++q) {
    const double v = warp_max(maxs[q]);
    if (lane == 0) red[w][NS + q] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < NS + NM; ++q) {
      double a = q < NS ? 0.0 : red[0][q];
      for (int k = 0; k < kThreads / 32; ++k) a = q < NS ? a + red[k][q] : fmax(a, red[k][q]);
      out[size_t(blockIdx.x) * (NS + NM) + q] = a;
    }
  }
}

// Pass 1: sum(num), sum(exact), max|num|, max|exact| (exact may be null).
template <typename T>
__global__ void __launch_bounds__(kThreads) k_stats(const T* __restrict__ num, const T* __restrict__ ex, size_t count,
                                                    double* out) {
  Neu sn, se;
  double mn = 0.0, me = 0.0;
  for (size_t i = size_t(blockIdx.x) * kThreads + threadIdx.x; i < count; i += size_t(gridDim.x) * kThreads) {
    const double a = ld(num, i);
    sn.add(a);
    mn = fmax(mn, fabs(a));
    if (ex) {
      const double b = ld(ex, i);
      se.add(b);
      me = fmax(me, fabs(b));
    }
  }
  const double sums[2] = {sn.value(), se.value()};
  const double maxs[2] = {mn, me};
  block_out<2, 2>(sums, maxs, out);
}

// Pass 2: sum (num + shift - exact)^2, sum (exact - mean_e)^2, max |num + shift - exact|.
template <typename T>
__global__ void __launch_bounds__(kThreads) k_err(const T* __restrict__ num, const T* __restrict__ ex, size_t count,
                                                  double shift, double mean_e, double* out) {
  Neu sd, se;
  double md = 0.0;
  for (size_t i = size_t(blockIdx.x) * kThreads + threadIdx.x; i < count; i += size_t(gridDim.x) * kThreads) {
    const double b = ld(ex, i);
    const double d = ld(num, i) + shift - b;
    const double c = b - mean_e;
    sd.add(d * d);
    se.add(c * c);
    md = fmax(md, fabs(d));
  }
  const double sums[2] = {sd.value(), se.value()};
  const double maxs[1] = {md};
  block_out<2, 1>(sums, maxs, out);
}

int grid_blocks() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms * 8;
}

// Run a reduction kernel and fold the per-block partials (NS sums, NM maxima) on the host.
template <typename Launch>
arena_status reduce(int nout_s, int nout_m, Launch&& launch, std::vector<long double>& sums, std::vector<double>& maxs) {
  const int blocks = grid_blocks();
  const int w = nout_s + nout_m;
  double* d = nullptr;
  cudaError_t e = cudaDeviceSynchronize();  // the fields may come from any stream
  if (e != cudaSuccess) return arena_fft::set_error(ARENA_ECUDA, std::string("verify: ") + cudaGetErrorString(e));
  e = cudaMalloc(&d, sizeof(double) * size_t(blocks) * w);
  if (e != cudaSuccess) return arena_fft::set_error(ARENA_ENOMEM, "verify partials");
  launch(blocks, d);
  e = cudaGetLastError();
  std::vector<double> h(size_t(blocks) * w);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), d, h.size() * sizeof(double), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (e != cudaSuccess) return arena_fft::set_error(ARENA_ECUDA, std::string("verify: ") + cudaGetErrorString(e));
  sums.assign(nout_s, 0.0L);
  maxs.assign(nout_m, 0.0);
  for (int b = 0; b < blocks; ++b) {
    for (int q = 0; q < nout_s; ++q) sums[q] += h[size_t(b) * w + q];
    for (int q = 0; q < nout_m; ++q) maxs[q] = std::fmax(maxs[q], h[size_t(b) * w + nout_s + q]);
  }
  return ARENA_OK;
}

template <typename T>
arena_status stats_t(size_t count, const void* f, double* mean, double* max_abs) {
  std::vector<long double> s;
  std::vector<double> m;
  arena_status st = reduce(
      2, 2,
      [&](int blocks, double* out) {
        k_stats<T><<<blocks, kThreads>>>(static_cast<const T*>(f), nullptr, count, out);
      },
      s, m);
  if (st != ARENA_OK) return st;
  if (mean) *mean = double(s[0] / (long double)count);
  if (max_abs) *max_abs = m[0];
  return ARENA_OK;
}

template <typename T>
arena_status compare_t(size_t count, const void* num, const void* ex, double* rel_l2, double* linf_rel,
                       double* gauge_shift) {
  std::vector<long double> s;
  std::vector<double> m;
  const T* a = static_cast<const T*>(num);
  const T* b = static_cast<const T*>(ex);
  arena_status st = reduce(2, 2, [&](int blocks, double* out) { k_stats<T><<<blocks, kThreads>>>(a, b, count, out); }, s, m);
  if (st != ARENA_OK) return st;
  const double ex_max = m[1];
  if (ex_max == 0.0) return arena_fft::set_error(ARENA_EINVAL, "exact solution vanishes on the grid");
  // problems.cpp:102 — shift aligns the means (periodic gauge)
  const double shift = double((s[1] - s[0]) / (long double)count);
  const double mean_e = double(s[1] / (long double)count);
  std::vector<long double> s2;
  std::vector<double> m2;
  st = reduce(
      2, 1, [&](int blocks, double* out) { k_err<T><<<blocks, kThreads>>>(a, b, count, shift, mean_e, out); }, s2, m2);
  if (st != ARENA_OK) return st;
  if (gauge_shift) *gauge_shift = shift;
  if (linf_rel) *linf_rel = m2[0] / ex_max;
  if (rel_l2) *rel_l2 = s2[1] > 0 ? double(std::sqrt(s2[0] / s2[1])) : double(std::sqrt(s2[0]));
  return ARENA_OK;
}

}  // namespace

extern "C" {

arena_status arena_field_stats(size_t count, int precision_bits, const void* d_field, double* mean, double* max_abs) {
  if (count < 1 || !d_field) return arena_fft::set_error(ARENA_EINVAL, "bad field");
  if (precision_bits == 64) return stats_t<double>(count, d_field, mean, max_abs);
  if (precision_bits == 32) return stats_t<float>(count, d_field, mean, max_abs);
  return arena_fft::set_error(ARENA_EINVAL, "precision_bits must be 32 or 64");
}

arena_status arena_field_compare(size_t count, int precision_bits, const void* d_num, const void* d_exact,
                                 double* rel_l2, double* linf_rel, double* gauge_shift) {
  if (count < 1 || !d_num || !d_exact) return arena_fft::set_error(ARENA_EINVAL, "bad field");
  if (precision_bits == 64) return compare_t<double>(count, d_num, d_exact, rel_l2, linf_rel, gauge_shift);
  if (precision_bits == 32) return compare_t<float>(count, d_num, d_exact, rel_l2, linf_rel, gauge_shift);
  return arena_fft::set_error(ARENA_EINVAL, "precision_bits must be 32 or 64");
}

}  // extern "C"
