// sources.cu — device-side generation of the BASELINE.json sources and
// analytic solutions.  Host sampling through
// std::function (grid.cpp:21-27) is infeasible at 1024^3-2048^3, so the bench
// and the large-size parity tests build f and the analytic u here.  Not part
// of the timed solve.
//
//  * Fourier-mode sums (configs 1, 2, 4):  out[i,j,k] = sum_m Re(c_m e^{2 pi i (kx i + ky j + kz k)/n})
//    with the phase index reduced exactly mod n and read from the W_n table.
//  * Periodised Gaussian (configs 3, 5): u = sum over the 27 nearest images of
//    exp(-alpha |x - c - m|^2), f = -Lap u = sum (6 alpha - 4 alpha^2 r^2) e^{-alpha r^2}.
//    (not the reference's TestCase::layer, §9 item 3.)
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/arena_fft.h"
#include "fft_engine.cuh"

namespace {

template <typename T>
__global__ void k_modes(T* __restrict__ out, int n, int i0, int ni, int j0, int nj, int nmodes,
                        const int* __restrict__ kv, const double* __restrict__ coef, const double2* __restrict__ tw) {
  const long long N = (long long)ni * nj * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int k = int(idx % n);
    const long long ij = idx / n;
    const int j = j0 + int(ij % nj), i = i0 + int(ij / nj);
    double acc = 0.0;
    for (int m = 0; m < nmodes; ++m) {
      long long p = ((long long)kv[3 * m] * i + (long long)kv[3 * m + 1] * j + (long long)kv[3 * m + 2] * k) % n;
      if (p < 0) p += n;
      const double2 w = __ldg(tw + p);  // cos(th) - i sin(th)
      acc += coef[2 * m] * w.x + coef[2 * m + 1] * w.y;  // Re((cr + i ci)(cos + i sin)) = cr cos - ci sin
    }
    out[idx] = T(acc);
  }
}

template <typename T>
__global__ void k_gauss(T* __restrict__ out, int n, int i0, int ni, int j0, int nj, double alpha, double cx, double cy,
                        double cz, int which) {
  const long long N = (long long)ni * nj * n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < N;
       idx += (long long)gridDim.x * blockDim.x) {
    const int k = int(idx % n);
    const long long ij = idx / n;
    const int j = j0 + int(ij % nj), i = i0 + int(ij / nj);
    const double x = double(i) / n, y = double(j) / n, z = double(k) / n;
    double acc = 0.0;
    for (int a = -1; a <= 1; ++a)
      for (int b = -1; b <= 1; ++b)
        for (int c = -1; c <= 1; ++c) {
          const double dx = x - cx - a, dy = y - cy - b, dz = z - cz - c;
          const double r2 = dx * dx + dy * dy + dz * dz;
          const double g = exp(-alpha * r2);
          acc += which == 0 ? g : (6.0 * alpha - 4.0 * alpha * alpha * r2) * g;
        }
    out[idx] = T(acc);
  }
}

thread_local std::string g_src_err;

}  // namespace

extern "C" {

// out (device, planes i0 .. i0+ni-1 of the n^3 field, precision_bits) =
// sum_m Re(coef_m e^{2 pi i k_m.x}); k: 3*nmodes ints, coef: 2*nmodes doubles (re, im), host arrays.
arena_status arena_source_modes_block(int n, int precision_bits, int nmodes, const int* k, const double* coef, int i0,
                                      int ni, int j0, int nj, void* d_out, void* stream) {
  if (n < 2 || nmodes < 0 || !d_out || (nmodes && (!k || !coef)) || i0 < 0 || ni < 1 || i0 + ni > n || j0 < 0 ||
      nj < 1 || j0 + nj > n)
    return ARENA_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<double> tw(2 * size_t(n));
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (int m = 0; m < n; ++m) {
    const long double a = two_pi * (long double)m / (long double)n;
    tw[2 * m] = double(cosl(a));
    tw[2 * m + 1] = double(-sinl(a));
  }
  void *d_tw = nullptr, *d_k = nullptr, *d_c = nullptr;
  const size_t bk = sizeof(int) * 3 * size_t(nmodes > 0 ? nmodes : 1), bc = sizeof(double) * 2 * size_t(nmodes > 0 ? nmodes : 1);
  if (cudaMalloc(&d_tw, tw.size() * sizeof(double)) || cudaMalloc(&d_k, bk) || cudaMalloc(&d_c, bc)) {
    cudaFree(d_tw); cudaFree(d_k); cudaFree(d_c);
    return ARENA_ENOMEM;
  }
  cudaMemcpy(d_tw, tw.data(), tw.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (nmodes) {
    cudaMemcpy(d_k, k, sizeof(int) * 3 * nmodes, cudaMemcpyHostToDevice);
    cudaMemcpy(d_c, coef, sizeof(double) * 2 * nmodes, cudaMemcpyHostToDevice);
  }
  if (precision_bits == 64)
    k_modes<double><<<148 * 16, 256, 0, s>>>(static_cast<double*>(d_out), n, i0, ni, j0, nj, nmodes, static_cast<int*>(d_k),
                                            static_cast<double*>(d_c), static_cast<double2*>(d_tw));
  else
    k_modes<float><<<148 * 16, 256, 0, s>>>(static_cast<float*>(d_out), n, i0, ni, j0, nj, nmodes, static_cast<int*>(d_k),
                                           static_cast<double*>(d_c), static_cast<double2*>(d_tw));
  cudaError_t e = cudaGetLastError();
  cudaStreamSynchronize(s);
  cudaFree(d_tw);
  cudaFree(d_k);
  cudaFree(d_c);
  return e == cudaSuccess ? ARENA_OK : ARENA_ECUDA;
}

arena_status arena_source_modes_slab(int n, int precision_bits, int nmodes, const int* k, const double* coef, int i0,
                                     int ni, void* d_out, void* stream) {
  return arena_source_modes_block(n, precision_bits, nmodes, k, coef, i0, ni, 0, n, d_out, stream);
}

arena_status arena_source_modes(int n, int precision_bits, int nmodes, const int* k, const double* coef, void* d_out,
                                void* stream) {
  return arena_source_modes_block(n, precision_bits, nmodes, k, coef, 0, n, 0, n, d_out, stream);
}

// which = 0: u (periodised Gaussian), 1: f = -Lap u; planes i0 .. i0+ni-1.
arena_status arena_source_gaussian_block(int n, int precision_bits, double alpha, double cx, double cy, double cz,
                                         int which, int i0, int ni, int j0, int nj, void* d_out, void* stream) {
  if (n < 2 || !d_out || (which != 0 && which != 1) || i0 < 0 || ni < 1 || i0 + ni > n || j0 < 0 || nj < 1 ||
      j0 + nj > n)
    return ARENA_EINVAL;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (precision_bits == 64)
    k_gauss<double><<<148 * 16, 256, 0, s>>>(static_cast<double*>(d_out), n, i0, ni, j0, nj, alpha, cx, cy, cz, which);
  else
    k_gauss<float><<<148 * 16, 256, 0, s>>>(static_cast<float*>(d_out), n, i0, ni, j0, nj, alpha, cx, cy, cz, which);
  return cudaGetLastError() == cudaSuccess ? ARENA_OK : ARENA_ECUDA;
}

arena_status arena_source_gaussian_slab(int n, int precision_bits, double alpha, double cx, double cy, double cz,
                                        int which, int i0, int ni, void* d_out, void* stream) {
  return arena_source_gaussian_block(n, precision_bits, alpha, cx, cy, cz, which, i0, ni, 0, n, d_out, stream);
}

arena_status arena_source_gaussian(int n, int precision_bits, double alpha, double cx, double cy, double cz, int which,
                                   void* d_out, void* stream) {
  return arena_source_gaussian_slab(n, precision_bits, alpha, cx, cy, cz, which, 0, n, d_out, stream);
}

}  // extern "C"
