// interpolant.cu — GPU evaluation of the sparse trigonometric interpolant of
// arena::SpectralInterpolant (/root/reference/proj/src/fft_solver.cpp:89-114;
// SURVEY.md §8(f)-4): out[p] = sum_m Re(a_m exp(2 pi i k_m . x_p)), a modes x
// points reduction.  The reference evaluates one point at a time on the host
// (fft_solver.cpp:107-114); this evaluates a batch (e.g. the SPEC's 10^4-point
// Halton set) with the modes staged through shared memory.  Phases use
// sincospi(2 t) so the 2*pi factor is not rounded separately.
#include <cuda_runtime.h>

#include <string>

#include "../../include/arena_fft.h"

namespace {

constexpr int kTile = 256;

__global__ void k_interp(const int* __restrict__ kv, const double2* __restrict__ amp, int nmodes,
                         const double* __restrict__ pts, int npts, double* __restrict__ out) {
  __shared__ int sk[3 * kTile];
  __shared__ double2 sa[kTile];
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  double x = 0, y = 0, z = 0;
  if (p < npts) {
    x = pts[3 * p];
    y = pts[3 * p + 1];
    z = pts[3 * p + 2];
  }
  double acc = 0.0;
  for (int m0 = 0; m0 < nmodes; m0 += kTile) {
    const int cnt = min(kTile, nmodes - m0);
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
      sk[3 * q] = kv[3 * (m0 + q)];
      sk[3 * q + 1] = kv[3 * (m0 + q) + 1];
      sk[3 * q + 2] = kv[3 * (m0 + q) + 2];
      sa[q] = amp[m0 + q];
    }
    __syncthreads();
    if (p < npts) {
      for (int q = 0; q < cnt; ++q) {
        const double t = sk[3 * q] * x + sk[3 * q + 1] * y + sk[3 * q + 2] * z;
        double s, c;
        sincospi(2.0 * t, &s, &c);
        acc += sa[q].x * c - sa[q].y * s;
      }
    }
    __syncthreads();
  }
  if (p < npts) out[p] = acc;
}

thread_local std::string g_err;

}  // namespace

extern "C" {

arena_status arena_interpolant_eval(int device, int nmodes, const int* k, const double* amp, int npts,
                                    const double* pts, double* out) {
  if (nmodes < 0 || npts < 0 || (nmodes && (!k || !amp)) || (npts && (!pts || !out))) return ARENA_EINVAL;
  if (npts == 0) return ARENA_OK;
  int prev = -1;
  cudaGetDevice(&prev);
  if (device >= 0 && cudaSetDevice(device) != cudaSuccess) return ARENA_EINVAL;
  void *dk = nullptr, *da = nullptr, *dp = nullptr, *dout = nullptr;
  const size_t bk = sizeof(int) * 3 * size_t(nmodes > 0 ? nmodes : 1), ba = 16 * size_t(nmodes > 0 ? nmodes : 1);
  arena_status st = ARENA_OK;
  if (cudaMalloc(&dk, bk) || cudaMalloc(&da, ba) || cudaMalloc(&dp, 24 * size_t(npts)) ||
      cudaMalloc(&dout, 8 * size_t(npts))) {
    st = ARENA_ENOMEM;
  } else {
    if (nmodes) {
      cudaMemcpy(dk, k, sizeof(int) * 3 * size_t(nmodes), cudaMemcpyHostToDevice);
      cudaMemcpy(da, amp, 16 * size_t(nmodes), cudaMemcpyHostToDevice);
    }
    cudaMemcpy(dp, pts, 24 * size_t(npts), cudaMemcpyHostToDevice);
    k_interp<<<(npts + 127) / 128, 128>>>(static_cast<int*>(dk), static_cast<double2*>(da), nmodes,
                                          static_cast<double*>(dp), npts, static_cast<double*>(dout));
    if (cudaGetLastError() != cudaSuccess ||
        cudaMemcpy(out, dout, 8 * size_t(npts), cudaMemcpyDeviceToHost) != cudaSuccess)
      st = ARENA_ECUDA;
  }
  cudaFree(dk);
  cudaFree(da);
  cudaFree(dp);
  cudaFree(dout);
  if (prev >= 0) cudaSetDevice(prev);
  return st;
}

}  // extern "C"
