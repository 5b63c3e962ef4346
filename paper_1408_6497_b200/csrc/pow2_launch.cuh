// pow2_launch.cuh — host-side launch sequence of the power-of-two path.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

#include "launchers.h"
#include "poisson_pow2.cuh"

namespace arena_fft {

// Raise the dynamic shared-memory limit of a kernel once per device (the
// kernel is a template argument so each instantiation has its own flag).
template <auto kernel>
inline cudaError_t ensure_smem(int bytes) {
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
  done_mask.fetch_or(bit);
  return cudaSuccess;
}

inline void mark(const Pow2Args& a, int i) {
  if (a.ev) cudaEventRecord(a.ev[i], a.stream);
}

template <typename T, int NR>
cudaError_t launch_pow2_n(const Pow2Args& a) {
  using V = vec2_t<T>;
  using CC = ContigCfg<T, NR>;
  using SC = StridedCfg<T, NR>;
  const V* tw = static_cast<const V*>(a.tw);
  V* S = static_cast<V*>(a.spec);
  cudaError_t e;
  if ((e = ensure_smem<k_zfwd<T, NR>>(CC::SMEM))) return e;
  if ((e = ensure_smem<k_zinv<T, NR>>(CC::SMEM))) return e;
  if ((e = ensure_smem<k_ypass<T, NR, -1>>(SC::SMEM))) return e;
  if ((e = ensure_smem<k_ypass<T, NR, +1>>(SC::SMEM))) return e;
  if ((e = ensure_smem<k_xmid<T, NR>>(SC::SMEM))) return e;
  const unsigned zgrid = unsigned((size_t(NR) * NR) / CC::L);
  const dim3 sgrid((a.nc + SC::L - 1) / SC::L, NR);
  const T scale = T(1.0 / (double(NR) * NR * NR));  // fft_solver.cpp:67
  const T four_pi2 = T(4.0 * M_PI * M_PI);           // fft_solver.cpp:66
  mark(a, 0);
  k_zfwd<T, NR><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(static_cast<const T*>(a.f), S, a.ncp, tw);
  mark(a, 1);
  k_ypass<T, NR, -1><<<sgrid, SC::THREADS, SC::SMEM, a.stream>>>(S, a.ncp, a.nc, tw);
  mark(a, 2);
  k_xmid<T, NR><<<sgrid, SC::THREADS, SC::SMEM, a.stream>>>(S, a.ncp, a.nc, tw, scale, four_pi2);
  mark(a, 3);
  k_ypass<T, NR, +1><<<sgrid, SC::THREADS, SC::SMEM, a.stream>>>(S, a.ncp, a.nc, tw);
  mark(a, 4);
  k_zinv<T, NR><<<zgrid, CC::THREADS, CC::SMEM, a.stream>>>(S, static_cast<T*>(a.u), a.ncp, tw);
  mark(a, 5);
  return cudaGetLastError();
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
