// tmem_probe.cu — checks the tcgen05 data paths the TMEM-staged x pass relies on
// (no library code): shared memory -> TMEM with tcgen05.cp (.128x128b, .128x256b,
// no-swizzle shared-memory descriptor), TMEM -> registers with tcgen05.ld.32x32b,
// and their throughput per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

// Blackwell shared-memory matrix descriptor, no swizzle (layout type 0), version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;  // version
  return d;
}

__device__ __forceinline__ void mbar_init(uint64_t* b, int n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, int phase) {
  asm volatile(
      "{\n .reg .pred P1;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n }" ::"r"(smem_u32(b)),
      "r"(phase));
}

template <int SHAPE>  // 128: .128x128b, 256: .128x256b
__global__ void k_probe(int* bad, unsigned long long* cyc, int reps) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint32_t* data = reinterpret_cast<uint32_t*>(sm);      // 8 KB pattern
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < 2048; i += blockDim.x) data[i] = 0x10000u + i;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&taddr_s)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // generic smem writes -> async proxy (tcgen05.cp reads)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = taddr_s;
  // 128 rows of 16 B (SHAPE 128) or 2 x 16 B, the second one LBO = 2 KB further (SHAPE 256)
  if (tid == 0) {
    const uint64_t d = sdesc(smem_u32(data), 2048, 128);
    if (SHAPE == 128)
      asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr), "l"(d));
    else
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(d));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp < 4) {
    const int row = warp * 32 + lane;  // TMEM lane
    uint32_t r[8];
    const uint32_t a = taddr + (uint32_t(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(a));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    const int nw = SHAPE == 128 ? 4 : 8;
    for (int c = 0; c < nw; ++c) {
      const uint32_t want = 0x10000u + (c < 4 ? row * 4 + c : 512 + row * 4 + (c - 4));
      if (r[c] != want) {
        if (atomicAdd(bad, 1) < 4) printf("SHAPE %d lane %d col %d: got %x want %x\n", SHAPE, row, c, r[c], want);
      }
    }
    // throughput: tcgen05.ld.32x32b.x128 into registers, repeated
    uint32_t acc = 0;
    const unsigned long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
      uint32_t v[32];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(a + uint32_t((it & 3) * 32)));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += v[k];
    }
    const unsigned long long t1 = clock64();
    if (lane == 0 && warp == 0) cyc[0] = t1 - t0;
    if (acc == 0xdeadbeef) bad[1] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(256));
}

int main() {
  int* bad;
  unsigned long long* cyc;
  cudaMalloc(&bad, 8);
  cudaMalloc(&cyc, 8);
  for (int shape : {128, 256}) {
    cudaMemset(bad, 0, 8);
    const int reps = 1000;
    if (shape == 128) k_probe<128><<<1, 128, 8192>>>(bad, cyc, reps);
    else k_probe<256><<<1, 128, 8192>>>(bad, cyc, reps);
    cudaError_t e = cudaDeviceSynchronize();
    int hb[2];
    unsigned long long hc;
    cudaMemcpy(hb, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
    printf("tcgen05.cp .128x%db: %s, mismatches %d; tcgen05.ld 32x32b.x32 (4 warps): %.1f cycles per load+wait "
           "(%.1f B/cycle/SM)\n",
           shape, cudaGetErrorString(e), hb[0], double(hc) / reps, 4.0 * 32 * 32 * 4 / (double(hc) / reps));
  }
  return 0;
}
