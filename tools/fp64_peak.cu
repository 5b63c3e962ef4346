// fp64_peak.cu — measured DFMA throughput of the B200 (the fp64 ridge point used
// in DESIGN.md's roofline discussion; MEASURED_PEAKS.json has no fp64 figure).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/fp64_peak.cu -o tools/fp64_peak
#include <cstdio>

__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) out[gridDim.x * blockDim.x + blockIdx.x] = double(t1 - t0);
}

int main() {
  int sms = 0, dev = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 1024, blocks = sms, iters = 1 << 16;  // one resident block per SM
  double* out;
  cudaMalloc(&out, sizeof(double) * (size_t(blocks) * threads + blocks));
  dfma_chains<<<blocks, threads>>>(out, 16, 0.999, 1e-3);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  dfma_chains<<<blocks, threads>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  double cyc = 0;
  cudaMemcpy(&cyc, out + size_t(blocks) * threads, sizeof(double), cudaMemcpyDeviceToHost);
  const double fmas = double(blocks) * threads * iters * 16;
  // one block per SM for ~cyc cycles: lanes/clk/SM = FMAs per SM / cycles
  printf("DFMA: %.2f TFLOP/s (2 flops/FMA) in %.3f ms; %.1f DFMA lanes/clk/SM (block 0: %.0f cycles, %.0f MHz)\n",
         2 * fmas / (ms * 1e-3) / 1e12, ms, fmas / sms / cyc, cyc, cyc / (ms * 1e3));
  return 0;
}
