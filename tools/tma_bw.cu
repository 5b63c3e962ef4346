// tma_bw.cu — microbenchmark: TMA load throughput for the strided-pass tile
// shapes (rows x row-bytes), no compute.  Not product code.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_1408_6497_b200/csrc/async_copy.cuh"

using namespace arena_fft;

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

// Each CTA streams `per_cta` tiles of `tile_bytes` through NB buffers (ring), touching one value.
__global__ void tload(const __grid_constant__ CUtensorMap map, int tiles, int kt_count, int rows_per_box,
                      int boxes, int tile_elems, int nb, double* sink) {
  extern __shared__ __align__(128) unsigned char smraw[];
  double2* buf = reinterpret_cast<double2*>(smraw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smraw + size_t(nb) * tile_elems * 16);
  if (threadIdx.x == 0) {
    for (int b = 0; b < nb; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int g, int b) {
    const int outer = g / kt_count, kt = g % kt_count;
    mbar_arrive_expect_tx(&bar[b], tile_elems * 16);
    for (int q = 0; q < boxes; ++q)
      tma_load_4d(buf + size_t(b) * tile_elems + size_t(q) * rows_per_box * (tile_elems / (rows_per_box * boxes)),
                  &map, &bar[b], 2 * kt * (tile_elems / (rows_per_box * boxes)), 0, outer, q * rows_per_box);
  };
  double acc = 0;
  int it = 0;
  if (threadIdx.x == 0)
    for (int p = 0; p < nb && blockIdx.x + p * gridDim.x < tiles; ++p) issue(blockIdx.x + p * gridDim.x, p);
  for (int g = blockIdx.x; g < tiles; g += gridDim.x, ++it) {
    const int b = it % nb;
    mbar_wait(&bar[b], (it / nb) & 1);
    acc += buf[size_t(b) * tile_elems + threadIdx.x].x;
    __syncthreads();
    const int gn = g + nb * gridDim.x;
    if (threadIdx.x == 0 && gn < tiles) {
      fence_proxy_async_smem();
      issue(gn, b);
    }
  }
  if (acc == 12345.678) sink[0] = acc;
}

int main() {
  const int n = 1024, ncp = 520, nc = 513;
  double2* a;
  const size_t elems = size_t(n) * n * ncp;
  CK(cudaMalloc(&a, elems * 16));
  CK(cudaMemset(a, 0, elems * 16));
  double* sink;
  CK(cudaMalloc(&sink, 8));
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  // view: {2*nc doubles, rows j (n), plane i (n)} with y tiles: fixed i, all j (row stride ncp*16)
  for (int L : {2, 4, 8, 16}) {
    for (int nb : {1, 2, 3}) {
      for (int ctas : {1, 2, 3}) {
        const int tile_elems = L * n;
        const size_t smem = size_t(nb) * tile_elems * 16 + 64;
        if (smem * ctas > 227 * 1024) continue;
        const int rows_per_box = 256, boxes = n / rows_per_box;
        CUtensorMap map;
        cuuint64_t dims[4] = {cuuint64_t(2 * nc), 1, cuuint64_t(n), cuuint64_t(n)};  // k, dummy, i, j... use j as dim3
        // dims: d0 = k reals, d1 = 1, d2 = i (plane), d3 = j (row)  -> row stride ncp*16, plane stride n*ncp*16
        cuuint64_t strides[3] = {cuuint64_t(ncp) * 16, cuuint64_t(ncp) * 16 * n, cuuint64_t(ncp) * 16};
        // reorder so that box over j uses the small stride: swap d2/d3 roles
        cuuint64_t dims2[4] = {cuuint64_t(2 * nc), 1, cuuint64_t(n), cuuint64_t(n)};
        cuuint64_t str2[3] = {cuuint64_t(ncp) * 16, cuuint64_t(ncp) * 16, cuuint64_t(ncp) * 16 * n};
        (void)dims;
        (void)strides;
        cuuint32_t box[4] = {cuuint32_t(2 * L), 1, 1, cuuint32_t(rows_per_box)};
        cuuint32_t es[4] = {1, 1, 1, 1};
        // d2 = plane i (stride n*ncp*16) is the "outer", d3 = j rows (stride ncp*16): fix by swapping
        cuuint64_t d3[4] = {cuuint64_t(2 * nc), 1, cuuint64_t(n), cuuint64_t(n)};
        cuuint64_t s3[3] = {cuuint64_t(ncp) * 16, cuuint64_t(ncp) * 16 * n, cuuint64_t(ncp) * 16};
        (void)dims2;
        (void)str2;
        if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, a, d3, s3, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
          printf("encode failed L=%d\n", L);
          continue;
        }
        CK(cudaFuncSetAttribute(tload, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        const int kt_count = (nc + L - 1) / L, tiles = n * kt_count;
        const int grid = 148 * ctas;
        cudaEvent_t s, e;
        cudaEventCreate(&s);
        cudaEventCreate(&e);
        tload<<<grid, 128, smem>>>(map, tiles, kt_count, rows_per_box, boxes, tile_elems, nb, sink);
        CK(cudaDeviceSynchronize());
        cudaEventRecord(s);
        tload<<<grid, 128, smem>>>(map, tiles, kt_count, rows_per_box, boxes, tile_elems, nb, sink);
        cudaEventRecord(e);
        CK(cudaEventSynchronize(e));
        float ms;
        cudaEventElapsedTime(&ms, s, e);
        const double bytes = double(n) * n * nc * 16;
        printf("L=%2d (%3d B rows) bufs=%d ctas/SM=%d : %7.1f GB/s read\n", L, 16 * L, nb, ctas, bytes / ms / 1e6);
      }
    }
  }
  return 0;
}
