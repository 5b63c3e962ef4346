// l2_probe.cu — per-kernel throughput of the 1024^3 pipeline when its working
// set is L2-resident (a few planes) versus HBM-streamed (many planes).  Tells
// whether a kernel is bound by HBM or by the SM side (issue / latency): only in
// the first case can L2 fusion of two passes pay.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//     -I include tools/l2_probe.cu paper_1408_6497_b200/csrc/pow2_f64.cu \
//     paper_1408_6497_b200/csrc/stage_twiddles.cu -lcuda -o tools/l2_probe
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "../paper_1408_6497_b200/csrc/launchers.h"

using namespace arena_fft;

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) {                                                          \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return 1;                                                                       \
    }                                                                                 \
  } while (0)

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 1024, nc = n / 2 + 1, ncp = (nc + 7) / 8 * 8;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  std::vector<double> tw(2 * n);
  for (int m = 0; m < n; ++m) {
    const long double a = 6.283185307179586476925286766559005768L * m / n;
    tw[2 * m] = double(cosl(a));
    tw[2 * m + 1] = double(-sinl(a));
  }
  std::vector<double> st(2 * stw_entries(n));
  stw_fill_host(n, 64, st.data());
  void *dtw, *dstw;
  CK(cudaMalloc(&dtw, tw.size() * 8));
  CK(cudaMalloc(&dstw, st.size() * 8));
  CK(cudaMemcpy(dtw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dstw, st.data(), st.size() * 8, cudaMemcpyHostToDevice));
  const int planes_list[] = {4, 8, n >= 2048 ? 128 : 512};
  printf("planes  MB(f+spec)   zfwd_us/plane  yfwd_us/plane  x_us/line-set  yinv_us/plane  zinv_us/plane\n");
  for (int planes : planes_list) {
    const size_t fb = size_t(planes) * n * n * 8, sb = size_t(planes) * n * ncp * 16;
    void *f, *u, *spec;
    CK(cudaMalloc(&f, fb));
    CK(cudaMalloc(&u, fb));
    CK(cudaMalloc(&spec, sb));
    CK(cudaMemset(f, 0, fb));
    CK(cudaMemset(spec, 0, sb));
    TmaCache cache{};
    cudaEvent_t ev[kPow2Launches + 1];
    for (auto& x : ev) CK(cudaEventCreate(&x));
    // ZY / YZ on `planes` local i planes (x all j); X on `planes` local j lines (x all i).
    Pow2Args a{f, u, spec, dtw, dstw, n, nc, ncp, 0, ev, &cache, sms, planes, planes, 1, 0, spec, kPhaseZY,
               nullptr, 2, 0};
    float tz = 0, ty = 0, tx = 0, tyi = 0, tzi = 0;
    const int reps = planes >= 64 ? 5 : 50;
    for (int r = 0; r < reps + 2; ++r) {
      float t0, t1, t2, t3;
      a.phases = kPhaseZY;
      CK(launch_pow2_f64(a));
      CK(cudaEventRecord(ev[5], 0));  // the ZY phase marks only the kernel starts
      CK(cudaEventSynchronize(ev[5]));
      CK(cudaEventElapsedTime(&t0, ev[0], ev[1]));
      CK(cudaEventElapsedTime(&t1, ev[1], ev[5]));
      a.phases = kPhaseYZ;
      CK(launch_pow2_f64(a));
      CK(cudaEventSynchronize(ev[2]));
      CK(cudaEventElapsedTime(&t2, ev[0], ev[1]));
      CK(cudaEventElapsedTime(&t3, ev[1], ev[2]));
      if (r >= 2) {
        tz += t0;
        ty += t1;
        tyi += t2;
        tzi += t3;
      }
    }
    // x pass: the C layout is (all i) x (planes local j) when nj = planes, nchunks = 1... the
    // single-chunk geometry needs ni = n for the x map, so time it with ni = n, nj = planes.
    {
      const size_t cb = size_t(n) * planes * ncp * 16;
      void* specC;
      CK(cudaMalloc(&specC, cb));
      CK(cudaMemset(specC, 0, cb));
      TmaCache cx{};
      Pow2Args ax = a;
      ax.tma = &cx;
      ax.ni = n;
      ax.nj = planes;
      ax.spec = specC;
      ax.specC = specC;
      ax.phases = kPhaseX;
      for (int r = 0; r < reps + 2; ++r) {
        float t;
        CK(launch_pow2_f64(ax));
        CK(cudaEventRecord(ev[5], 0));
        CK(cudaEventSynchronize(ev[5]));
        CK(cudaEventElapsedTime(&t, ev[0], ev[5]));
        if (r >= 2) tx += t;
      }
      CK(cudaFree(specC));
    }
    const double k = 1000.0 / reps / planes;
    printf("%6d  %10.1f   %13.2f  %13.2f  %13.2f  %13.2f  %13.2f\n", planes, (fb + sb) / 1e6, tz * k, ty * k,
           tx * k, tyi * k, tzi * k);
    CK(cudaFree(f));
    CK(cudaFree(u));
    CK(cudaFree(spec));
  }
  printf("(HBM-bound reference at 6441 GB/s: %.2f us per plane per pass)\n", 16.03 * n * n / 6441e9 * 1e6);
  return 0;
}
