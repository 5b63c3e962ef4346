// plan.cu — the C ABI (include/arena_fft.h): plans, workspace, host boundary;
// the multi-GPU decompositions follow in plan_slab.cuh, plan_mgpu.cuh and
// plan_pencil.cuh (included at the end: one translation unit).
//
// Replaces the per-call FFTW planning/execution of
// /root/reference/proj/src/fft_solver.cpp:51-87 with a once-per-(n, precision,
// device) plan ("Setup") whose solve only enqueues kernels.
// No CPU fallback: a plan can only be created on a device this library was
// compiled for (sm_100a); anything else is ARENA_EUNSUPPORTED.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <thread>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/arena_fft.h"
#include "host_staging.h"
#include "launchers.h"

using namespace arena_fft;

namespace {

thread_local std::string g_last_error;

arena_status fail(arena_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

arena_status cuda_fail(cudaError_t e, const char* what) {
  return fail(ARENA_ECUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

bool is_pow2(int n) { return n >= 2 && (n & (n - 1)) == 0; }

}  // namespace

// For the other translation units (verify.cu): set the thread's arena_last_error.
namespace arena_fft {
arena_status set_error(arena_status s, const std::string& msg) { return fail(s, msg); }
}  // namespace arena_fft

namespace {

// stage names by fused mask (0: none, 1: forward pair fused, 2: inverse pair, 3: both)
const char* kStageNames[4][kPow2Launches] = {
    {"zfwd_r2c", "yfwd", "xmid_fwd_scale_inv", "yinv", "zinv_c2r"},
    {"zy_fused_fwd", "xmid_fwd_scale_inv", "yinv", "zinv_c2r", nullptr},
    {"zfwd_r2c", "yfwd", "xmid_fwd_scale_inv", "yz_fused_inv", nullptr},
    {"zy_fused_fwd", "xmid_fwd_scale_inv", "yz_fused_inv", nullptr, nullptr}};
const char* kSplit3Names[kSplit3Launches] = {"zsplit_r2c", "split3_fwd", "yfwd", "xmid_fwd_scale_inv", "yinv",
                                             "split3_inv", "zsplit_c2r"};
const char* kGenNames[kGenLaunches] = {"gen_z_r2c", "gen_y_fwd", "gen_xmid_fwd_scale_inv", "gen_y_inv",
                                       "gen_z_c2r"};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace

struct arena_fft_plan {
  int n = 0, prec = 64, device = 0, path = ARENA_PATH_POW2;
  int nc = 0, ncp = 0;
  size_t elem = 8;  // bytes per real
  void* spec = nullptr;  // half spectrum workspace
  size_t spec_bytes = 0;
  void* tw = nullptr;  // W_n^m table, vec2 of the precision
  void* stw = nullptr;  // stage-twiddle tables (power-of-two path)
  GenPlan gplan{};
  TmaCache* tma = nullptr;  // TMA descriptors (power-of-two path), nullptr = classic kernels
  int* ctrs = nullptr;      // fused z+y schedule counters (n + 1 ints), nullptr = unfused
  // CUDA graphs of the launch sequence for small n (launch-bound), keyed by (f, u)
  struct GraphEntry {
    const void* f;
    void* u;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  bool use_graphs = false;
  int lag = 2;
  int fuse = 0;             // kFuseFwd | kFuseInv
  int quad = 0;             // quadrant formulation (poisson_quad.cuh)
  bool split3 = false;      // generic n = 3M: radix-3 split onto the power-of-two passes (poisson_split3.cuh)
  void* Q = nullptr;        // split3: nine-chunk workspace
  void* stwz = nullptr;     // split3: stage tables of the M/2-point z sub-FFTs (nullptr: generic z passes)
  int sm_count = 148;
  // host-boundary resources (lazily allocated)
  void* d_in = nullptr;   // dft3 host paths: n^3 complex
  void* d_out = nullptr;
  void* d_real = nullptr;  // Poisson host solve: one n^3 real field, solved in place
  void* d_work = nullptr;  // n^3 complex, dft3 only
  cudaStream_t hstream = nullptr;
  std::mutex host_mu;  // one host-path call in flight per plan
  Stager* stager = nullptr;  // pinned staging ring for pageable host buffers (lazy)
  // batched host path: double-buffered device fields, copy-in / copy-out streams
  void* bin[2] = {nullptr, nullptr};
  void* bout[2] = {nullptr, nullptr};
  cudaStream_t s_in = nullptr, s_out = nullptr;
  // stage timing
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  int ev_sets_used = 0;
  std::vector<double> stage_ms;
  int solves = 0;
  std::mutex ev_mu;
  // Every solve on this plan reads and writes the plan's workspace (spec, Q) and
  // may update the graph / TMA caches.  enq_mu serialises the enqueues, and
  // ws_ev (recorded after each solve's last launch) makes the next solve's
  // stream wait for the previous one, whatever streams the callers use.
  std::mutex enq_mu;
  cudaEvent_t ws_ev = nullptr;
  bool ws_ev_live = false;

  int launches() const {
    if (path != ARENA_PATH_POW2) return split3 ? kSplit3Launches : kGenLaunches;
    return kPow2Launches - ((ctrs && (fuse & kFuseFwd)) ? 1 : 0) - ((ctrs && (fuse & kFuseInv)) ? 1 : 0);
  }
  size_t real_bytes() const { return size_t(n) * n * n * elem; }
};

namespace {

arena_status make_twiddles(arena_fft_plan* p) {
  // W_n^m = exp(-2 pi i m / n), m in [0, n), computed in 80-bit long double
  // and rounded once to the plan's precision.
  const int n = p->n;
  const long double two_pi = 6.283185307179586476925286766559005768L;
  const size_t vb = 2 * p->elem;
  std::vector<unsigned char> host(size_t(n) * vb);
  for (int m = 0; m < n; ++m) {
    const long double a = two_pi * (long double)m / (long double)n;
    const long double c = cosl(a), s = -sinl(a);
    if (p->prec == 64) {
      double v[2] = {double(c), double(s)};
      memcpy(host.data() + m * vb, v, vb);
    } else {
      float v[2] = {float(c), float(s)};
      memcpy(host.data() + m * vb, v, vb);
    }
  }
  cudaError_t e = cudaMalloc(&p->tw, host.size());
  if (e != cudaSuccess) return e == cudaErrorMemoryAllocation ? fail(ARENA_ENOMEM, "twiddle table") : cuda_fail(e, "cudaMalloc");
  e = cudaMemcpy(p->tw, host.data(), host.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "twiddle upload");
  if (p->path == ARENA_PATH_POW2 || p->split3) {
    const int nt = p->split3 ? 2 * (n / split_radix(n)) : n;  // split: M-point lines = the n/2 tables of n' = 2M
    const size_t ns = stw_entries(nt);
    std::vector<unsigned char> st(std::max<size_t>(ns, 1) * vb);
    stw_fill_host(nt, p->prec, st.data());
    if ((e = cudaMalloc(&p->stw, st.size())) != cudaSuccess) return fail(ARENA_ENOMEM, "stage twiddle tables");
    if ((e = cudaMemcpy(p->stw, st.data(), st.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return cuda_fail(e, "stage twiddle upload");
  }
  const char* zk = std::getenv("ARENA_FFT_SPLITZ");  // "0": the generic z passes on the split path
  if (p->split3 && !(zk && std::string(zk) == "0")) {
    const int nz = n / split_radix(n);  // tables of an n'' = M plan: M/2-point lines (which = 0)
    std::vector<unsigned char> st(std::max<size_t>(stw_entries(nz), 1) * vb);
    stw_fill_host(nz, p->prec, st.data());
    if ((e = cudaMalloc(&p->stwz, st.size())) != cudaSuccess) return fail(ARENA_ENOMEM, "z stage twiddle tables");
    if ((e = cudaMemcpy(p->stwz, st.data(), st.size(), cudaMemcpyHostToDevice)) != cudaSuccess)
      return cuda_fail(e, "z stage twiddle upload");
  }
  return ARENA_OK;
}

void free_plan(arena_fft_plan* p) {
  if (!p) return;
  DeviceGuard g(p->device);
  if (p->spec) cudaFree(p->spec);
  if (p->Q) cudaFree(p->Q);
  if (p->stwz) cudaFree(p->stwz);
  if (p->tw) cudaFree(p->tw);
  if (p->stw) cudaFree(p->stw);
  if (p->ctrs) cudaFree(p->ctrs);
  if (p->d_in) cudaFree(p->d_in);
  if (p->d_out) cudaFree(p->d_out);
  if (p->d_real) cudaFree(p->d_real);
  if (p->d_work) cudaFree(p->d_work);
  if (p->hstream) cudaStreamDestroy(p->hstream);
  for (int b = 0; b < 2; ++b) {
    if (p->bin[b]) cudaFree(p->bin[b]);
    if (p->bout[b]) cudaFree(p->bout[b]);
  }
  if (p->s_in) cudaStreamDestroy(p->s_in);
  for (auto& ge : p->graphs) cudaGraphExecDestroy(ge.exec);
  if (p->s_out) cudaStreamDestroy(p->s_out);
  delete p->tma;
  delete p->stager;
  for (cudaEvent_t e : p->ev_pool) cudaEventDestroy(e);
  if (p->ws_ev) cudaEventDestroy(p->ws_ev);
  delete p;
}

// Events for one timed solve (launches + 1), recycled after each query.
cudaEvent_t* timing_events(arena_fft_plan* p) {
  if (!p->timing) return nullptr;
  std::lock_guard<std::mutex> lk(p->ev_mu);
  const int per = p->launches() + 1;
  const int need = (p->ev_sets_used + 1) * per;
  while (int(p->ev_pool.size()) < need) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    p->ev_pool.push_back(e);
  }
  cudaEvent_t* ev = p->ev_pool.data() + p->ev_sets_used * per;
  ++p->ev_sets_used;
  return ev;
}

arena_status enqueue_kernels(arena_fft_plan* p, const void* d_f, void* d_u, cudaStream_t s, cudaEvent_t* ev);

// Small grids are launch-bound (five launches of a few microseconds each), so
// their launch sequence is captured once per (f, u) into a CUDA graph and
// replayed with one cudaGraphLaunch.  Not used with stage timing or on the
// legacy default stream (which cannot be captured).
arena_status enqueue_solve_locked(arena_fft_plan* p, const void* d_f, void* d_u, cudaStream_t s) {
  if (p->use_graphs && !p->timing && s != nullptr) {
    for (auto& ge : p->graphs)
      if (ge.f == d_f && ge.u == d_u) {
        cudaError_t e = cudaGraphLaunch(ge.exec, s);
        return e == cudaSuccess ? ARENA_OK : cuda_fail(e, "cudaGraphLaunch");
      }
    // first solve for this (f, u): run it eagerly (sets kernel attributes), then capture
    arena_status st = enqueue_kernels(p, d_f, d_u, s, nullptr);
    if (st != ARENA_OK) return st;
    cudaStream_t cap;
    if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess) return ARENA_OK;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool ok = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      const bool launched = enqueue_kernels(p, d_f, d_u, cap, nullptr) == ARENA_OK;
      ok = cudaStreamEndCapture(cap, &graph) == cudaSuccess && launched;
    }
    if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    cudaStreamDestroy(cap);
    cudaGetLastError();  // a failed capture only means no graph: clear it
    if (ok) {
      if (p->graphs.size() >= 8) {
        cudaGraphExecDestroy(p->graphs.front().exec);
        p->graphs.erase(p->graphs.begin());
      }
      p->graphs.push_back({d_f, d_u, exec});
    }
    return ARENA_OK;
  }
  return enqueue_kernels(p, d_f, d_u, s, timing_events(p));
}

// Workspace ordering across callers and streams (see arena_fft_plan::enq_mu).
arena_status enqueue_solve(arena_fft_plan* p, const void* d_f, void* d_u, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(p->enq_mu);
  cudaError_t e;
  if (!p->ws_ev && (e = cudaEventCreateWithFlags(&p->ws_ev, cudaEventDisableTiming)) != cudaSuccess)
    return cuda_fail(e, "cudaEventCreate");
  if (p->ws_ev_live && (e = cudaStreamWaitEvent(s, p->ws_ev, 0)) != cudaSuccess)
    return cuda_fail(e, "cudaStreamWaitEvent (previous solve on this plan)");
  arena_status st = enqueue_solve_locked(p, d_f, d_u, s);
  if (st != ARENA_OK) return st;
  if ((e = cudaEventRecord(p->ws_ev, s)) != cudaSuccess) return cuda_fail(e, "cudaEventRecord");
  p->ws_ev_live = true;
  return ARENA_OK;
}

arena_status enqueue_kernels(arena_fft_plan* p, const void* d_f, void* d_u, cudaStream_t s, cudaEvent_t* ev) {
  cudaError_t e;
  if (p->path == ARENA_PATH_POW2) {
    Pow2Args a{d_f, d_u, p->spec, p->tw, p->stw, p->n, p->nc, p->ncp, s, ev, p->tma, p->sm_count,
               /*ni*/ p->n, /*nj*/ p->n, /*nchunks*/ 1, /*j0*/ 0, /*specC*/ p->spec, kPhaseAll, p->ctrs, p->lag, p->fuse};
    a.quad = p->quad;
    e = p->prec == 64 ? launch_pow2_f64(a) : launch_pow2_f32(a);
  } else if (p->split3) {
    const int R = split_radix(p->n);
    Split3Args a{d_f, d_u, p->spec, p->Q, p->tw, p->stw, p->stwz, p->n, R, p->n / R, p->nc, p->ncp, s, ev, p->tma,
                 p->sm_count, &p->gplan};
    e = p->prec == 64 ? launch_split3_f64(a) : launch_split3_f32(a);
  } else {
    GenArgs a{&p->gplan, p->tw, p->n, p->nc, p->ncp, s, ev};
    e = p->prec == 64 ? gen_poisson_f64(a, d_f, d_u, p->spec) : gen_poisson_f32(a, d_f, d_u, p->spec);
  }
  if (e != cudaSuccess) return cuda_fail(e, "poisson solve launch");
  return ARENA_OK;
}

arena_status ensure_host_stream(arena_fft_plan* p) {
  cudaError_t e;
  if (!p->hstream && (e = cudaStreamCreateWithFlags(&p->hstream, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_fail(e, "cudaStreamCreate");
  return ARENA_OK;
}

// The Poisson host solve moves f in, solves in place (every path reads all of
// f before it writes u) and moves u out: f + workspace on the device, so a
// 2048^3 fp64 GridField (68.7 GB) fits one B200 with its 69 GB workspace.
arena_status ensure_real_buffer(arena_fft_plan* p) {
  arena_status st = ensure_host_stream(p);
  if (st != ARENA_OK) return st;
  cudaError_t e;
  if (!p->d_real && (e = cudaMalloc(&p->d_real, p->real_bytes())) != cudaSuccess)
    return fail(ARENA_ENOMEM, "device field buffer: " + std::string(cudaGetErrorString(e)));
  return ARENA_OK;
}

arena_status ensure_host_buffers(arena_fft_plan* p, bool work) {
  cudaError_t e;
  arena_status st = ensure_host_stream(p);
  if (st != ARENA_OK) return st;
  const size_t cb = size_t(p->n) * p->n * p->n * 2 * p->elem;  // n^3 complex (covers n^3 real)
  if (!p->d_in && (e = cudaMalloc(&p->d_in, cb)) != cudaSuccess)
    return fail(ARENA_ENOMEM, "device input buffer: " + std::string(cudaGetErrorString(e)));
  if (!p->d_out && (e = cudaMalloc(&p->d_out, cb)) != cudaSuccess)
    return fail(ARENA_ENOMEM, "device output buffer: " + std::string(cudaGetErrorString(e)));
  if (work && !p->d_work && (e = cudaMalloc(&p->d_work, cb)) != cudaSuccess)
    return fail(ARENA_ENOMEM, "device work buffer: " + std::string(cudaGetErrorString(e)));
  return ARENA_OK;
}

// Host <-> device copy on the plan's host stream: pinned buffers directly,
// pageable ones through the staging ring (host_staging.h).  to_host waits.
cudaError_t host_copy(arena_fft_plan* p, void* dst, const void* src, size_t bytes, bool to_host) {
  const void* host = to_host ? dst : src;
  if (host_ptr_pinned(host)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice,
                                    p->hstream);
    return (e || !to_host) ? e : cudaStreamSynchronize(p->hstream);
  }
  if (!p->stager) {
    p->stager = new (std::nothrow) Stager;
    if (!p->stager) return cudaErrorMemoryAllocation;
    cudaError_t e = p->stager->init();
    if (e != cudaSuccess) {
      delete p->stager;
      p->stager = nullptr;
      return e;
    }
  }
  return to_host ? p->stager->d2h(dst, src, bytes, p->hstream) : p->stager->h2d(dst, src, bytes, p->hstream);
}

}  // namespace

extern "C" {

const char* arena_last_error(void) { return g_last_error.c_str(); }

int arena_fft_abi_version(void) { return 101; }

int arena_current_device(void) {
  int d = -1;
  return cudaGetDevice(&d) == cudaSuccess ? d : -1;
}

}  // extern "C"

// Plan construction shared by single-GPU plans and slab ranks (which own
// their own, smaller workspaces and pass alloc_spec = false).
static arena_status create_plan(arena_fft_plan** out, int n, int precision_bits, int device, bool alloc_spec) {
  if (!out) return fail(ARENA_EINVAL, "plan pointer is NULL");
  *out = nullptr;
  if (n < 2) return fail(ARENA_EINVAL, "GridField: n >= 2 required");  // grid.hpp:18
  if (precision_bits != 64 && precision_bits != 32) return fail(ARENA_EINVAL, "precision_bits must be 64 or 32");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) return fail(ARENA_EUNSUPPORTED, "no CUDA device visible (this library has no CPU path)");
  if (device < 0 && cudaGetDevice(&device) != cudaSuccess) return fail(ARENA_ECUDA, "cudaGetDevice");
  if (device >= ndev) return fail(ARENA_EINVAL, "device ordinal out of range");
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(ARENA_EUNSUPPORTED, "device is sm_" + std::to_string(prop.major * 10 + prop.minor) +
                                        "; this library is built for sm_100a (B200) only");
  DeviceGuard g(device);
  arena_fft_plan* p = new (std::nothrow) arena_fft_plan;
  if (!p) return fail(ARENA_ENOMEM, "plan");
  p->n = n;
  p->prec = precision_bits;
  p->device = device;
  p->elem = precision_bits == 64 ? 8 : 4;
  p->nc = n / 2 + 1;
  p->ncp = spec_pitch(n);  // poisson_pow2.cuh (the kernels check it)
  p->sm_count = prop.multiProcessorCount;
  if (const char* sms = std::getenv("ARENA_FFT_SMS")) {  // experiments: persistent kernels on fewer SMs
    const int v = std::atoi(sms);
    if (v >= 1 && v < p->sm_count) p->sm_count = v;
  }
  {
    const char* gr = std::getenv("ARENA_FFT_GRAPHS");  // "0" disables graph replay
    p->use_graphs = n <= 256 && !(gr && std::string(gr) == "0");
  }
  if (is_pow2(n) && n <= kPow2MaxN) {
    p->path = ARENA_PATH_POW2;
    const char* kern = std::getenv("ARENA_FFT_KERNELS");  // "classic" selects the non-TMA strided kernels
    if (!(kern && std::string(kern) == "classic")) p->tma = new (std::nothrow) TmaCache;
    // L2-fused z+y pairs (halve the DRAM traffic of K1+K2 / K4+K5).  B200 A/B (r01,
    // final kernel configuration, 1024^3): unfused 18.7 ms, inverse pair fused 19.1,
    // forward 19.3, both 20.5; at 512^3 fusion also lost.  Default: off.
    // ARENA_FFT_FUSED = 0 | fwd | inv | 1 (both).
    const char* fz = std::getenv("ARENA_FFT_FUSED");
    const bool fused_ok = precision_bits == 64 ? pow2_fused_ok_f64(n) : pow2_fused_ok_f32(n);
    int fuse = 0;
    if (fz) {
      const std::string v(fz);
      fuse = v == "0" ? 0 : v == "fwd" ? kFuseFwd : v == "inv" ? kFuseInv : (kFuseFwd | kFuseInv);
    }
    if (p->tma && fused_ok && fuse) {
      p->fuse = fuse;
      if ((e = cudaMalloc(&p->ctrs, sizeof(int) * size_t(n + 1))) != cudaSuccess) {
        free_plan(p);
        return fail(ARENA_ENOMEM, "fused schedule counters");
      }
    }
    if (const char* lg = std::getenv("ARENA_FFT_FUSED_LAG")) p->lag = std::atoi(lg);
    // Quadrant formulation (poisson_quad.cuh): default for n >= 2048, where the n-point
    // y / x tiles no longer fit 128-byte rows in shared memory, and for fp64 n = 512.
    // B200 A/B (ms per solve, plain / quadrant): 2048^3 fp64 178 / 148, fp32 95 / 84;
    // 1024^3 17.5 / 18.2; 512^3 fp64 2.10 / 2.01, fp32 1.10 / 1.10; 256^3 0.295 / 0.307.
    // ARENA_FFT_QUAD = 0 | 1 overrides (any n >= 32 with the TMA kernels).
    {
      const char* qz = std::getenv("ARENA_FFT_QUAD");
      int want = 0;
      if (qz) {
        const std::string v(qz);
        want = v == "1" ? 1 : 0;
      } else {
        want = (n >= 2048 || (n == 512 && precision_bits == 64)) ? 1 : 0;
      }
      p->quad = (want && p->tma && n >= 32 && !p->fuse) ? want : 0;
    }
  } else {
    p->path = ARENA_PATH_GENERIC;
    if (!gen_plan_make(n, &p->gplan)) {
      free_plan(p);
      return fail(ARENA_EUNSUPPORTED, "cannot factor n");
    }
    if (n > gen_max_n(int(2 * p->elem))) {
      free_plan(p);
      return fail(ARENA_EUNSUPPORTED, "n = " + std::to_string(n) + " exceeds the generic path's shared-memory line limit");
    }
    // n = 3M, M a power of two in [16, 512]: y / x passes on the power-of-two TMA kernels
    // (poisson_split3.cuh).  ARENA_FFT_SPLIT3 = 0 keeps the generic stages.
    {
      const char* sz = std::getenv("ARENA_FFT_SPLIT3");
      const char* kern = std::getenv("ARENA_FFT_KERNELS");
      if (split_radix(n) && !(sz && std::string(sz) == "0") && !(kern && std::string(kern) == "classic")) {
        p->split3 = true;
        p->tma = new (std::nothrow) TmaCache;
        if (!p->tma) {
          free_plan(p);
          return fail(ARENA_ENOMEM, "TMA cache");
        }
      }
    }
  }
  arena_status st = make_twiddles(p);
  if (st != ARENA_OK) {
    free_plan(p);
    return st;
  }
  if (alloc_spec) {
    p->spec_bytes = size_t(n) * n * p->ncp * 2 * p->elem;
    if ((e = cudaMalloc(&p->spec, p->spec_bytes)) != cudaSuccess) {
      free_plan(p);
      return fail(ARENA_ENOMEM,
                  "half-spectrum workspace (" + std::to_string(p->spec_bytes) + " B): " + cudaGetErrorString(e));
    }
    if (p->split3 && (e = cudaMalloc(&p->Q, p->spec_bytes)) != cudaSuccess) {
      free_plan(p);
      return fail(ARENA_ENOMEM, "split3 workspace: " + std::string(cudaGetErrorString(e)));
    }
  }
  *out = p;
  g_last_error.clear();
  return ARENA_OK;
}

extern "C" {

arena_status arena_fft_plan_create(arena_fft_plan** out, int n, int precision_bits, int device) {
  return create_plan(out, n, precision_bits, device, true);
}

void arena_fft_plan_destroy(arena_fft_plan* plan) { free_plan(plan); }

arena_status arena_fft_plan_info(const arena_fft_plan* p, int* n, int* precision_bits, int* path, int* device,
                                 size_t* workspace_bytes) {
  if (!p) return fail(ARENA_EINVAL, "plan is NULL");
  if (n) *n = p->n;
  if (precision_bits) *precision_bits = p->prec;
  if (path) *path = p->path;
  if (device) *device = p->device;
  if (workspace_bytes) *workspace_bytes = p->spec_bytes + (p->Q ? p->spec_bytes : 0);  // split plans own Q too
  return ARENA_OK;
}

int arena_poisson_launches_per_solve(const arena_fft_plan* p) { return p ? p->launches() : 0; }

int arena_pow2_kernel_geometry(int n, int precision_bits, int* out15) {
  KernelGeom g[3];
  const bool ok = precision_bits == 64 ? pow2_config_f64(n, g) : pow2_config_f32(n, g);
  if (!ok || !out15) return ARENA_EINVAL;
  int* out10 = out15;
  for (int i = 0; i < 3; ++i) {
    out10[5 * i + 0] = g[i].line;
    out10[5 * i + 1] = g[i].E;
    out10[5 * i + 2] = g[i].L;
    out10[5 * i + 3] = g[i].threads;
    out10[5 * i + 4] = g[i].smem;
  }
  return ARENA_OK;
}

arena_status arena_poisson_solve_device(arena_fft_plan* p, const void* d_f, void* d_u, void* stream) {
  if (!p || !d_f || !d_u) return fail(ARENA_EINVAL, "NULL plan or buffer");
  DeviceGuard g(p->device);
  return enqueue_solve(p, d_f, d_u, static_cast<cudaStream_t>(stream));
}

arena_status arena_poisson_solve_host(arena_fft_plan* p, const void* f, void* u) {
  if (!p || !f || !u) return fail(ARENA_EINVAL, "NULL plan or buffer");
  DeviceGuard g(p->device);
  std::lock_guard<std::mutex> lk(p->host_mu);
  arena_status st = ensure_real_buffer(p);
  if (st != ARENA_OK) return st;
  const size_t bytes = p->real_bytes();
  cudaError_t e = host_copy(p, p->d_real, f, bytes, false);  // pageable GridField data: staged
  if (e != cudaSuccess) return cuda_fail(e, "H2D f");
  if ((st = enqueue_solve(p, p->d_real, p->d_real, p->hstream)) != ARENA_OK) return st;
  if ((e = host_copy(p, u, p->d_real, bytes, true)) != cudaSuccess) return cuda_fail(e, "D2H u");
  return ARENA_OK;
}

// Batched host solves: field s+1 is copied in and field s-1 copied out while
// field s is solved (PCIe is full duplex), so a stream of solves runs at
// max(H2D, D2H, solve) per field instead of their sum.
arena_status arena_poisson_solve_host_batch(arena_fft_plan* p, int count, const void* const* f, void* const* u) {
  if (!p || count < 0 || (count && (!f || !u))) return fail(ARENA_EINVAL, "NULL plan or buffer list");
  DeviceGuard g(p->device);
  std::lock_guard<std::mutex> lk(p->host_mu);
  arena_status st = ensure_host_stream(p);
  if (st != ARENA_OK) return st;
  cudaError_t e;
  const size_t bytes = p->real_bytes();
  for (int b = 0; b < 2; ++b) {
    if (!p->bin[b] && (e = cudaMalloc(&p->bin[b], bytes)) != cudaSuccess) return fail(ARENA_ENOMEM, "batch input buffer");
    if (!p->bout[b] && (e = cudaMalloc(&p->bout[b], bytes)) != cudaSuccess) return fail(ARENA_ENOMEM, "batch output buffer");
  }
  if (!p->s_in && (e = cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking))) return cuda_fail(e, "stream");
  if (!p->s_out && (e = cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking))) return cuda_fail(e, "stream");
  std::vector<cudaEvent_t> ev;
  auto mkev = [&]() {
    cudaEvent_t x;
    if (cudaEventCreateWithFlags(&x, cudaEventDisableTiming) != cudaSuccess) return (cudaEvent_t) nullptr;
    ev.push_back(x);
    return x;
  };
  std::vector<cudaEvent_t> in_done(count), solved(count), out_done(count);
  for (int s = 0; s < count; ++s) {
    in_done[s] = mkev();
    solved[s] = mkev();
    out_done[s] = mkev();
    if (!in_done[s] || !solved[s] || !out_done[s]) {
      for (cudaEvent_t x : ev) cudaEventDestroy(x);
      return fail(ARENA_ECUDA, "cudaEventCreate");
    }
  }
  st = ARENA_OK;
  for (int s = 0; s < count && st == ARENA_OK; ++s) {
    const int b = s & 1;
    // copy-in of field s into bin[b] once solve s-2 (the buffer's last reader) is done
    if (s >= 2) cudaStreamWaitEvent(p->s_in, solved[s - 2], 0);
    if ((e = cudaMemcpyAsync(p->bin[b], f[s], bytes, cudaMemcpyHostToDevice, p->s_in))) {
      st = cuda_fail(e, "batch H2D");
      break;
    }
    cudaEventRecord(in_done[s], p->s_in);
    // solve s once its input arrived and copy-out s-2 (last reader of bout[b]) finished
    cudaStreamWaitEvent(p->hstream, in_done[s], 0);
    if (s >= 2) cudaStreamWaitEvent(p->hstream, out_done[s - 2], 0);
    if ((st = enqueue_solve(p, p->bin[b], p->bout[b], p->hstream)) != ARENA_OK) break;
    cudaEventRecord(solved[s], p->hstream);
    // copy-out of field s
    cudaStreamWaitEvent(p->s_out, solved[s], 0);
    if ((e = cudaMemcpyAsync(u[s], p->bout[b], bytes, cudaMemcpyDeviceToHost, p->s_out))) {
      st = cuda_fail(e, "batch D2H");
      break;
    }
    cudaEventRecord(out_done[s], p->s_out);
  }
  if ((e = cudaStreamSynchronize(p->s_out)) != cudaSuccess && st == ARENA_OK) st = cuda_fail(e, "batch solve");
  cudaStreamSynchronize(p->hstream);
  cudaStreamSynchronize(p->s_in);
  for (cudaEvent_t x : ev) cudaEventDestroy(x);
  return st;
}

static arena_status dft3_fwd_enqueue(arena_fft_plan* p, const void* d_g, void* d_spec, cudaStream_t s) {
  GenArgs a{nullptr, p->tw, p->n, p->nc, p->ncp, s, nullptr};
  GenPlan gp;
  if (!gen_plan_make(p->n, &gp)) return fail(ARENA_EUNSUPPORTED, "cannot factor n");
  if (p->n > gen_max_n(int(2 * p->elem))) return fail(ARENA_EUNSUPPORTED, "n too large for dft3");
  a.plan = &gp;
  cudaError_t e = p->prec == 64 ? gen_dft3_forward_f64(a, d_g, d_spec) : gen_dft3_forward_f32(a, d_g, d_spec);
  return e == cudaSuccess ? ARENA_OK : cuda_fail(e, "dft3_forward");
}

static arena_status dft3_inv_enqueue(arena_fft_plan* p, const void* d_spec, void* d_g, void* d_work, cudaStream_t s) {
  GenArgs a{nullptr, p->tw, p->n, p->nc, p->ncp, s, nullptr};
  GenPlan gp;
  if (!gen_plan_make(p->n, &gp)) return fail(ARENA_EUNSUPPORTED, "cannot factor n");
  if (p->n > gen_max_n(int(2 * p->elem))) return fail(ARENA_EUNSUPPORTED, "n too large for dft3");
  a.plan = &gp;
  cudaError_t e = p->prec == 64 ? gen_dft3_inverse_f64(a, d_spec, d_g, d_work)
                                : gen_dft3_inverse_f32(a, d_spec, d_g, d_work);
  return e == cudaSuccess ? ARENA_OK : cuda_fail(e, "dft3_inverse");
}

arena_status arena_dft3_forward_device(arena_fft_plan* p, const void* d_g, void* d_spec, void* stream) {
  if (!p || !d_g || !d_spec) return fail(ARENA_EINVAL, "NULL plan or buffer");
  DeviceGuard g(p->device);
  return dft3_fwd_enqueue(p, d_g, d_spec, static_cast<cudaStream_t>(stream));
}

arena_status arena_dft3_inverse_device(arena_fft_plan* p, const void* d_spec, void* d_g, void* stream) {
  if (!p || !d_spec || !d_g) return fail(ARENA_EINVAL, "NULL plan or buffer");
  DeviceGuard g(p->device);
  std::lock_guard<std::mutex> lk(p->host_mu);  // d_work is plan-owned
  arena_status st = ensure_host_buffers(p, true);
  if (st != ARENA_OK) return st;
  return dft3_inv_enqueue(p, d_spec, d_g, p->d_work, static_cast<cudaStream_t>(stream));
}

arena_status arena_dft3_forward_host(arena_fft_plan* p, const void* g_host, void* spec_host) {
  if (!p || !g_host || !spec_host) return fail(ARENA_EINVAL, "NULL plan or buffer");
  DeviceGuard g(p->device);
  std::lock_guard<std::mutex> lk(p->host_mu);
  arena_status st = ensure_host_buffers(p, false);
  if (st != ARENA_OK) return st;
  cudaError_t e = host_copy(p, p->d_in, g_host, p->real_bytes(), false);
  if (e != cudaSuccess) return cuda_fail(e, "H2D g");
  if ((st = dft3_fwd_enqueue(p, p->d_in, p->d_out, p->hstream)) != ARENA_OK) return st;
  if ((e = host_copy(p, spec_host, p->d_out, 2 * p->real_bytes(), true))) return cuda_fail(e, "dft3_forward");
  return ARENA_OK;
}

arena_status arena_dft3_inverse_host(arena_fft_plan* p, const void* spec_host, void* g_host) {
  if (!p || !spec_host || !g_host) return fail(ARENA_EINVAL, "NULL plan or buffer");
  DeviceGuard g(p->device);
  std::lock_guard<std::mutex> lk(p->host_mu);
  arena_status st = ensure_host_buffers(p, true);
  if (st != ARENA_OK) return st;
  cudaError_t e = host_copy(p, p->d_in, spec_host, 2 * p->real_bytes(), false);
  if (e != cudaSuccess) return cuda_fail(e, "H2D spec");
  if ((st = dft3_inv_enqueue(p, p->d_in, p->d_out, p->d_work, p->hstream)) != ARENA_OK) return st;
  if ((e = host_copy(p, g_host, p->d_out, p->real_bytes(), true))) return cuda_fail(e, "dft3_inverse");
  return ARENA_OK;
}

arena_status arena_fft_set_stage_timing(arena_fft_plan* p, int enable) {
  if (!p) return fail(ARENA_EINVAL, "plan is NULL");
  std::lock_guard<std::mutex> lk(p->ev_mu);
  p->timing = enable != 0;
  p->ev_sets_used = 0;
  p->stage_ms.assign(p->launches(), 0.0);
  p->solves = 0;
  return ARENA_OK;
}

arena_status arena_fft_stage_times(arena_fft_plan* p, double* ms, const char** names, int max_stages, int* n_stages,
                                   int* n_solves) {
  if (!p) return fail(ARENA_EINVAL, "plan is NULL");
  DeviceGuard g(p->device);
  std::lock_guard<std::mutex> lk(p->ev_mu);
  const int L = p->launches(), per = L + 1;
  if (int(p->stage_ms.size()) != L) p->stage_ms.assign(L, 0.0);
  for (int s = 0; s < p->ev_sets_used; ++s) {
    cudaEvent_t* ev = p->ev_pool.data() + s * per;
    cudaError_t e = cudaEventSynchronize(ev[L]);
    if (e != cudaSuccess) return cuda_fail(e, "stage timing sync");
    for (int k = 0; k < L; ++k) {
      float t = 0;
      if ((e = cudaEventElapsedTime(&t, ev[k], ev[k + 1])) != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
      p->stage_ms[k] += t;
    }
    ++p->solves;
  }
  p->ev_sets_used = 0;
  const char** nm = p->path == ARENA_PATH_POW2 ? kStageNames[p->ctrs ? p->fuse : 0] : p->split3 ? kSplit3Names : kGenNames;
  for (int k = 0; k < L && k < max_stages; ++k) {
    if (ms) ms[k] = p->stage_ms[k];
    if (names) names[k] = nm[k];
  }
  if (n_stages) *n_stages = L;
  if (n_solves) *n_solves = p->solves;
  return ARENA_OK;
}

}  // extern "C"

// ============================================================================
// Multi-GPU decompositions (same translation unit: they reuse the plan internals).
#include "plan_slab.cuh"
#include "plan_mgpu.cuh"
#include "plan_pencil.cuh"
