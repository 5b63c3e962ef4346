// plan.cu — the C ABI (include/arena_fft.h): plans, workspace, host boundary.
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
  int xtmem = 0;            // x pass with TMEM-staged tiles (poisson_xtmem.cuh)
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
    a.xtmem = p->xtmem;
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
    // i-split formulation (poisson_hq.cuh): only the i transform's first radix-2 step
    // moves into the z passes, so the x pass runs n/2-point lines at twice the
    // occupancy while the y lines keep all n points.  ARENA_FFT_QUAD = hq selects it.
    {
      const char* qz = std::getenv("ARENA_FFT_QUAD");
      int want = 0;
      if (qz) {
        const std::string v(qz);
        want = v == "1" ? 1 : (v == "hq" || v == "2") ? 2 : 0;
      } else {
        want = (n >= 2048 || (n == 512 && precision_bits == 64)) ? 1 : 0;
      }
      p->quad = (want && p->tma && n >= 32 && !p->fuse) ? want : 0;
    }
    // x pass with the next tile staged in tensor memory (fp64 n = 1024).  ARENA_FFT_XTMEM = 0 | 1.
    {
      const char* xt = std::getenv("ARENA_FFT_XTMEM");
      const bool want = xt ? std::string(xt) == "1" : false;
      p->xtmem = (want && p->tma && !p->quad && n == 1024 && precision_bits == 64) ? 1 : 0;
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
// Slab decomposition over P ranks: rank r owns the f / u planes
// i in [r*n/P, (r+1)*n/P) (a contiguous part of GridField.data).  Per solve:
//   K1 z-r2c, K2 y-fwd on the rank's planes          (workspace B, layout B)
//   all-to-all #1: chunk d of B (j in rank d's range) -> rank d's C chunk r
//   K3 x-fwd * symbol * x-inv on the rank's j lines  (workspace C, layout C)
//   all-to-all #2: the reverse
//   K4 y-inv, K5 z-c2r                               (workspace B)
// Every chunk is one contiguous block of ni*nj rows (Layout, poisson_pow2.cuh),
// so the exchanges are plain grouped ncclSend/ncclRecv (NCCL has no all-to-all
// primitive) — or, for P virtual ranks on one device ("loopback", used to test
// the decomposition with one GPU), device-to-device cudaMemcpyAsync.
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;  // optional (hang / error detection)
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  bool ok = false;
};

// NCCL is loaded lazily (the single-GPU path never needs it); in a process that
// already loaded one (e.g. torch's), dlopen returns that same library.
NcclApi* nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      api.h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [](const char* s) { return dlsym(api.h, s); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd && api.Send &&
             api.Recv && api.GetErrorString;
  });
  return api.ok ? &api : nullptr;
}

arena_status nccl_fail(ncclResult_t r, const char* what) {
  NcclApi* a = nccl_api();
  return fail(ARENA_ENCCL, std::string(what) + ": " + (a ? a->GetErrorString(r) : "NCCL unavailable"));
}

struct SlabRank {
  void* B = nullptr;  // workspace B: ni * n rows
  void* C = nullptr;  // workspace C: n * nj rows
  int* ctrs = nullptr;  // fused z+y counters (ni + 1), nullptr = unfused
  TmaCache tma;
  // Peer exchange: rank d's C / B advanced to this rank's chunk (K2 / K3 store there).
  void* peerC[kMaxPeers] = {};
  void* peerB[kMaxPeers] = {};
};

// Barrier flags of the peer exchange: flags[d] of rank r = last epoch rank d
// announced to r (written by d over NVLink).
struct PeerFlags {
  unsigned* peer[kMaxPeers];  // rank d's flag array
  unsigned* mine;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Every rank announces `epoch` to every rank (release, system scope: the
// rank's earlier peer stores — previous kernels on the stream — become visible
// first), then waits until every rank has announced it (acquire).  Gives up
// after 20 s and sets *err instead of hanging the GPU.
__device__ void peer_barrier_body(const PeerFlags& pf, int rank, int P, unsigned epoch, int* err) {
  const int d = threadIdx.x;
  if (d < P) {
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(pf.peer[d] + rank), "r"(epoch) : "memory");
    const unsigned long long t0 = globaltimer_ns();
    for (;;) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(pf.mine + d) : "memory");
      if (int(v - epoch) >= 0) break;
      if (globaltimer_ns() - t0 > 20000000000ull) {
        atomicExch(err, 1);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

__global__ void k_peer_barrier(const __grid_constant__ PeerFlags pf, int rank, int P, unsigned epoch, int* err) {
  peer_barrier_body(pf, rank, P, epoch, err);
}

// Protocol self-test on ONE device: block r plays rank r (one cooperative
// launch, so all blocks are co-resident).  Each round every block publishes
// data[r] = round, passes the barrier, and checks it sees every block's value.
__global__ void k_peer_barrier_selftest(unsigned* flags, volatile int* data, int P, int rounds, int* err, int* bad) {
  const int r = blockIdx.x;
  PeerFlags pf;
  for (int d = 0; d < kMaxPeers; ++d) pf.peer[d] = flags + size_t(d < P ? d : 0) * P;
  pf.mine = flags + size_t(r) * P;
  for (int e = 1; e <= rounds; ++e) {
    if (threadIdx.x == 0) {
      __nanosleep(unsigned(r * 7919 + e * 104729) % 4000u);
      data[r] = e;
    }
    __syncthreads();
    peer_barrier_body(pf, r, P, unsigned(e), err);
    if (threadIdx.x < P && data[threadIdx.x] < e) atomicAdd(bad, 1);
    __syncthreads();
  }
}

// Peer-exchange state shared by the slab and pencil decompositions: this rank's
// barrier flags, the peers' flag arrays, the IPC mappings to close.
struct PeerSync {
  unsigned* flags = nullptr;  // P
  int* err = nullptr;
  PeerFlags pf{};
  unsigned epoch = 0;
  std::vector<void*> opened;

  cudaError_t init(int P) {
    cudaError_t e;
    if ((e = cudaMalloc(&flags, sizeof(unsigned) * size_t(P))) != cudaSuccess) return e;
    if ((e = cudaMemset(flags, 0, sizeof(unsigned) * size_t(P))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&err, sizeof(int))) != cudaSuccess) return e;
    return cudaMemset(err, 0, sizeof(int));
  }
  void release() {
    for (void* p : opened) cudaIpcCloseMemHandle(p);
    opened.clear();
    if (flags) cudaFree(flags);
    if (err) cudaFree(err);
    flags = nullptr;
    err = nullptr;
  }
  // Handles of `bufs` and of the flags, in that order.
  arena_status export_handles(const std::vector<void*>& bufs, void* out) const {
    std::vector<cudaIpcMemHandle_t> h(bufs.size() + 1);
    for (size_t k = 0; k <= bufs.size(); ++k) {
      cudaError_t e = cudaIpcGetMemHandle(&h[k], k < bufs.size() ? bufs[k] : static_cast<void*>(flags));
      if (e != cudaSuccess) return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    memcpy(out, h.data(), h.size() * sizeof(cudaIpcMemHandle_t));
    return ARENA_OK;
  }
  // ptrs[d][k]: buffer k of rank d (own buffers for d == rank); flag arrays into pf.
  arena_status attach(const void* all, int P, int rank, const std::vector<void*>& mine,
                      std::vector<std::vector<void*>>& ptrs) {
    const size_t nb = mine.size() + 1, hb = nb * sizeof(cudaIpcMemHandle_t);
    ptrs.assign(P, mine);
    for (int d = 0; d < P; ++d) {
      void* fl = flags;
      if (d != rank) {
        std::vector<cudaIpcMemHandle_t> h(nb);
        memcpy(h.data(), static_cast<const char*>(all) + size_t(d) * hb, hb);
        for (size_t k = 0; k < nb; ++k) {
          void* ptr = nullptr;
          cudaError_t e = cudaIpcOpenMemHandle(&ptr, h[k], cudaIpcMemLazyEnablePeerAccess);
          if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
          opened.push_back(ptr);
          if (k < mine.size()) ptrs[d][k] = ptr;
          else fl = ptr;
        }
      }
      pf.peer[d] = static_cast<unsigned*>(fl);
    }
    pf.mine = flags;
    return ARENA_OK;
  }
  arena_status barrier(cudaStream_t st, int rank, int P) {
    ++epoch;
    k_peer_barrier<<<1, 32, 0, st>>>(pf, rank, P, epoch, err);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? ARENA_OK : cuda_fail(e, "peer barrier");
  }
  arena_status status() const {
    int h = 0;
    cudaError_t e = cudaMemcpy(&h, err, sizeof h, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_fail(e, "barrier status");
    return h ? fail(ARENA_ECUDA, "peer barrier timed out (a rank did not arrive within 20 s)") : ARENA_OK;
  }
};

}  // namespace

struct arena_fft_slab {
  arena_fft_plan* base = nullptr;  // twiddles, stage tables, device, precision (no workspace)
  int n = 0, P = 1, rank = 0, loopback = 0;
  int ni = 0, nj = 0;
  size_t chunk_elems = 0;  // reals per exchange chunk
  size_t ws_bytes = 0;     // bytes of one workspace (B or C)
  std::vector<SlabRank> ranks;  // loopback: P virtual ranks; NCCL: this rank only
  ncclComm_t comm = nullptr;
  int xmode = ARENA_XCHG_COPY;  // ARENA_XCHG_PEER: K2 / K3 store into the peers' workspaces
  bool attached = false;        // peer pointers of the other ranks opened (multi-process)
  PeerSync sync;
  // Chunked COPY exchange (NCCL or loopback copies): the all-to-alls run on comm_st in
  // sub-steps, each gated by an event after the kernels that produced its rows, so
  // exchange s overlaps the transform of sub-range s + 1.
  int chunk_fwd = 1, chunk_bwd = 1;  // sub-steps per direction (1 = the whole chunk at once)
  cudaStream_t comm_st = nullptr;
  std::vector<cudaEvent_t> xev;      // chunk_fwd + chunk_bwd + 2 ordering events
  bool aborted = false;              // NCCL communicator aborted after an error / timeout
  // stage timing (arena_slab_set_stage_timing): kSlabMarks events per solve
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  int ev_sets = 0;
  double stage_ms[5] = {0, 0, 0, 0, 0};
  int solves = 0;
};

namespace {

constexpr int kSlabMarks = 6;  // K1+K2 | exchange #1 | K3 | exchange #2 | K4+K5

void free_slab(arena_fft_slab* s) {
  if (!s) return;
  if (s->base) {
    DeviceGuard g(s->base->device);
    for (cudaEvent_t e : s->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : s->xev) cudaEventDestroy(e);
    if (s->comm_st) cudaStreamDestroy(s->comm_st);
    s->sync.release();
    for (SlabRank& r : s->ranks) {
      if (r.B) cudaFree(r.B);
      if (r.C) cudaFree(r.C);
      if (r.ctrs) cudaFree(r.ctrs);
    }
    if (s->comm && !s->aborted) {
      if (NcclApi* a = nccl_api()) a->CommDestroy(s->comm);
    }
  }
  free_plan(s->base);
  delete s;
}

arena_status slab_init(arena_fft_slab** out, int n, int prec, int device, int P, int rank, int loopback,
                       const void* id) {
  if (!out) return fail(ARENA_EINVAL, "slab pointer is NULL");
  *out = nullptr;
  if (P < 1 || rank < 0 || rank >= P) return fail(ARENA_EINVAL, "bad rank / size");
  if (!is_pow2(n) || n > kPow2MaxN || n < 4) return fail(ARENA_EUNSUPPORTED, "slab path needs power-of-two 4 <= n <= 2048");
  if ((P & (P - 1)) || P > n) return fail(ARENA_EUNSUPPORTED, "slab count must be a power of two <= n");
  arena_fft_slab* s = new (std::nothrow) arena_fft_slab;
  if (!s) return fail(ARENA_ENOMEM, "slab");
  arena_status st = create_plan(&s->base, n, prec, device, false);
  if (st != ARENA_OK) {
    delete s;
    return st;
  }
  if (!s->base->tma) {
    free_slab(s);
    return fail(ARENA_EUNSUPPORTED, "slab path needs the TMA kernels (unset ARENA_FFT_KERNELS)");
  }
  DeviceGuard g(s->base->device);
  s->n = n;
  s->P = P;
  s->rank = rank;
  s->loopback = loopback;
  s->ni = n / P;
  s->nj = n / P;
  const size_t ncp = size_t(s->base->ncp);
  s->chunk_elems = size_t(s->ni) * s->nj * ncp * 2;
  s->ws_bytes = size_t(s->ni) * n * ncp * 2 * s->base->elem;
  s->ranks.resize(loopback ? P : 1);
  for (SlabRank& r : s->ranks) {
    cudaError_t e;
    if ((e = cudaMalloc(&r.B, s->ws_bytes)) != cudaSuccess || (e = cudaMalloc(&r.C, s->ws_bytes)) != cudaSuccess) {
      free_slab(s);
      return fail(ARENA_ENOMEM, "slab workspaces: " + std::string(cudaGetErrorString(e)));
    }
    if (s->base->ctrs && (e = cudaMalloc(&r.ctrs, sizeof(int) * size_t(s->ni + 1))) != cudaSuccess) {
      free_slab(s);
      return fail(ARENA_ENOMEM, "slab counters");
    }
  }
  if (cudaError_t e = s->sync.init(P)) {
    free_slab(s);
    return fail(ARENA_ENOMEM, "slab barrier flags: " + std::string(cudaGetErrorString(e)));
  }
  if (!loopback && id) {
    NcclApi* a = nccl_api();
    if (!a) {
      free_slab(s);
      return fail(ARENA_ENCCL, "libnccl.so.2 not found");
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclResult_t r = a->CommInitRank(&s->comm, P, uid, rank);
    if (r != ncclSuccess) {
      s->comm = nullptr;
      free_slab(s);
      return nccl_fail(r, "ncclCommInitRank");
    }
  }
  {
    // Chunked COPY exchange: ARENA_SLAB_CHUNKS sub-steps per all-to-all (default 4; 1 = whole
    // chunks after whole passes).  Forward sub-steps split the rank's i planes; backward ones
    // whole JB blocks of its j lines (the rows of a layout-C chunk are contiguous per block).
    int want = 4;
    if (const char* c = std::getenv("ARENA_SLAB_CHUNKS")) want = std::max(1, std::atoi(c));
    const int JB = layout_jb(s->nj);
    s->chunk_fwd = std::min(want, s->ni);
    s->chunk_bwd = std::min(want, s->nj / JB);
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&s->comm_st, cudaStreamNonBlocking)) != cudaSuccess) {
      free_slab(s);
      return cuda_fail(e, "slab exchange stream");
    }
    s->xev.resize(size_t(s->ni + s->nj / JB + 2), nullptr);  // enough for any chunking
    for (cudaEvent_t& x : s->xev)
      if ((e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming)) != cudaSuccess) {
        free_slab(s);
        return cuda_fail(e, "slab exchange events");
      }
  }
  *out = s;
  return ARENA_OK;
}

Pow2Args slab_args(arena_fft_slab* s, SlabRank& r, int rank, const void* f, void* u, cudaStream_t st, int phases) {
  arena_fft_plan* p = s->base;
  return Pow2Args{f, u, r.B, p->tw, p->stw, p->n, p->nc, p->ncp, st, nullptr, &r.tma, p->sm_count,
                  s->ni, s->nj, s->P, rank * s->nj, r.C, phases, r.ctrs, p->lag, p->fuse};
}

cudaError_t slab_phase(arena_fft_slab* s, SlabRank& r, int rank, const void* f, void* u, cudaStream_t st, int phases,
                       int sub0 = 0, int subn = 0) {
  Pow2Args a = slab_args(s, r, rank, f, u, st, phases);
  a.sub0 = sub0;
  a.subn = subn;
  if (s->xmode == ARENA_XCHG_PEER) {
    a.peer_y = r.peerC;
    a.peer_x = r.peerB;
  }
  return s->base->prec == 64 ? launch_pow2_f64(a) : launch_pow2_f32(a);
}

// Loopback ranks in peer mode: rank v's tables point at the virtual ranks' buffers.
void slab_fill_loopback_peers(arena_fft_slab* s) {
  const size_t cb = s->chunk_elems * s->base->elem;
  for (int v = 0; v < s->P; ++v)
    for (int d = 0; d < s->P; ++d) {
      s->ranks[v].peerC[d] = static_cast<char*>(s->ranks[d].C) + size_t(v) * cb;
      s->ranks[v].peerB[d] = static_cast<char*>(s->ranks[d].B) + size_t(v) * cb;
    }
}

arena_status slab_peer_barrier(arena_fft_slab* s, cudaStream_t st) { return s->sync.barrier(st, s->rank, s->P); }

// In-chunk row ranges {first row, rows} that sub-step [lo, hi) of an exchange moves:
// forward — local i planes [lo, hi) of a layout-B chunk, one range per JB block of j
// (row (jb ni + il) JB + jl % JB); backward — local j lines [lo, hi) (whole JB blocks) of
// a layout-C chunk, one contiguous range.  Chunk d of B and chunk r of C share the
// in-chunk order, so the same ranges serve the sender and the receiver.
void slab_piece_rows(int ni, int nj, bool forward, int lo, int hi, std::vector<std::pair<size_t, size_t>>& out) {
  const int JB = layout_jb(nj);
  out.clear();
  if (forward) {
    for (int jb = 0; jb < nj / JB; ++jb) out.emplace_back((size_t(jb) * ni + lo) * JB, size_t(hi - lo) * JB);
  } else {
    out.emplace_back(size_t(lo / JB) * ni * JB, size_t((hi - lo) / JB) * ni * JB);
  }
}

// One sub-step of a chunked exchange on stream st (every rank's rows [lo, hi)).
arena_status slab_exchange_sub(arena_fft_slab* s, cudaStream_t st, bool forward, int lo, int hi) {
  std::vector<std::pair<size_t, size_t>> pcs;
  slab_piece_rows(s->ni, s->nj, forward, lo, hi, pcs);
  const size_t rowb = size_t(s->base->ncp) * 2 * s->base->elem;
  const size_t chunk_rows = size_t(s->ni) * s->nj;
  if (s->loopback) {
    for (int r = 0; r < s->P; ++r)
      for (int d = 0; d < s->P; ++d) {
        const char* src = static_cast<const char*>(forward ? s->ranks[r].B : s->ranks[r].C) + d * chunk_rows * rowb;
        char* dst = static_cast<char*>(forward ? s->ranks[d].C : s->ranks[d].B) + r * chunk_rows * rowb;
        for (const auto& pc : pcs) {
          cudaError_t e = cudaMemcpyAsync(dst + pc.first * rowb, src + pc.first * rowb, pc.second * rowb,
                                          cudaMemcpyDeviceToDevice, st);
          if (e != cudaSuccess) return cuda_fail(e, "loopback exchange");
        }
      }
    return ARENA_OK;
  }
  NcclApi* a = nccl_api();
  if (s->aborted) return fail(ARENA_ENCCL, "the slab's NCCL communicator was aborted");
  const ncclDataType_t dt = s->base->prec == 64 ? ncclFloat64 : ncclFloat32;
  const size_t elems_per_row = size_t(s->base->ncp) * 2;
  SlabRank& me = s->ranks[0];
  const char* src = static_cast<const char*>(forward ? me.B : me.C);
  char* dst = static_cast<char*>(forward ? me.C : me.B);
  ncclResult_t res = a->GroupStart();
  if (res != ncclSuccess) return nccl_fail(res, "ncclGroupStart");
  for (int d = 0; d < s->P; ++d)
    for (const auto& pc : pcs) {
      const size_t off = (d * chunk_rows + pc.first) * rowb;
      if ((res = a->Send(src + off, pc.second * elems_per_row, dt, d, s->comm, st)) != ncclSuccess)
        return nccl_fail(res, "ncclSend");
      if ((res = a->Recv(dst + off, pc.second * elems_per_row, dt, d, s->comm, st)) != ncclSuccess)
        return nccl_fail(res, "ncclRecv");
    }
  if ((res = a->GroupEnd()) != ncclSuccess) return nccl_fail(res, "ncclGroupEnd");
  return ARENA_OK;
}

// All-to-all between workspaces: forward (B chunk d of rank r -> C chunk r of rank d)
// or backward (C chunk d of rank r -> B chunk r of rank d).
arena_status slab_exchange(arena_fft_slab* s, cudaStream_t st, bool forward) {
  const size_t bytes = s->chunk_elems * s->base->elem;
  if (s->loopback) {
    for (int r = 0; r < s->P; ++r)
      for (int d = 0; d < s->P; ++d) {
        const char* src = static_cast<const char*>(forward ? s->ranks[r].B : s->ranks[r].C) + size_t(d) * bytes;
        char* dst = static_cast<char*>(forward ? s->ranks[d].C : s->ranks[d].B) + size_t(r) * bytes;
        cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "loopback exchange");
      }
    return ARENA_OK;
  }
  NcclApi* a = nccl_api();
  const ncclDataType_t dt = s->base->prec == 64 ? ncclFloat64 : ncclFloat32;
  SlabRank& me = s->ranks[0];
  const char* src = static_cast<const char*>(forward ? me.B : me.C);
  char* dst = static_cast<char*>(forward ? me.C : me.B);
  ncclResult_t res = a->GroupStart();
  if (res != ncclSuccess) return nccl_fail(res, "ncclGroupStart");
  for (int d = 0; d < s->P; ++d) {
    if ((res = a->Send(src + size_t(d) * bytes, s->chunk_elems, dt, d, s->comm, st)) != ncclSuccess)
      return nccl_fail(res, "ncclSend");
    if ((res = a->Recv(dst + size_t(d) * bytes, s->chunk_elems, dt, d, s->comm, st)) != ncclSuccess)
      return nccl_fail(res, "ncclRecv");
  }
  if ((res = a->GroupEnd()) != ncclSuccess) return nccl_fail(res, "ncclGroupEnd");
  return ARENA_OK;
}

}  // namespace

extern "C" {

arena_status arena_nccl_unique_id(void* out, int len) {
  if (!out || len < int(sizeof(ncclUniqueId))) return fail(ARENA_EINVAL, "unique id buffer too small");
  NcclApi* a = nccl_api();
  if (!a) return fail(ARENA_ENCCL, "libnccl.so.2 not found");
  ncclUniqueId uid;
  ncclResult_t r = a->GetUniqueId(&uid);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(out, &uid, sizeof uid);
  return ARENA_OK;
}

int arena_nccl_unique_id_bytes(void) { return int(sizeof(ncclUniqueId)); }

arena_status arena_slab_create(arena_fft_slab** out, int n, int precision_bits, int device, int nranks, int rank,
                               const void* nccl_id) {
  if (!nccl_id) return fail(ARENA_EINVAL, "NCCL unique id is NULL");
  return slab_init(out, n, precision_bits, device, nranks, rank, 0, nccl_id);
}

arena_status arena_slab_create_loopback(arena_fft_slab** out, int n, int precision_bits, int device, int nvranks) {
  return slab_init(out, n, precision_bits, device, nvranks, 0, 1, nullptr);
}

void arena_slab_destroy(arena_fft_slab* s) { free_slab(s); }

int arena_slab_launches_per_solve(const arena_fft_slab* s) {
  if (!s) return 0;
  const bool barrier = s->xmode == ARENA_XCHG_PEER && !s->loopback && s->P > 1;
  return s->base->launches() * int(s->ranks.size()) + (barrier ? 2 : 0);
}

arena_status arena_slab_info(const arena_fft_slab* s, int* ni, int* nj, size_t* chunk_bytes, size_t* workspace_bytes) {
  if (!s) return fail(ARENA_EINVAL, "slab is NULL");
  if (ni) *ni = s->ni;
  if (nj) *nj = s->nj;
  if (chunk_bytes) *chunk_bytes = s->chunk_elems * s->base->elem;
  if (workspace_bytes) *workspace_bytes = s->ws_bytes;
  return ARENA_OK;
}

// One third of a slab solve.  Phase 0: K1, K2 (+ exchange #1 unless the
// exchange is K2's own peer stores); 1: K3 (+ exchange #2); 2: K4, K5.  In peer
// mode every rank must have finished phase p before any rank starts phase p+1
// (arena_slab_solve_device inserts a device barrier; a caller driving the
// phases itself synchronises the ranks between them).
static arena_status slab_run_kernels(arena_fft_slab* s, int phase, const void* d_f, void* d_u, cudaStream_t st) {
  static const int kPh[3] = {kPhaseZY, kPhaseX, kPhaseYZ};
  static const char* kWhat[3] = {"slab K1+K2", "slab K3", "slab K4+K5"};
  if (phase < 0 || phase > 2) return fail(ARENA_EINVAL, "slab phase must be 0, 1 or 2");
  if (s->xmode == ARENA_XCHG_PEER && !s->loopback && !s->attached)
    return fail(ARENA_EINVAL, "peer exchange: call arena_slab_peer_attach first");
  const size_t slab_bytes = size_t(s->ni) * s->n * s->n * s->base->elem;
  const int nr = int(s->ranks.size());
  for (int v = 0; v < nr; ++v) {
    const int rank = s->loopback ? v : s->rank;
    const char* f = static_cast<const char*>(d_f) + (s->loopback ? size_t(v) * slab_bytes : 0);
    char* u = static_cast<char*>(d_u) + (s->loopback ? size_t(v) * slab_bytes : 0);
    cudaError_t e = slab_phase(s, s->ranks[v], rank, f, u, st, kPh[phase]);
    if (e != cudaSuccess) return cuda_fail(e, kWhat[phase]);
  }
  return ARENA_OK;
}

static arena_status slab_run_phase(arena_fft_slab* s, int phase, const void* d_f, void* d_u, cudaStream_t st) {
  arena_status stt = slab_run_kernels(s, phase, d_f, d_u, st);
  if (stt != ARENA_OK) return stt;
  if (phase < 2 && s->xmode != ARENA_XCHG_PEER) return slab_exchange(s, st, phase == 0);
  return ARENA_OK;
}

// Events of one timed solve (kSlabMarks), recycled by arena_slab_stage_times.
static cudaEvent_t* slab_timing_events(arena_fft_slab* s) {
  if (!s->timing) return nullptr;
  const size_t need = size_t(s->ev_sets + 1) * kSlabMarks;
  while (s->ev_pool.size() < need) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    s->ev_pool.push_back(e);
  }
  return s->ev_pool.data() + size_t(s->ev_sets++) * kSlabMarks;
}

// Kernels of one phase over every (virtual) rank, restricted to a sub-range when subn > 0.
static arena_status slab_kernels_sub(arena_fft_slab* s, int phases, int sub0, int subn, const void* d_f, void* d_u,
                                     cudaStream_t st) {
  const size_t slab_bytes = size_t(s->ni) * s->n * s->n * s->base->elem;
  for (int v = 0; v < int(s->ranks.size()); ++v) {
    const int rank = s->loopback ? v : s->rank;
    const char* f = static_cast<const char*>(d_f) + (s->loopback ? size_t(v) * slab_bytes : 0);
    char* u = static_cast<char*>(d_u) + (s->loopback ? size_t(v) * slab_bytes : 0);
    cudaError_t e = slab_phase(s, s->ranks[v], rank, f, u, st, phases, sub0, subn);
    if (e != cudaSuccess) return cuda_fail(e, "slab sub-range kernels");
  }
  return ARENA_OK;
}

// COPY exchange, chunked: the transform of sub-range k+1 overlaps the all-to-all of
// sub-range k, which runs on the slab's exchange stream gated by an event.
static arena_status slab_solve_chunked(arena_fft_slab* s, const void* d_f, void* d_u, cudaStream_t st,
                                       cudaEvent_t* ev) {
  const int cf = s->chunk_fwd, cb = s->chunk_bwd;
  const int JB = layout_jb(s->nj), nb = s->nj / JB;
  cudaEvent_t* x = s->xev.data();
  arena_status stt;
  if (ev) cudaEventRecord(ev[0], st);
  for (int k = 0; k < cf; ++k) {
    const int lo = k * s->ni / cf, hi = (k + 1) * s->ni / cf;
    if ((stt = slab_kernels_sub(s, kPhaseZY, lo, hi - lo, d_f, d_u, st)) != ARENA_OK) return stt;
    cudaEventRecord(x[k], st);
    cudaStreamWaitEvent(s->comm_st, x[k], 0);
    if ((stt = slab_exchange_sub(s, s->comm_st, true, lo, hi)) != ARENA_OK) return stt;
  }
  if (ev) cudaEventRecord(ev[1], st);
  cudaEventRecord(x[cf + cb], s->comm_st);
  cudaStreamWaitEvent(st, x[cf + cb], 0);
  if (ev) cudaEventRecord(ev[2], st);
  for (int k = 0; k < cb; ++k) {
    const int lo = (k * nb / cb) * JB, hi = ((k + 1) * nb / cb) * JB;
    if ((stt = slab_kernels_sub(s, kPhaseX, lo, hi - lo, d_f, d_u, st)) != ARENA_OK) return stt;
    cudaEventRecord(x[cf + k], st);
    cudaStreamWaitEvent(s->comm_st, x[cf + k], 0);
    if ((stt = slab_exchange_sub(s, s->comm_st, false, lo, hi)) != ARENA_OK) return stt;
  }
  if (ev) cudaEventRecord(ev[3], st);
  cudaEventRecord(x[cf + cb + 1], s->comm_st);
  cudaStreamWaitEvent(st, x[cf + cb + 1], 0);
  if (ev) cudaEventRecord(ev[4], st);
  if ((stt = slab_run_kernels(s, 2, d_f, d_u, st)) != ARENA_OK) return stt;
  if (ev) cudaEventRecord(ev[5], st);
  return ARENA_OK;
}

arena_status arena_slab_solve_device(arena_fft_slab* s, const void* d_f, void* d_u, void* stream) {
  if (!s || !d_f || !d_u) return fail(ARENA_EINVAL, "NULL slab or buffer");
  DeviceGuard g(s->base->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool barrier = s->xmode == ARENA_XCHG_PEER && !s->loopback && s->P > 1;
  cudaEvent_t* ev = slab_timing_events(s);
  if (s->xmode != ARENA_XCHG_PEER && (s->chunk_fwd > 1 || s->chunk_bwd > 1) && !s->base->ctrs)
    return slab_solve_chunked(s, d_f, d_u, st, ev);
  for (int phase = 0; phase < 3; ++phase) {
    if (ev) cudaEventRecord(ev[2 * phase], st);
    arena_status stt = slab_run_kernels(s, phase, d_f, d_u, st);
    if (stt != ARENA_OK) return stt;
    if (ev) cudaEventRecord(ev[2 * phase + 1], st);
    if (phase == 2) break;
    if (s->xmode != ARENA_XCHG_PEER) stt = slab_exchange(s, st, phase == 0);
    else if (barrier) stt = slab_peer_barrier(s, st);
    if (stt != ARENA_OK) return stt;
  }
  return ARENA_OK;
}

arena_status arena_slab_set_chunking(arena_fft_slab* s, int fwd, int bwd) {
  if (!s || fwd < 1 || bwd < 1) return fail(ARENA_EINVAL, "bad slab chunking");
  const int JB = layout_jb(s->nj);
  if (fwd > s->ni || bwd > s->nj / JB) return fail(ARENA_EINVAL, "more sub-steps than the slab has planes / j blocks");
  s->chunk_fwd = fwd;
  s->chunk_bwd = bwd;
  return ARENA_OK;
}

arena_status arena_slab_get_chunking(const arena_fft_slab* s, int* fwd, int* bwd) {
  if (!s) return fail(ARENA_EINVAL, "slab is NULL");
  if (fwd) *fwd = s->chunk_fwd;
  if (bwd) *bwd = s->chunk_bwd;
  return ARENA_OK;
}

int arena_slab_exchange_pieces(int n, int nranks, int forward, int lo, int hi, size_t* first, size_t* rows, int max) {
  if (n < 4 || nranks < 1 || n % nranks) return -1;
  const int ni = n / nranks, nj = n / nranks;
  const int JB = layout_jb(nj);
  const int lim = forward ? ni : nj;
  if (lo < 0 || hi > lim || lo >= hi || (!forward && (lo % JB || hi % JB))) return -1;
  std::vector<std::pair<size_t, size_t>> pcs;
  slab_piece_rows(ni, nj, forward != 0, lo, hi, pcs);
  for (int k = 0; k < int(pcs.size()) && k < max; ++k) {
    if (first) first[k] = pcs[k].first;
    if (rows) rows[k] = pcs[k].second;
  }
  return int(pcs.size());
}

// Wait for a solve enqueued on `stream` (and the slab's exchange stream) with NCCL
// error / hang detection: polls ncclCommGetAsyncError and aborts the communicator
// after timeout_s, instead of blocking forever on a stuck peer.
arena_status arena_slab_wait(arena_fft_slab* s, void* stream, double timeout_s) {
  if (!s) return fail(ARENA_EINVAL, "slab is NULL");
  DeviceGuard g(s->base->device);
  NcclApi* a = s->comm ? nccl_api() : nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    cudaError_t q1 = cudaStreamQuery(static_cast<cudaStream_t>(stream));
    cudaError_t q2 = s->comm_st ? cudaStreamQuery(s->comm_st) : cudaSuccess;
    if (q1 == cudaSuccess && q2 == cudaSuccess) break;
    if (q1 != cudaSuccess && q1 != cudaErrorNotReady) return cuda_fail(q1, "slab solve");
    if (q2 != cudaSuccess && q2 != cudaErrorNotReady) return cuda_fail(q2, "slab exchange");
    if (a && a->CommGetAsyncError && !s->aborted) {
      ncclResult_t r = ncclSuccess;
      if (a->CommGetAsyncError(s->comm, &r) == ncclSuccess && r != ncclSuccess && r != ncclInProgress) {
        if (a->CommAbort) a->CommAbort(s->comm);
        s->aborted = true;
        return nccl_fail(r, "NCCL asynchronous error (communicator aborted)");
      }
    }
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > timeout_s) {
      if (a && a->CommAbort && !s->aborted) {
        a->CommAbort(s->comm);
        s->aborted = true;
      }
      return fail(ARENA_ENCCL, "slab solve did not complete within " + std::to_string(timeout_s) +
                                   " s (a peer is stuck or gone); NCCL communicator aborted");
    }
    std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
  if (s->xmode == ARENA_XCHG_PEER && !s->loopback) return s->sync.status();
  return ARENA_OK;
}

arena_status arena_slab_set_stage_timing(arena_fft_slab* s, int enable) {
  if (!s) return fail(ARENA_EINVAL, "slab is NULL");
  s->timing = enable != 0;
  s->ev_sets = 0;
  for (double& x : s->stage_ms) x = 0.0;
  s->solves = 0;
  return ARENA_OK;
}

arena_status arena_slab_stage_times(arena_fft_slab* s, double* ms5, int* n_solves) {
  if (!s) return fail(ARENA_EINVAL, "slab is NULL");
  DeviceGuard g(s->base->device);
  for (int k = 0; k < s->ev_sets; ++k) {
    cudaEvent_t* ev = s->ev_pool.data() + size_t(k) * kSlabMarks;
    cudaError_t e = cudaEventSynchronize(ev[kSlabMarks - 1]);
    if (e != cudaSuccess) return cuda_fail(e, "slab stage timing sync");
    for (int m = 0; m + 1 < kSlabMarks; ++m) {
      float t = 0.f;
      if ((e = cudaEventElapsedTime(&t, ev[m], ev[m + 1])) != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
      s->stage_ms[m] += t;
    }
    ++s->solves;
  }
  s->ev_sets = 0;
  if (ms5)
    for (int m = 0; m < 5; ++m) ms5[m] = s->stage_ms[m];
  if (n_solves) *n_solves = s->solves;
  return ARENA_OK;
}

arena_status arena_slab_solve_phase(arena_fft_slab* s, int phase, const void* d_f, void* d_u, void* stream) {
  if (!s || !d_f || !d_u) return fail(ARENA_EINVAL, "NULL slab or buffer");
  DeviceGuard g(s->base->device);
  return slab_run_phase(s, phase, d_f, d_u, static_cast<cudaStream_t>(stream));
}

arena_status arena_slab_create_peer(arena_fft_slab** out, int n, int precision_bits, int device, int nranks,
                                    int rank) {
  if (nranks > kMaxPeers) return fail(ARENA_EUNSUPPORTED, "peer exchange supports at most 8 ranks");
  arena_status st = slab_init(out, n, precision_bits, device, nranks, rank, 0, nullptr);
  if (st == ARENA_OK) (*out)->xmode = ARENA_XCHG_PEER;
  return st;
}

int arena_slab_peer_handle_bytes(void) { return int(3 * sizeof(cudaIpcMemHandle_t)); }

arena_status arena_slab_peer_export(arena_fft_slab* s, void* out, int len) {
  if (!s || !out || len < arena_slab_peer_handle_bytes()) return fail(ARENA_EINVAL, "handle buffer too small");
  if (s->loopback) return fail(ARENA_EINVAL, "loopback slabs have no peers to export to");
  DeviceGuard g(s->base->device);
  return s->sync.export_handles({s->ranks[0].B, s->ranks[0].C}, out);
}

arena_status arena_slab_peer_attach(arena_fft_slab* s, const void* all, int len) {
  const int hb = arena_slab_peer_handle_bytes();
  if (!s || !all || len < hb * (s ? s->P : 0)) return fail(ARENA_EINVAL, "need every rank's handles");
  if (s->loopback) return fail(ARENA_EINVAL, "loopback slabs need no attach");
  if (s->P > kMaxPeers) return fail(ARENA_EUNSUPPORTED, "peer exchange supports at most 8 ranks");
  if (s->attached) return ARENA_OK;
  DeviceGuard g(s->base->device);
  SlabRank& me = s->ranks[0];
  std::vector<std::vector<void*>> ptrs;
  arena_status st = s->sync.attach(all, s->P, s->rank, {me.B, me.C}, ptrs);
  if (st != ARENA_OK) return st;
  const size_t cb = s->chunk_elems * s->base->elem;
  for (int d = 0; d < s->P; ++d) {
    me.peerB[d] = static_cast<char*>(ptrs[d][0]) + size_t(s->rank) * cb;
    me.peerC[d] = static_cast<char*>(ptrs[d][1]) + size_t(s->rank) * cb;
  }
  s->attached = true;
  s->xmode = ARENA_XCHG_PEER;
  return ARENA_OK;
}

arena_status arena_slab_set_exchange(arena_fft_slab* s, int mode) {
  if (!s) return fail(ARENA_EINVAL, "slab is NULL");
  if (mode == ARENA_XCHG_COPY) {
    if (!s->loopback && !s->comm) return fail(ARENA_EINVAL, "this slab has no NCCL communicator");
    s->xmode = mode;
    return ARENA_OK;
  }
  if (mode != ARENA_XCHG_PEER) return fail(ARENA_EINVAL, "unknown exchange mode");
  if (s->P > kMaxPeers) return fail(ARENA_EUNSUPPORTED, "peer exchange supports at most 8 ranks");
  if (s->loopback) {
    slab_fill_loopback_peers(s);
  } else if (!s->attached) {
    return fail(ARENA_EINVAL, "peer exchange: call arena_slab_peer_attach first");
  }
  s->xmode = mode;
  return ARENA_OK;
}

arena_status arena_slab_barrier_status(arena_fft_slab* s) {
  if (!s) return fail(ARENA_EINVAL, "slab is NULL");
  DeviceGuard g(s->base->device);
  return s->sync.status();
}

arena_status arena_peer_barrier_selftest(int device, int nranks, int rounds, int* bad) {
  if (nranks < 1 || nranks > kMaxPeers || rounds < 1 || !bad) return fail(ARENA_EINVAL, "bad self-test arguments");
  DeviceGuard g(device);
  unsigned* flags = nullptr;
  int *data = nullptr, *err = nullptr, *dbad = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&flags, sizeof(unsigned) * nranks * nranks)) != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  cudaMalloc(&data, sizeof(int) * nranks);
  cudaMalloc(&err, sizeof(int));
  cudaMalloc(&dbad, sizeof(int));
  cudaMemset(flags, 0, sizeof(unsigned) * nranks * nranks);
  cudaMemset(data, 0, sizeof(int) * nranks);
  cudaMemset(err, 0, sizeof(int));
  cudaMemset(dbad, 0, sizeof(int));
  volatile int* vdata = data;
  void* args[] = {&flags, (void*)&vdata, &nranks, &rounds, &err, &dbad};
  e = cudaLaunchCooperativeKernel((const void*)k_peer_barrier_selftest, dim3(nranks), dim3(32), args, 0, nullptr);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  int herr = 0;
  if (e == cudaSuccess) e = cudaMemcpy(bad, dbad, sizeof(int), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(&herr, err, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(flags);
  cudaFree(data);
  cudaFree(err);
  cudaFree(dbad);
  if (e != cudaSuccess) return cuda_fail(e, "barrier self-test");
  return herr ? fail(ARENA_ECUDA, "barrier self-test timed out") : ARENA_OK;
}

}  // extern "C"

// ============================================================================
// One process, P GPUs (the drop-in's multi-GPU path, ARENA_FFT_NGPU): rank v = a
// slab rank on devices[v] holding planes [v n/P, (v+1) n/P).  Its K2 / K3 store the
// exchange chunks straight into the other ranks' workspaces through peer access
// (cudaDeviceEnablePeerAccess: NVLink on a B200 box), exactly the peer-exchange
// kernels of the multi-process slab, and the phases are ordered by cross-device
// events instead of a device flag barrier (all ranks' streams belong to this
// process).  The host path moves the P slabs of a GridField over P PCIe links in
// parallel (one host thread and one staging ring per GPU).
struct arena_fft_mgpu {
  int n = 0, P = 1, prec = 64;
  size_t elem = 8, slab_bytes = 0;
  std::vector<int> dev;
  std::vector<arena_fft_slab*> sl;
  std::vector<cudaStream_t> st;
  std::vector<cudaEvent_t> ev;  // 2 * P: after phase 0 / 1 of each rank
  std::vector<void*> fbuf;      // host path: each rank's real slab (solved in place)
  std::vector<Stager*> stg;
  std::mutex mu;
};

namespace {

void free_mgpu(arena_fft_mgpu* m) {
  if (!m) return;
  for (int v = 0; v < int(m->sl.size()); ++v) {
    DeviceGuard g(m->dev[v]);
    if (v < int(m->fbuf.size()) && m->fbuf[v]) cudaFree(m->fbuf[v]);
    if (v < int(m->stg.size())) delete m->stg[v];
    if (v < int(m->st.size()) && m->st[v]) cudaStreamDestroy(m->st[v]);
    for (int ph = 0; ph < 2; ++ph) {
      const size_t k = size_t(ph) * m->P + v;
      if (k < m->ev.size() && m->ev[k]) cudaEventDestroy(m->ev[k]);
    }
    m->sl[v]->attached = false;  // peer pointers are plain device pointers here: nothing to close
    free_slab(m->sl[v]);
  }
  delete m;
}

arena_status mgpu_enqueue(arena_fft_mgpu* m, const void* const* f, void* const* u, const cudaStream_t* st) {
  for (int phase = 0; phase < 3; ++phase) {
    for (int v = 0; v < m->P; ++v) {
      DeviceGuard g(m->dev[v]);
      arena_status stt = slab_run_kernels(m->sl[v], phase, f[v], u[v], st[v]);
      if (stt != ARENA_OK) return stt;
      if (phase < 2 && cudaEventRecord(m->ev[size_t(phase) * m->P + v], st[v]) != cudaSuccess)
        return fail(ARENA_ECUDA, "multi-GPU phase event");
    }
    if (phase == 2) break;
    // every rank's next phase reads what every rank's previous phase stored into it
    for (int w = 0; w < m->P; ++w) {
      DeviceGuard g(m->dev[w]);
      for (int v = 0; v < m->P; ++v)
        if (cudaStreamWaitEvent(st[w], m->ev[size_t(phase) * m->P + v], 0) != cudaSuccess)
          return fail(ARENA_ECUDA, "multi-GPU cross-device wait");
    }
  }
  return ARENA_OK;
}

cudaError_t mgpu_copy(arena_fft_mgpu* m, int v, void* dst, const void* src, size_t bytes, bool to_host) {
  const void* host = to_host ? dst : src;
  if (host_ptr_pinned(host)) {
    cudaError_t e = cudaMemcpyAsync(dst, src, bytes, to_host ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice,
                                    m->st[v]);
    return (e || !to_host) ? e : cudaStreamSynchronize(m->st[v]);
  }
  if (!m->stg[v]) {
    m->stg[v] = new (std::nothrow) Stager;
    if (!m->stg[v]) return cudaErrorMemoryAllocation;
    cudaError_t e = m->stg[v]->init(std::max(2, 16 / m->P));
    if (e != cudaSuccess) {
      delete m->stg[v];
      m->stg[v] = nullptr;
      return e;
    }
  }
  return to_host ? m->stg[v]->d2h(dst, src, bytes, m->st[v]) : m->stg[v]->h2d(dst, src, bytes, m->st[v]);
}

}  // namespace

extern "C" {

arena_status arena_mgpu_create(arena_fft_mgpu** out, int n, int precision_bits, int nranks, const int* devices) {
  if (!out) return fail(ARENA_EINVAL, "multi-GPU pointer is NULL");
  *out = nullptr;
  if (nranks < 1 || nranks > kMaxPeers) return fail(ARENA_EUNSUPPORTED, "1 to 8 GPUs per process");
  if (!is_pow2(n) || n < 16 || n % nranks || n / nranks < 4)
    return fail(ARENA_EUNSUPPORTED, "multi-GPU path needs a power-of-two n >= 16 with n / P >= 4");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(ARENA_EUNSUPPORTED, "no CUDA device visible (this library has no CPU path)");
  arena_fft_mgpu* m = new (std::nothrow) arena_fft_mgpu;
  if (!m) return fail(ARENA_ENOMEM, "multi-GPU object");
  m->n = n;
  m->P = nranks;
  m->prec = precision_bits;
  m->elem = precision_bits == 64 ? 8 : 4;
  m->slab_bytes = size_t(n / nranks) * n * n * m->elem;
  for (int v = 0; v < nranks; ++v) m->dev.push_back(devices ? devices[v] : v % ndev);
  for (int v = 0; v < nranks; ++v) {
    if (m->dev[v] < 0 || m->dev[v] >= ndev) {
      free_mgpu(m);
      return fail(ARENA_EINVAL, "device ordinal out of range");
    }
    arena_fft_slab* s = nullptr;
    arena_status st = slab_init(&s, n, precision_bits, m->dev[v], nranks, v, 0, nullptr);
    if (st != ARENA_OK) {
      free_mgpu(m);
      return st;
    }
    m->sl.push_back(s);
  }
  // peer access between every pair of distinct devices
  for (int v = 0; v < nranks; ++v)
    for (int d = 0; d < nranks; ++d) {
      if (m->dev[v] == m->dev[d]) continue;
      DeviceGuard g(m->dev[v]);
      int can = 0;
      cudaDeviceCanAccessPeer(&can, m->dev[v], m->dev[d]);
      if (!can) {
        free_mgpu(m);
        return fail(ARENA_EUNSUPPORTED, "no peer access between devices " + std::to_string(m->dev[v]) + " and " +
                                            std::to_string(m->dev[d]));
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(m->dev[d], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        free_mgpu(m);
        return cuda_fail(e, "cudaDeviceEnablePeerAccess");
      }
    }
  const size_t cb = m->sl[0]->chunk_elems * m->elem;
  for (int v = 0; v < nranks; ++v) {
    SlabRank& me = m->sl[v]->ranks[0];
    for (int d = 0; d < nranks; ++d) {
      me.peerB[d] = static_cast<char*>(m->sl[d]->ranks[0].B) + size_t(v) * cb;
      me.peerC[d] = static_cast<char*>(m->sl[d]->ranks[0].C) + size_t(v) * cb;
    }
    m->sl[v]->attached = true;
    m->sl[v]->xmode = ARENA_XCHG_PEER;
  }
  m->st.assign(nranks, nullptr);
  m->ev.assign(size_t(2) * nranks, nullptr);
  m->fbuf.assign(nranks, nullptr);
  m->stg.assign(nranks, nullptr);
  for (int v = 0; v < nranks; ++v) {
    DeviceGuard g(m->dev[v]);
    cudaError_t e;
    if ((e = cudaStreamCreateWithFlags(&m->st[v], cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&m->ev[v], cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&m->ev[size_t(nranks) + v], cudaEventDisableTiming)) != cudaSuccess) {
      free_mgpu(m);
      return cuda_fail(e, "multi-GPU streams / events");
    }
  }
  *out = m;
  g_last_error.clear();
  return ARENA_OK;
}

void arena_mgpu_destroy(arena_fft_mgpu* m) { free_mgpu(m); }

arena_status arena_mgpu_info(const arena_fft_mgpu* m, int* nranks, int* devices, size_t* slab_bytes) {
  if (!m) return fail(ARENA_EINVAL, "multi-GPU object is NULL");
  if (nranks) *nranks = m->P;
  if (devices)
    for (int v = 0; v < m->P; ++v) devices[v] = m->dev[v];
  if (slab_bytes) *slab_bytes = m->slab_bytes;
  return ARENA_OK;
}

arena_status arena_mgpu_solve_device(arena_fft_mgpu* m, const void* const* f, void* const* u, void* const* streams) {
  if (!m || !f || !u) return fail(ARENA_EINVAL, "NULL multi-GPU object or shard list");
  for (int v = 0; v < m->P; ++v)
    if (!f[v] || !u[v]) return fail(ARENA_EINVAL, "NULL shard");
  std::lock_guard<std::mutex> lk(m->mu);
  std::vector<cudaStream_t> st(m->P);
  for (int v = 0; v < m->P; ++v) st[v] = streams ? static_cast<cudaStream_t>(streams[v]) : m->st[v];
  return mgpu_enqueue(m, f, u, st.data());
}

arena_status arena_mgpu_solve_host(arena_fft_mgpu* m, const void* f, void* u) {
  if (!m || !f || !u) return fail(ARENA_EINVAL, "NULL multi-GPU object or buffer");
  std::lock_guard<std::mutex> lk(m->mu);
  for (int v = 0; v < m->P; ++v) {
    if (m->fbuf[v]) continue;
    DeviceGuard g(m->dev[v]);
    if (cudaMalloc(&m->fbuf[v], m->slab_bytes) != cudaSuccess)
      return fail(ARENA_ENOMEM, "multi-GPU slab buffer (" + std::to_string(m->slab_bytes) + " B)");
  }
  // P slabs over P links at once: one host thread per GPU
  std::vector<cudaError_t> err(m->P, cudaSuccess);
  auto par = [&](bool to_host) {
    std::vector<std::thread> th;
    for (int v = 0; v < m->P; ++v)
      th.emplace_back([&, v] {
        cudaSetDevice(m->dev[v]);
        const size_t off = size_t(v) * m->slab_bytes;
        err[v] = to_host ? mgpu_copy(m, v, static_cast<char*>(u) + off, m->fbuf[v], m->slab_bytes, true)
                         : mgpu_copy(m, v, m->fbuf[v], static_cast<const char*>(f) + off, m->slab_bytes, false);
      });
    for (auto& t : th) t.join();
    for (cudaError_t e : err)
      if (e != cudaSuccess) return e;
    return cudaSuccess;
  };
  cudaError_t e = par(false);
  if (e != cudaSuccess) return cuda_fail(e, "multi-GPU H2D");
  std::vector<const void*> fs(m->fbuf.begin(), m->fbuf.end());
  arena_status st = mgpu_enqueue(m, fs.data(), m->fbuf.data(), m->st.data());
  if (st != ARENA_OK) return st;
  if ((e = par(true)) != cudaSuccess) return cuda_fail(e, "multi-GPU D2H");
  return ARENA_OK;
}

}  // extern "C"

// ============================================================================
// Pencil decomposition over Pr x Pc ranks (BASELINE config 5):
// rank (r, c) owns the f / u block i in [r n/Pr, ..), j in [c n/Pc, ..), all k.
//   K1 z-r2c, k split into Pc chunks (buf1 = R) -> row all-to-all (same r) ->
//   K2 y-fwd on (il, local k) lines over all j (buf2 = Y -> buf1 = B2, j re-chunked
//   by n/Pr) -> column all-to-all (same c) -> K3 on (local j, local k) lines over
//   all i (buf2 = C) -> the reverse.  Four all-to-alls per solve, as in the
//   paper's pencil scheme.  Row / column communicators come from
//   ncclCommSplit; the loopback mode runs all Pr*Pc ranks on one device.
namespace {

struct PencilRank {
  void* buf1 = nullptr;
  void* buf2 = nullptr;
  void* fblk = nullptr;  // loopback only: the rank's f / u blocks
  void* ublk = nullptr;
  TmaCache tma, tma2;
  // Peer exchange destinations (PencilArgs::pz ...), per row / column peer q.
  void* pz[kMaxPeers] = {};
  void* py1[kMaxPeers] = {};
  void* px[kMaxPeers] = {};
  void* py2[kMaxPeers] = {};
};

}  // namespace

struct arena_fft_pencil {
  arena_fft_plan* base = nullptr;
  int n = 0, Pr = 1, Pc = 1, rank = 0, loopback = 0, kq = 0;
  size_t buf_bytes = 0, blk_bytes = 0;
  std::vector<PencilRank> ranks;
  ncclComm_t world = nullptr, row = nullptr, col = nullptr;
  int xmode = ARENA_XCHG_COPY;
  bool attached = false;
  PeerSync sync;
  int fold = 0;  // ARENA_PENCIL_FOLDED (poisson_qpencil.cuh)
  // bytes of one exchange chunk (folded: of one quadrant's H problem, at the same offset in
  // each quadrant region)
  size_t row_chunk_bytes() const { return size_t(n / Pr) * (n / Pc) * kq * 2 * base->elem / (fold ? 4 : 1); }
  size_t col_chunk_bytes() const { return size_t(n / Pr) * (n / Pr) * kq * 2 * base->elem / (fold ? 4 : 1); }
};

namespace {

void free_pencil(arena_fft_pencil* s) {
  if (!s) return;
  if (s->base) {
    DeviceGuard g(s->base->device);
    for (PencilRank& r : s->ranks)
      for (void* p : {r.buf1, r.buf2, r.fblk})  // ublk aliases fblk
        if (p) cudaFree(p);
    s->sync.release();
    if (NcclApi* a = nccl_api()) {
      for (ncclComm_t c : {s->row, s->col, s->world})
        if (c) a->CommDestroy(c);
    }
  }
  free_plan(s->base);
  delete s;
}

arena_status pencil_init(arena_fft_pencil** out, int n, int prec, int device, int Pr, int Pc, int rank, int loopback,
                         const void* id) {
  if (!out) return fail(ARENA_EINVAL, "pencil pointer is NULL");
  *out = nullptr;
  if (Pr < 1 || Pc < 1 || (Pr & (Pr - 1)) || (Pc & (Pc - 1)) || Pr > n || Pc > n)
    return fail(ARENA_EINVAL, "process grid must be powers of two <= n");
  if (rank < 0 || rank >= Pr * Pc) return fail(ARENA_EINVAL, "bad rank");
  if (!is_pow2(n) || n < 64 || n > kPow2MaxN) return fail(ARENA_EUNSUPPORTED, "pencil path needs power-of-two 64 <= n <= 2048");
  const int ni = n / Pr, nj = n / Pc;
  arena_fft_pencil* s = new (std::nothrow) arena_fft_pencil;
  if (!s) return fail(ARENA_ENOMEM, "pencil");
  arena_status st = create_plan(&s->base, n, prec, device, false);
  if (st != ARENA_OK) {
    delete s;
    return st;
  }
  if (!s->base->tma) {
    free_pencil(s);
    return fail(ARENA_EUNSUPPORTED, "pencil path needs the TMA kernels (unset ARENA_FFT_KERNELS)");
  }
  DeviceGuard g(s->base->device);
  s->n = n;
  s->Pr = Pr;
  s->Pc = Pc;
  s->rank = rank;
  s->loopback = loopback;
  s->kq = pencil_kq(n, Pc);
  const size_t elem = s->base->elem;
  s->buf_bytes = size_t(ni) * n * s->kq * 2 * elem;
  s->blk_bytes = size_t(ni) * nj * n * elem;
  if ((size_t(ni) * nj) % 32) {
    free_pencil(s);
    return fail(ARENA_EUNSUPPORTED, "rank block too small");
  }
  s->ranks.resize(loopback ? Pr * Pc : 1);
  for (PencilRank& r : s->ranks) {
    cudaError_t e = cudaSuccess;
    // loopback: one block per virtual rank for f and u (K1 reads it in phase 0, K5 writes
    // it in phase 4), so a 2048^3 fp32 field solved in place fits one GPU
    if ((e = cudaMalloc(&r.buf1, s->buf_bytes)) || (e = cudaMalloc(&r.buf2, s->buf_bytes)) ||
        (loopback && (e = cudaMalloc(&r.fblk, s->blk_bytes)))) {
      free_pencil(s);
      return fail(ARENA_ENOMEM, "pencil buffers: " + std::string(cudaGetErrorString(e)));
    }
    r.ublk = r.fblk;
  }
  if (cudaError_t e = s->sync.init(Pr * Pc)) {
    free_pencil(s);
    return fail(ARENA_ENOMEM, "pencil barrier flags: " + std::string(cudaGetErrorString(e)));
  }
  if (!loopback && id) {
    NcclApi* a = nccl_api();
    auto split = reinterpret_cast<ncclResult_t (*)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*)>(
        a ? dlsym(a->h, "ncclCommSplit") : nullptr);
    if (!a || !split) {
      free_pencil(s);
      return fail(ARENA_ENCCL, "libnccl.so.2 (with ncclCommSplit) not found");
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclResult_t res = a->CommInitRank(&s->world, Pr * Pc, uid, rank);
    if (res != ncclSuccess) {
      s->world = nullptr;
      free_pencil(s);
      return nccl_fail(res, "ncclCommInitRank");
    }
    const int r = rank / Pc, c = rank % Pc;
    if ((res = split(s->world, r, c, &s->row, nullptr)) != ncclSuccess ||
        (res = split(s->world, c, r, &s->col, nullptr)) != ncclSuccess) {
      free_pencil(s);
      return nccl_fail(res, "ncclCommSplit");
    }
  }
  *out = s;
  return ARENA_OK;
}

PencilArgs pencil_args(arena_fft_pencil* s, PencilRank& pr, int rank, const void* f, void* u, cudaStream_t st) {
  arena_fft_plan* p = s->base;
  PencilArgs a{};
  a.f = f;
  a.u = u;
  a.buf1 = pr.buf1;
  a.buf2 = pr.buf2;
  a.tw = p->tw;
  a.stw = p->stw;
  a.n = s->n;
  a.Pr = s->Pr;
  a.Pc = s->Pc;
  a.r = rank / s->Pc;
  a.c = rank % s->Pc;
  a.kq = s->kq;
  a.stream = st;
  a.tma = &pr.tma;
  a.tma2 = &pr.tma2;
  a.sm_count = p->sm_count;
  a.fold = s->fold;
  if (s->xmode == ARENA_XCHG_PEER) {
    a.pz = pr.pz;
    a.py1 = pr.py1;
    a.px = pr.px;
    a.py2 = pr.py2;
  }
  return a;
}

// Peer destinations of virtual rank rk = (r, c) given every rank's buffers.
void pencil_fill_peers(arena_fft_pencil* s, PencilRank& me, int rk, const std::vector<std::vector<void*>>& bufs) {
  const int r = rk / s->Pc, c = rk % s->Pc;
  const size_t rb = s->row_chunk_bytes(), cb = s->col_chunk_bytes();
  for (int q = 0; q < s->Pc; ++q) {  // row peers (r, q)
    me.pz[q] = static_cast<char*>(bufs[r * s->Pc + q][1]) + size_t(c) * rb;
    me.py2[q] = static_cast<char*>(bufs[r * s->Pc + q][0]) + size_t(c) * rb;
  }
  for (int q = 0; q < s->Pr; ++q) {  // column peers (q, c)
    me.py1[q] = static_cast<char*>(bufs[q * s->Pc + c][0]) + size_t(r) * cb;
    me.px[q] = static_cast<char*>(bufs[q * s->Pc + c][1]) + size_t(r) * cb;
  }
}

// Row (same r) or column (same c) all-to-all from buf `from` to buf `to`
// (1 = buf1, 2 = buf2); chunk q of a rank's source goes to peer q's chunk
// (sender's index in the group).
arena_status pencil_exchange(arena_fft_pencil* s, cudaStream_t st, bool rowgrp, int from, int to) {
  // folded: the same exchange for each quadrant's H problem, quadrant q's region at q qbytes
  const int nq = s->fold ? 4 : 1, ne = s->fold ? s->n / 2 : s->n;
  const int ni = ne / s->Pr;
  const int grp = rowgrp ? s->Pc : s->Pr;
  const size_t chunk_rows = size_t(ni) * (rowgrp ? ne / s->Pc : ne / s->Pr);
  const size_t bytes = chunk_rows * s->kq * 2 * s->base->elem;
  const size_t qbytes = size_t(ni) * ne * s->kq * 2 * s->base->elem;
  auto buf = [&](PencilRank& r, int which) { return static_cast<char*>(which == 1 ? r.buf1 : r.buf2); };
  if (s->loopback) {
    for (int rk = 0; rk < s->Pr * s->Pc; ++rk) {
      const int r = rk / s->Pc, c = rk % s->Pc;
      const int me = rowgrp ? c : r;
      for (int q = 0; q < grp; ++q) {
        const int peer = rowgrp ? r * s->Pc + q : q * s->Pc + c;
        for (int qd = 0; qd < nq; ++qd) {
          cudaError_t e = cudaMemcpyAsync(buf(s->ranks[peer], to) + qd * qbytes + size_t(me) * bytes,
                                          buf(s->ranks[rk], from) + qd * qbytes + size_t(q) * bytes, bytes,
                                          cudaMemcpyDeviceToDevice, st);
          if (e != cudaSuccess) return cuda_fail(e, "loopback pencil exchange");
        }
      }
    }
    return ARENA_OK;
  }
  NcclApi* a = nccl_api();
  const ncclDataType_t dt = s->base->prec == 64 ? ncclFloat64 : ncclFloat32;
  const size_t count = chunk_rows * s->kq * 2;
  ncclComm_t comm = rowgrp ? s->row : s->col;
  PencilRank& me = s->ranks[0];
  ncclResult_t res = a->GroupStart();
  if (res != ncclSuccess) return nccl_fail(res, "ncclGroupStart");
  for (int q = 0; q < grp; ++q)
    for (int qd = 0; qd < nq; ++qd) {
      if ((res = a->Send(buf(me, from) + qd * qbytes + size_t(q) * bytes, count, dt, q, comm, st)) != ncclSuccess)
        return nccl_fail(res, "ncclSend");
      if ((res = a->Recv(buf(me, to) + qd * qbytes + size_t(q) * bytes, count, dt, q, comm, st)) != ncclSuccess)
        return nccl_fail(res, "ncclRecv");
    }
  if ((res = a->GroupEnd()) != ncclSuccess) return nccl_fail(res, "ncclGroupEnd");
  return ARENA_OK;
}

}  // namespace

extern "C" {

arena_status arena_pencil_create(arena_fft_pencil** out, int n, int precision_bits, int device, int pr, int pc,
                                 int rank, const void* nccl_id) {
  if (!nccl_id) return fail(ARENA_EINVAL, "NCCL unique id is NULL");
  return pencil_init(out, n, precision_bits, device, pr, pc, rank, 0, nccl_id);
}

arena_status arena_pencil_create_loopback(arena_fft_pencil** out, int n, int precision_bits, int device, int pr,
                                          int pc) {
  return pencil_init(out, n, precision_bits, device, pr, pc, 0, 1, nullptr);
}

void arena_pencil_destroy(arena_fft_pencil* s) { free_pencil(s); }

int arena_pencil_launches_per_solve(const arena_fft_pencil* s) {
  if (!s) return 0;
  const bool barrier = s->xmode == ARENA_XCHG_PEER && !s->loopback && s->Pr * s->Pc > 1;
  return 5 * int(s->ranks.size()) + (barrier ? 4 : 0);
}

arena_status arena_pencil_info(const arena_fft_pencil* s, int* kq, size_t* buffer_bytes, size_t* block_bytes) {
  if (!s) return fail(ARENA_EINVAL, "pencil is NULL");
  if (kq) *kq = s->kq;
  if (buffer_bytes) *buffer_bytes = s->buf_bytes;
  if (block_bytes) *block_bytes = s->blk_bytes;
  return ARENA_OK;
}

// Phase p of a pencil solve: 0 K1 (+ row exchange), 1 K2 (+ column exchange),
// 2 K3 (+ column exchange back), 3 K4 (+ row exchange back), 4 K5.  Loopback
// phases 0 / 4 also scatter f into / gather u from the virtual ranks' blocks.
static arena_status pencil_run_phase(arena_fft_pencil* s, int phase, const void* d_f, void* d_u, cudaStream_t st) {
  static const int kPh[5] = {kPencilZ1, kPencilY1, kPencilX, kPencilY2, kPencilZ2};
  if (phase < 0 || phase > 4) return fail(ARENA_EINVAL, "pencil phase must be 0 .. 4");
  if (s->xmode == ARENA_XCHG_PEER && !s->loopback && !s->attached)
    return fail(ARENA_EINVAL, "peer exchange: call arena_pencil_peer_attach first");
  const int n = s->n, ni = n / s->Pr, nj = n / s->Pc;
  const size_t elem = s->base->elem;
  const int nr = int(s->ranks.size());
  cudaError_t e;
  // The rank's block as sub-blocks of the full field: plain — one (ni x nj) block at
  // (r ni, c nj); folded — four (ni/2 x nj/2) blocks at (r ni/2 + a H, c nj/2 + b H).
  auto blocks = [&](int rk, auto&& fn) -> cudaError_t {
    const int r = rk / s->Pc, c = rk % s->Pc;
    if (!s->fold) return fn(size_t(r) * ni, size_t(c) * nj, size_t(0), size_t(0), ni, nj);
    const int H = n / 2, hi = ni / 2, hj = nj / 2;
    for (int a2 = 0; a2 < 2; ++a2)
      for (int b2 = 0; b2 < 2; ++b2) {
        cudaError_t e2 = fn(size_t(a2) * H + size_t(r) * hi, size_t(b2) * H + size_t(c) * hj, size_t(a2) * hi,
                            size_t(b2) * hj, hi, hj);
        if (e2 != cudaSuccess) return e2;
      }
    return cudaSuccess;
  };
  if (s->loopback && phase == 0) {  // scatter the full field into the virtual ranks' blocks
    for (int rk = 0; rk < nr; ++rk) {
      e = blocks(rk, [&](size_t gi, size_t gj, size_t li, size_t lj, int bi, int bj) {
        const char* src = static_cast<const char*>(d_f) + (gi * n + gj) * n * elem;
        char* dst = static_cast<char*>(s->ranks[rk].fblk) + (li * nj + lj) * n * elem;
        return cudaMemcpy2DAsync(dst, size_t(nj) * n * elem, src, size_t(n) * n * elem, size_t(bj) * n * elem, bi,
                                 cudaMemcpyDeviceToDevice, st);
      });
      if (e != cudaSuccess) return cuda_fail(e, "pencil scatter");
    }
  }
  for (int v = 0; v < nr; ++v) {
    const int rank = s->loopback ? v : s->rank;
    PencilRank& pr = s->ranks[v];
    const void* f = s->loopback ? pr.fblk : d_f;
    void* u = s->loopback ? pr.ublk : d_u;
    const PencilArgs a = pencil_args(s, pr, rank, f, u, st);
    cudaError_t err = s->base->prec == 64 ? pencil_phase_f64(a, kPh[phase]) : pencil_phase_f32(a, kPh[phase]);
    if (err != cudaSuccess) return cuda_fail(err, "pencil phase");
  }
  if (s->xmode != ARENA_XCHG_PEER) {
    arena_status r = ARENA_OK;
    if (phase == 0) r = pencil_exchange(s, st, true, 1, 2);   // R -> Y
    if (phase == 1) r = pencil_exchange(s, st, false, 1, 2);  // B2 -> C
    if (phase == 2) r = pencil_exchange(s, st, false, 2, 1);  // C -> B2
    if (phase == 3) r = pencil_exchange(s, st, true, 2, 1);   // Y -> R
    if (r != ARENA_OK) return r;
  }
  if (s->loopback && phase == 4) {
    for (int rk = 0; rk < nr; ++rk) {
      e = blocks(rk, [&](size_t gi, size_t gj, size_t li, size_t lj, int bi, int bj) {
        char* dst = static_cast<char*>(d_u) + (gi * n + gj) * n * elem;
        const char* src = static_cast<const char*>(s->ranks[rk].ublk) + (li * nj + lj) * n * elem;
        return cudaMemcpy2DAsync(dst, size_t(n) * n * elem, src, size_t(nj) * n * elem, size_t(bj) * n * elem, bi,
                                 cudaMemcpyDeviceToDevice, st);
      });
      if (e != cudaSuccess) return cuda_fail(e, "pencil gather");
    }
  }
  return ARENA_OK;
}

arena_status arena_pencil_solve_device(arena_fft_pencil* s, const void* d_f, void* d_u, void* stream) {
  if (!s || !d_f || !d_u) return fail(ARENA_EINVAL, "NULL pencil or buffer");
  DeviceGuard g(s->base->device);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int P = s->Pr * s->Pc;
  const bool barrier = s->xmode == ARENA_XCHG_PEER && !s->loopback && P > 1;
  for (int phase = 0; phase < 5; ++phase) {
    arena_status r = pencil_run_phase(s, phase, d_f, d_u, st);
    if (r != ARENA_OK) return r;
    if (barrier && phase < 4 && (r = s->sync.barrier(st, s->rank, P)) != ARENA_OK) return r;
  }
  return ARENA_OK;
}

arena_status arena_pencil_solve_phase(arena_fft_pencil* s, int phase, const void* d_f, void* d_u, void* stream) {
  if (!s || !d_f || !d_u) return fail(ARENA_EINVAL, "NULL pencil or buffer");
  DeviceGuard g(s->base->device);
  return pencil_run_phase(s, phase, d_f, d_u, static_cast<cudaStream_t>(stream));
}

arena_status arena_pencil_create_peer(arena_fft_pencil** out, int n, int precision_bits, int device, int pr, int pc,
                                      int rank) {
  if (pr * pc > kMaxPeers) return fail(ARENA_EUNSUPPORTED, "peer exchange supports at most 8 ranks");
  arena_status st = pencil_init(out, n, precision_bits, device, pr, pc, rank, 0, nullptr);
  if (st == ARENA_OK) (*out)->xmode = ARENA_XCHG_PEER;
  return st;
}

int arena_pencil_peer_handle_bytes(void) { return int(3 * sizeof(cudaIpcMemHandle_t)); }

arena_status arena_pencil_peer_export(arena_fft_pencil* s, void* out, int len) {
  if (!s || !out || len < arena_pencil_peer_handle_bytes()) return fail(ARENA_EINVAL, "handle buffer too small");
  if (s->loopback) return fail(ARENA_EINVAL, "loopback pencils have no peers to export to");
  DeviceGuard g(s->base->device);
  return s->sync.export_handles({s->ranks[0].buf1, s->ranks[0].buf2}, out);
}

arena_status arena_pencil_peer_attach(arena_fft_pencil* s, const void* all, int len) {
  const int P = s ? s->Pr * s->Pc : 0;
  if (!s || !all || len < arena_pencil_peer_handle_bytes() * P) return fail(ARENA_EINVAL, "need every rank's handles");
  if (s->loopback) return fail(ARENA_EINVAL, "loopback pencils need no attach");
  if (P > kMaxPeers) return fail(ARENA_EUNSUPPORTED, "peer exchange supports at most 8 ranks");
  if (s->attached) return ARENA_OK;
  DeviceGuard g(s->base->device);
  std::vector<std::vector<void*>> bufs;
  arena_status st = s->sync.attach(all, P, s->rank, {s->ranks[0].buf1, s->ranks[0].buf2}, bufs);
  if (st != ARENA_OK) return st;
  pencil_fill_peers(s, s->ranks[0], s->rank, bufs);
  s->attached = true;
  s->xmode = ARENA_XCHG_PEER;
  return ARENA_OK;
}

arena_status arena_pencil_set_exchange(arena_fft_pencil* s, int mode) {
  if (!s) return fail(ARENA_EINVAL, "pencil is NULL");
  if (mode == ARENA_XCHG_COPY) {
    if (!s->loopback && !s->world) return fail(ARENA_EINVAL, "this pencil has no NCCL communicators");
    s->xmode = mode;
    return ARENA_OK;
  }
  if (mode != ARENA_XCHG_PEER) return fail(ARENA_EINVAL, "unknown exchange mode");
  if (s->Pr * s->Pc > kMaxPeers) return fail(ARENA_EUNSUPPORTED, "peer exchange supports at most 8 ranks");
  if (s->loopback) {
    std::vector<std::vector<void*>> bufs;
    for (PencilRank& r : s->ranks) bufs.push_back({r.buf1, r.buf2});
    for (int rk = 0; rk < int(s->ranks.size()); ++rk) pencil_fill_peers(s, s->ranks[rk], rk, bufs);
  } else if (!s->attached) {
    return fail(ARENA_EINVAL, "peer exchange: call arena_pencil_peer_attach first");
  }
  s->xmode = mode;
  return ARENA_OK;
}

arena_status arena_pencil_set_layout(arena_fft_pencil* s, int layout) {
  if (!s) return fail(ARENA_EINVAL, "pencil is NULL");
  if (layout != ARENA_PENCIL_PLAIN && layout != ARENA_PENCIL_FOLDED) return fail(ARENA_EINVAL, "unknown pencil layout");
  if (layout == ARENA_PENCIL_FOLDED && (s->n / 2 / s->Pr < 1 || s->n / 2 / s->Pc < 1 || s->n < 64))
    return fail(ARENA_EUNSUPPORTED, "folded pencil needs n >= 64 and n/2 divisible by the grid");
  if (s->attached) return fail(ARENA_EINVAL, "set the pencil layout before arena_pencil_peer_attach");
  s->fold = layout == ARENA_PENCIL_FOLDED ? 1 : 0;
  if (s->loopback && s->xmode == ARENA_XCHG_PEER) {  // peer chunk offsets depend on the layout
    std::vector<std::vector<void*>> bufs;
    for (PencilRank& r : s->ranks) bufs.push_back({r.buf1, r.buf2});
    for (int rk = 0; rk < int(s->ranks.size()); ++rk) pencil_fill_peers(s, s->ranks[rk], rk, bufs);
  }
  return ARENA_OK;
}

arena_status arena_pencil_barrier_status(arena_fft_pencil* s) {
  if (!s) return fail(ARENA_EINVAL, "pencil is NULL");
  DeviceGuard g(s->base->device);
  return s->sync.status();
}

}  // extern "C"
