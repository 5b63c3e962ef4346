// plan_slab.cuh — slab decomposition, its NCCL / loopback / peer exchanges
//
// Part of the plan.cu translation unit (included at its end: it shares the
// plan's internal types and helpers), kept in its own file for readability.
#pragma once

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
