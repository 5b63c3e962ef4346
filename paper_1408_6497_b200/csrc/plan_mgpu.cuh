// plan_mgpu.cuh — one process driving several GPUs (the drop-in's ARENA_FFT_NGPU path)
//
// Part of the plan.cu translation unit (included at its end: it shares the
// plan's internal types and helpers), kept in its own file for readability.
#pragma once

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
