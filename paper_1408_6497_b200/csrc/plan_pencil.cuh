// plan_pencil.cuh — pencil decomposition (plain and folded layouts)
//
// Part of the plan.cu translation unit (included at its end: it shares the
// plan's internal types and helpers), kept in its own file for readability.
#pragma once

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
