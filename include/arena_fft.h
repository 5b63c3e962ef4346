/*
 * arena_fft.h — C ABI of the B200-native spectral Poisson solver.
 *
 * This is the drop-in boundary for the reference's FFT hot path.  The
 * reference exposes no FFI of its own: its only interface for the path is the
 * C++ free function
 *     arena::GridField arena::poisson_spectral_solve(const arena::GridField&)
 *       /root/reference/proj/include/arena/fft_solver.hpp:23
 *       /root/reference/proj/src/fft_solver.cpp:51-87
 * plus its siblings dft3_forward / dft3_inverse (fft_solver.hpp:13,16).
 * include/arena/fft_solver.hpp re-declares exactly those C++ signatures and
 * paper_1408_6497_b200/csrc/fft_solver_dropin.cpp implements them over the
 * entry points below.  Every entry point is extern "C", takes plain pointers
 * and sizes, and never throws; errors are status codes plus a thread-local
 * message (arena_last_error).  See INTEGRATION.md for the bindings a
 * maintainer would add.
 *
 * Data layout at the boundary (identical to GridField, grid.hpp:11-27): an
 * n x n x n row-major array of values sampled at (i/n, j/n, k/n), element
 * (i, j, k) at ((i*n)+j)*n+k, k contiguous.  fp64 buffers are double, fp32
 * buffers float.  Complex spectra (dft3_*) are interleaved (re, im) n^3
 * arrays in the same row-major order, i.e. std::vector<std::complex<double>>.
 */
#ifndef ARENA_FFT_H
#define ARENA_FFT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum arena_status {
  ARENA_OK = 0,
  ARENA_EINVAL = 1,      /* bad argument: n < 2 (GridField throws, grid.hpp:18), NULL pointer, ... */
  ARENA_ENOMEM = 2,      /* device or pinned-host allocation failed (std::bad_alloc analogue) */
  ARENA_ECUDA = 3,       /* CUDA runtime / launch error */
  ARENA_ENCCL = 4,       /* NCCL error (multi-GPU plans) */
  ARENA_EUNSUPPORTED = 5 /* valid request this build cannot serve (e.g. no sm_100a device) */
} arena_status;

typedef struct arena_fft_plan arena_fft_plan;

/* Execution path chosen for a plan (arena_fft_plan_info). */
enum { ARENA_PATH_POW2 = 0, ARENA_PATH_GENERIC = 1 };

/* Setup ("Setup" in the paper's Setup/Solve split; replaces the
 * per-call fftw_plan_* at fft_solver.cpp:60-63 with a once-per-(n, precision,
 * device) object): twiddle tables, the device half-spectrum workspace and
 * kernel attributes.  precision_bits is 64 (the reference's double) or 32.
 * device is a CUDA ordinal; -1 means the calling thread's current device. */
arena_status arena_fft_plan_create(arena_fft_plan** plan, int n, int precision_bits, int device);
void arena_fft_plan_destroy(arena_fft_plan* plan);

/* Query: n, precision bits, path (ARENA_PATH_*), device, bytes of device workspace. */
arena_status arena_fft_plan_info(const arena_fft_plan* plan, int* n, int* precision_bits, int* path,
                                 int* device, size_t* workspace_bytes);

/* The solve, device-resident (the timed hot path).  d_f, d_u: caller-owned
 * device buffers of n^3 values (may alias: u may overwrite f).  stream: a
 * cudaStream_t (NULL = legacy default stream).  Asynchronous: returns after
 * enqueueing; errors from the launches are reported, kernel faults surface on
 * the caller's next synchronisation.  Semantics of fft_solver.cpp:51-87:
 * u = IFFT( FFT(f) * (k2 == 0 ? 0 : (1/n^3) / (4 pi^2 k2)) ), k2 = |signed k|^2.
 * Thread-safe; the plan's workspace is shared by all its solves, so a solve
 * enqueued on one stream waits (cudaStreamWaitEvent) for the plan's previous
 * solve on any stream — solves on one plan never overlap.  Use one plan per
 * stream for concurrent solves. */
arena_status arena_poisson_solve_device(arena_fft_plan* plan, const void* d_f, void* d_u, void* stream);

/* The drop-in path: host buffers in and out (pageable or pinned), copies
 * inside.  Synchronous.  This is what arena::poisson_spectral_solve calls. */
arena_status arena_poisson_solve_host(arena_fft_plan* plan, const void* f, void* u);

/* Batched drop-in path: `count` independent fields f[s] -> u[s] (host buffers;
 * pinned for full PCIe speed).  The copy-in of field s+1 and copy-out of field
 * s-1 overlap the solve of field s on separate streams.  Synchronous. */
arena_status arena_poisson_solve_host_batch(arena_fft_plan* plan, int count, const void* const* f, void* const* u);

/* arena::dft3_forward (fft_solver.cpp:13-29): real n^3 -> full complex n^3
 * spectrum (interleaved), unnormalised, sign -1.  Host and device variants. */
arena_status arena_dft3_forward_host(arena_fft_plan* plan, const void* g, void* spec);
arena_status arena_dft3_forward_device(arena_fft_plan* plan, const void* d_g, void* d_spec, void* stream);
/* arena::dft3_inverse (fft_solver.cpp:31-49): complex n^3 -> Re(backward)/n^3. */
arena_status arena_dft3_inverse_host(arena_fft_plan* plan, const void* spec, void* g);
arena_status arena_dft3_inverse_device(arena_fft_plan* plan, const void* d_spec, void* d_g, void* stream);

/* Measurement hooks (bench.py): when enabled, every solve records a CUDA event
 * before each kernel and after the last one on the solve's stream; query the
 * accumulated per-kernel milliseconds (sum over recorded solves; names[i] is
 * the kernel label) with arena_fft_stage_times, which synchronises. */
arena_status arena_fft_set_stage_timing(arena_fft_plan* plan, int enable);
arena_status arena_fft_stage_times(arena_fft_plan* plan, double* ms, const char** names, int max_stages,
                                   int* n_stages, int* n_solves);

/* Number of kernel launches one arena_poisson_solve_device call enqueues. */
int arena_poisson_launches_per_solve(const arena_fft_plan* plan);

/* Device-side input generation (replaces host sampling
 * through std::function, grid.cpp:21-27, which is infeasible at 1024^3+).
 * Not part of the solve.  d_out: device buffer of n^3 values.
 *   arena_source_modes:    out = sum_m Re(coef_m exp(2 pi i k_m . x)), x = (i,j,k)/n;
 *                          k: 3*nmodes host ints, coef: 2*nmodes host doubles (re, im).
 *   arena_source_gaussian: periodised Gaussian over the 27 nearest images,
 *                          which = 0: u = sum exp(-alpha r^2), 1: f = -Lap u. */
arena_status arena_source_modes(int n, int precision_bits, int nmodes, const int* k, const double* coef, void* d_out,
                                void* stream);
arena_status arena_source_gaussian(int n, int precision_bits, double alpha, double cx, double cy, double cz, int which,
                                   void* d_out, void* stream);
/* Slab variants: only planes i0 .. i0+ni-1 of the n^3 field (ni*n*n values). */
arena_status arena_source_modes_slab(int n, int precision_bits, int nmodes, const int* k, const double* coef, int i0,
                                     int ni, void* d_out, void* stream);
arena_status arena_source_gaussian_slab(int n, int precision_bits, double alpha, double cx, double cy, double cz,
                                        int which, int i0, int ni, void* d_out, void* stream);

/* Block variants (pencil ranks): planes i0 .. i0+ni-1, rows j0 .. j0+nj-1, stored ni x nj x n. */
arena_status arena_source_modes_block(int n, int precision_bits, int nmodes, const int* k, const double* coef, int i0,
                                      int ni, int j0, int nj, void* d_out, void* stream);
arena_status arena_source_gaussian_block(int n, int precision_bits, double alpha, double cx, double cy, double cz,
                                         int which, int i0, int ni, int j0, int nj, void* d_out, void* stream);

/* ---- Slab decomposition over P GPUs ------------------------
 * One process per GPU.  Rank r owns planes i in [r*n/P, (r+1)*n/P) of f and u
 * (a contiguous n/P * n * n slice of the GridField layout).  The two global
 * transposes are grouped ncclSend/ncclRecv all-to-alls (NCCL loaded at run time).
 * Create: rank 0 calls arena_nccl_unique_id, the id (arena_nccl_unique_id_bytes()
 * bytes) is broadcast out of band (e.g. torch.distributed), every rank calls
 * arena_slab_create.  arena_slab_create_loopback runs P virtual ranks on ONE
 * device (exchanges are device copies) — used to test the decomposition without
 * a multi-GPU box; its solve takes the full n^3 field.  Power-of-two n, P | n. */
typedef struct arena_fft_slab arena_fft_slab;
int arena_nccl_unique_id_bytes(void);
arena_status arena_nccl_unique_id(void* out, int len);
arena_status arena_slab_create(arena_fft_slab** slab, int n, int precision_bits, int device, int nranks, int rank,
                               const void* nccl_id);
arena_status arena_slab_create_loopback(arena_fft_slab** slab, int n, int precision_bits, int device, int nvranks);
void arena_slab_destroy(arena_fft_slab* slab);
arena_status arena_slab_info(const arena_fft_slab* slab, int* ni, int* nj, size_t* chunk_bytes, size_t* workspace_bytes);
int arena_slab_launches_per_solve(const arena_fft_slab* slab);
/* d_f, d_u: this rank's slab (loopback: the full field); asynchronous on stream. */
arena_status arena_slab_solve_device(arena_fft_slab* slab, const void* d_f, void* d_u, void* stream);

/* Exchange modes.  COPY: K2 / K3 work in place and the all-to-alls are NCCL
 * grouped send/recv (loopback: device copies).  PEER: the ranks' workspaces are
 * mapped into each other's address space (CUDA IPC over NVLink / NVSwitch) and
 * K2 / K3 store every output chunk straight into the owning rank's workspace —
 * the all-to-all is fused into the transform; a device-side flag barrier
 * (release / acquire, system scope) separates the phases.  Not in the reference
 * code (its FFT is single-process); the paper's distributed solve. */
enum { ARENA_XCHG_COPY = 0, ARENA_XCHG_PEER = 1 };
/* One rank of a peer-exchange slab (no NCCL).  Before solving: export this
 * rank's handles, gather every rank's (rank order) out of band, attach. */
arena_status arena_slab_create_peer(arena_fft_slab** slab, int n, int precision_bits, int device, int nranks, int rank);
int arena_slab_peer_handle_bytes(void);
arena_status arena_slab_peer_export(arena_fft_slab* slab, void* out, int len);
arena_status arena_slab_peer_attach(arena_fft_slab* slab, const void* all_handles, int len);
/* Switch the exchange of a loopback slab (or an attached NCCL slab). */
arena_status arena_slab_set_exchange(arena_fft_slab* slab, int mode);
/* COPY exchange in sub-steps (default 4 per direction, env ARENA_SLAB_CHUNKS): the
 * all-to-all of sub-range k (forward: the rank's i planes; backward: whole 64-row j
 * blocks of its j lines) runs on the slab's exchange stream while K1+K2 (K3) of
 * sub-range k+1 run on the solve's stream.  1, 1 = whole passes, then whole chunks. */
arena_status arena_slab_set_chunking(arena_fft_slab* slab, int fwd_substeps, int bwd_substeps);
arena_status arena_slab_get_chunking(const arena_fft_slab* slab, int* fwd_substeps, int* bwd_substeps);
/* Host-only (no device needed): the in-chunk row ranges {first[k], rows[k]} a sub-step
 * [lo, hi) of an exchange moves between every pair of ranks; returns their count
 * (-1: bad arguments).  For the CPU model tests of the chunked schedule. */
int arena_slab_exchange_pieces(int n, int nranks, int forward, int lo, int hi, size_t* first, size_t* rows, int max);
/* Wait for a solve enqueued on `stream` with NCCL error / hang detection: polls
 * ncclCommGetAsyncError, aborts the communicator (ARENA_ENCCL) on an asynchronous
 * error or when the solve has not completed after timeout_s seconds. */
arena_status arena_slab_wait(arena_fft_slab* slab, void* stream, double timeout_s);
/* Per-stage CUDA-event timing of arena_slab_solve_device on the solve's stream:
 * ms5 = total ms over the timed solves of {K1+K2, exchange #1, K3, exchange #2,
 * K4+K5} (PEER mode: the exchanges are inside K2 / K3 and the "exchange" stages
 * are the device barriers, i.e. the wait for the slowest rank). */
arena_status arena_slab_set_stage_timing(arena_fft_slab* slab, int enable);
arena_status arena_slab_stage_times(arena_fft_slab* slab, double* ms5, int* n_solves);
/* Phase p in {0, 1, 2} of a solve (K1+K2, K3, K4+K5, with the COPY exchanges
 * after phases 0 and 1).  In PEER mode the caller must synchronise all ranks
 * between phases (arena_slab_solve_device does it on the device). */
arena_status arena_slab_solve_phase(arena_fft_slab* slab, int phase, const void* d_f, void* d_u, void* stream);
/* Device-side verification (synchronous; fp64 accumulation with compensated
 * sums).  arena_field_stats = GridField::mean / max_abs (grid.cpp:9-19) of a
 * device field.  arena_field_compare = the gauge-aligned error of
 * linf_rel_error (problems.cpp:88-106) on the grid: shift = mean(exact) -
 * mean(num); linf_rel = max|num + shift - exact| / max|exact|; rel_l2 =
 * ||num + shift - exact||_2 / ||exact - mean(exact)||_2.  Fields are `count`
 * contiguous values (n^3 for a GridField).  Any output may be NULL. */
arena_status arena_field_stats(size_t count, int precision_bits, const void* d_field, double* mean, double* max_abs);
arena_status arena_field_compare(size_t count, int precision_bits, const void* d_num, const void* d_exact,
                                 double* rel_l2, double* linf_rel, double* gauge_shift);

/* ARENA_OK, or ARENA_ECUDA if a device barrier gave up waiting (20 s). */
arena_status arena_slab_barrier_status(arena_fft_slab* slab);
/* Check the peer barrier protocol on one device: one cooperative launch, block r
 * plays rank r for `rounds` barriers; *bad = visibility violations seen (0). */
arena_status arena_peer_barrier_selftest(int device, int nranks, int rounds, int* bad);

/* ---- Pencil decomposition over Pr x Pc GPUs (BASELINE config 5) --------------
 * Rank r*Pc + c owns the f / u block i in [r n/Pr, (r+1) n/Pr), j in
 * [c n/Pc, (c+1) n/Pc), all k, stored contiguously as (n/Pr) x (n/Pc) x n.
 * Four all-to-alls per solve on row / column communicators (ncclCommSplit of a
 * world communicator made from nccl_id).  Loopback: all ranks on one device, the
 * solve takes the full n^3 field.  Power-of-two 64 <= n <= 2048. */
typedef struct arena_fft_pencil arena_fft_pencil;
arena_status arena_pencil_create(arena_fft_pencil** pencil, int n, int precision_bits, int device, int pr, int pc,
                                 int rank, const void* nccl_id);
arena_status arena_pencil_create_loopback(arena_fft_pencil** pencil, int n, int precision_bits, int device, int pr,
                                          int pc);
void arena_pencil_destroy(arena_fft_pencil* pencil);
arena_status arena_pencil_info(const arena_fft_pencil* pencil, int* kq, size_t* buffer_bytes, size_t* block_bytes);
int arena_pencil_launches_per_solve(const arena_fft_pencil* pencil);
arena_status arena_pencil_solve_device(arena_fft_pencil* pencil, const void* d_f, void* d_u, void* stream);
/* Peer exchange for the pencil (see ARENA_XCHG_PEER): K1 / K2 / K3 / K4 store
 * their output chunks straight into the row / column peers' buffers; four
 * device barriers per solve.  Phases of arena_pencil_solve_phase: 0 K1, 1 K2,
 * 2 K3, 3 K4, 4 K5 (COPY mode: with the exchange after phases 0-3). */
arena_status arena_pencil_create_peer(arena_fft_pencil** pencil, int n, int precision_bits, int device, int pr, int pc,
                                      int rank);
int arena_pencil_peer_handle_bytes(void);
arena_status arena_pencil_peer_export(arena_fft_pencil* pencil, void* out, int len);
arena_status arena_pencil_peer_attach(arena_fft_pencil* pencil, const void* all_handles, int len);
arena_status arena_pencil_set_exchange(arena_fft_pencil* pencil, int mode);
arena_status arena_pencil_solve_phase(arena_fft_pencil* pencil, int phase, const void* d_f, void* d_u, void* stream);
arena_status arena_pencil_barrier_status(arena_fft_pencil* pencil);
/* Folded distribution (config 5 at 2048^3): rank (r, c) owns i in I_r U (I_r + n/2),
 * j in J_c U (J_c + n/2) (I_r, J_c: its n/(2 Pr), n/(2 Pc) slices of [0, n/2)) as a
 * (n/Pr) x (n/Pc) x n block whose local i < n/(2 Pr) is I_r and the rest I_r + n/2
 * (j alike).  The first radix-2 steps of the i and j transforms then run in the
 * rank's z passes and the strided passes are n/2-point (128-byte-row tiles at
 * 2048^3).  Set before the first solve (and before arena_pencil_peer_attach); both
 * exchanges (COPY, PEER) are supported. */
enum { ARENA_PENCIL_PLAIN = 0, ARENA_PENCIL_FOLDED = 1 };
arena_status arena_pencil_set_layout(arena_fft_pencil* pencil, int layout);

/* One process driving P GPUs (P <= 8; the drop-in's multi-GPU path, selected by
 * ARENA_FFT_NGPU): rank v lives on devices[v] (NULL: v mod device count) and holds
 * the planes i in [v n/P, (v+1) n/P) — a contiguous slab of GridField.data.  The
 * all-to-alls are fused into K2 / K3 as stores into the other GPUs' workspaces
 * through peer access (NVLink), the phases ordered by cross-device events.
 * Power-of-two n >= 16, n/P >= 4.  solve_device: per-rank shard pointers (and
 * streams, NULL = the object's own); solve_host: the whole n^3 host field, moved
 * slab by slab over the P PCIe links in parallel (synchronous). */
typedef struct arena_fft_mgpu arena_fft_mgpu;
arena_status arena_mgpu_create(arena_fft_mgpu** mgpu, int n, int precision_bits, int nranks, const int* devices);
void arena_mgpu_destroy(arena_fft_mgpu* mgpu);
arena_status arena_mgpu_info(const arena_fft_mgpu* mgpu, int* nranks, int* devices, size_t* slab_bytes);
arena_status arena_mgpu_solve_device(arena_fft_mgpu* mgpu, const void* const* d_f, void* const* d_u,
                                     void* const* streams);
arena_status arena_mgpu_solve_host(arena_fft_mgpu* mgpu, const void* f, void* u);

/* Batch evaluation of arena::SpectralInterpolant (fft_solver.cpp:89-114) on the
 * GPU: out[p] = sum_m Re(amp_m exp(2 pi i k_m . x_p)).  k: 3*nmodes ints (signed
 * frequencies), amp: 2*nmodes doubles (re, im — already divided by n^3 as in
 * SpectralInterpolant::build), pts: 3*npts doubles, out: npts doubles; all host
 * arrays.  device < 0: current device.  Synchronous. */
arena_status arena_interpolant_eval(int device, int nmodes, const int* k, const double* amp, int npts,
                                    const double* pts, double* out);

/* Tile geometry of the power-of-two kernels for (n, precision): out15[0..4] =
 * {line length, points/thread, lines/CTA, threads/CTA, shared bytes} of the
 * contiguous-axis (z) kernels, out15[5..9] the y kernels, out15[10..14] the x
 * kernel.  Host-only (no device needed); used by the CPU index-model tests. */
int arena_pow2_kernel_geometry(int n, int precision_bits, int* out15);

/* The calling thread's current CUDA device ordinal, or -1 when none is usable
 * (lets a plan cache keyed by device resolve "current device" before keying). */
int arena_current_device(void);

/* Thread-local description of the last failure on this thread ("" if none). */
const char* arena_last_error(void);

/* ABI version of this library (major * 100 + minor). */
int arena_fft_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif
