// launchers.h — host-side entry points of the kernel translation units
// (no device code; included by plan.cu).
#pragma once

#include <cuda_runtime.h>

#ifndef ARENA_JBLOCK
#define ARENA_JBLOCK 64  // j-block of the half-spectrum layout (see Layout).  B200 A/B (ms per solve,
                         // JB = 8 / 32 / 64): 1024^3 fp64 16.68 / 16.40 / 16.38 (y passes 3.41 -> 3.19,
                         // x 4.13 -> 4.23), 512^3 2.007 / 1.957 / 1.945, 2048^3 143.3 / 141.6 / 141.5;
                         // JB = 4: 16.87, 128: 16.36 fp64 but fp32 worse
#endif
// Rows per j block of a half-spectrum layout with nj j lines (poisson_pow2.cuh Layout).
inline int layout_jb(int nj) { return nj < ARENA_JBLOCK ? nj : ARENA_JBLOCK; }

namespace arena_fft {

constexpr int kPow2MaxN = 2048;

// Row pitch (complex elements) of the half spectrum for an n-point grid: nc =
// n/2 + 1 rounded up to 8 (128-byte fp64 rows), plus ARENA_PITCH_PAD extra units.
#ifndef ARENA_PITCH_PAD
#define ARENA_PITCH_PAD 0
#endif
__host__ __device__ constexpr int spec_pitch(int n) { return (n / 2 + 1 + 7) / 8 * 8 + 8 * ARENA_PITCH_PAD; }
constexpr int kMaxPeers = 8;  // ranks a slab solve can scatter to directly (peer-mapped workspaces)
constexpr int kPow2Launches = 5;

// Plan-owned cache of the TMA descriptors over the half-spectrum workspaces
// (encoded on first use; they depend only on the buffers and the geometry).
struct alignas(64) TmaCache {
  unsigned char maps[4][128];  // CUtensorMap: y boxes over B, x boxes over C, fused-kernel y boxes over B,
                              // (spare)
  const void* specB = nullptr;
  const void* specC = nullptr;
  int n = 0, ni = 0, nj = 0, nchunks = 0, quad = 0;
};

// Solve phases (bit mask): the slab path runs them around its two exchanges.
enum : int { kPhaseZY = 1, kPhaseX = 2, kPhaseYZ = 4, kPhaseAll = 7 };

// Stage-twiddle tables (fft_engine.cuh stage_tw_*) a plan holds: for line
// lengths N = n/2 (which = 0) and N = n (which = 1) and every points-per-thread
// E in {2, 4, 8, 16, 32} (clamped to N), concatenated in that order.
size_t stw_entries(int n);
size_t stw_offset(int n, int which, int E);
void stw_fill_host(int n, int precision_bits, void* host);  // stw_entries(n) vec2 values

struct Pow2Args {
  const void* f;
  void* u;
  void* spec;
  const void* tw;   // W_n^m, m in [0, n)
  const void* stw;  // stage-twiddle tables (stw_offset)
  int n, nc, ncp;
  cudaStream_t stream;
  cudaEvent_t* ev;  // nullable; kPow2Launches + 1 events: before each kernel and after the last
  TmaCache* tma;    // nullable: classic (non-TMA) strided kernels (single GPU only)
  int sm_count;
  // Slab geometry.  Single GPU: ni = nj = n, nchunks = 1, j0 = 0, specC = spec.
  int ni;        // local i planes (rows of f / u and of workspace B)
  int nj;        // local j lines of workspace C (x pass)
  int nchunks;   // P: number of slabs
  int j0;        // global j of local j = 0 (x pass)
  void* specC;   // workspace C (x pass); == spec on one GPU
  int phases;    // kPhase* mask
  int* ctrs;     // fused z+y passes: device counters (ni + 1 ints); nullptr = unfused kernels
  int lag;       // fused schedule lag in planes
  int fuse;      // kFuseFwd | kFuseInv: which z+y pairs run fused (needs ctrs)
  // Slab with peer-mapped workspaces: K2 / K3 store chunk c straight into
  // peer_y[c] / peer_x[c] (rank c's C / B, advanced to this rank's chunk);
  // nullptr = in-place (the exchange is a separate step).
  void* const* peer_y = nullptr;
  void* const* peer_x = nullptr;
  // Slab chunked exchange: with subn > 0 and phases == kPhaseZY (kPhaseX) only local i
  // planes (local j lines, whole JB blocks) [sub0, sub0 + subn) are transformed.
  int sub0 = 0, subn = 0;
  // Single GPU: 1 = quadrant formulation (poisson_quad.cuh, H = n/2-point y / x lines).
  int quad = 0;
};
enum : int { kFuseFwd = 1, kFuseInv = 2 };

cudaError_t launch_pow2_f64(const Pow2Args& a);
cudaError_t launch_pow2_f32(const Pow2Args& a);

// Pencil decomposition (Pr x Pc ranks): one phase of a rank's solve.
struct PencilArgs {
  const void* f;     // rank's f block: (n/Pr) x (n/Pc) x n
  void* u;           // rank's u block
  void* buf1;        // R (k-chunked z output) / B2 (y output, j chunks of n/Pr)
  void* buf2;        // Y (after the row exchange, j chunks of n/Pc) / C (x pass)
  const void* tw;
  const void* stw;
  int n, Pr, Pc, r, c;
  int kq;            // k-chunk pitch (complex)
  cudaStream_t stream;
  TmaCache* tma;     // maps[0]: y over buf2 (Y), maps[1]: x over buf2 (C); y-inv map in tma2
  TmaCache* tma2;    // maps[0]: y-inverse over buf1 (B2); peer mode: maps[1] x over buf1, maps[2] y-inverse over buf2
  int sm_count;
  // Peer exchange: every all-to-all is the stores of the pass before it.  The
  // spectrum then lives in buf2 (Y, then B2 for the way back) and buf1 (C, then
  // R for the way back): K1 -> row peer q's buf2, K2 -> column peer q's buf1,
  // K3 -> column peer q's buf2, K4 -> row peer q's buf1, each advanced to this
  // rank's chunk.  nullptr = NCCL / copy exchanges.
  void* const* pz = nullptr;
  void* const* py1 = nullptr;
  void* const* px = nullptr;
  void* const* py2 = nullptr;
  int fold = 0;  // folded distribution (poisson_qpencil.cuh): quadrant z passes, H-point strided passes
};
enum : int { kPencilZ1 = 0, kPencilY1, kPencilX, kPencilY2, kPencilZ2 };
cudaError_t pencil_phase_f64(const PencilArgs& a, int phase);
cudaError_t pencil_phase_f32(const PencilArgs& a, int phase);
// k-chunk pitch: ceil(nc / Pc) rounded up to 8 (128-byte rows), or to 2 when
// that would leave a rank without k (small n); every chunk is non-empty.
inline int pencil_kq(int n, int Pc) {
  const int nc = n / 2 + 1, w = (nc + Pc - 1) / Pc;
  for (int q : {8, 4, 2}) {
    const int kq = (w + q - 1) / q * q;
    if ((Pc - 1) * kq < nc) return kq;
  }
  return w;
}

// Line length, points per thread, lines per CTA, threads, shared bytes.
struct KernelGeom {
  int line, E, L, threads, smem;
};
// g[0]: z kernels (M = n/2 point lines), g[1]: y kernels, g[2]: x kernel (n-point lines).
bool pow2_config_f64(int n, KernelGeom* g);
bool pow2_config_f32(int n, KernelGeom* g);
// Whether the L2-fused z+y kernels exist for this n (they need 128-thread y tiles).
bool pow2_fused_ok_f64(int n);
bool pow2_fused_ok_f32(int n);

// Generic mixed-radix path (any n >= 2).  One Stockham plan for an n-point line.
constexpr int kGenMaxStages = 40;
struct GenPlan {
  int n;
  int nst;
  int radix[kGenMaxStages];
};
bool gen_plan_make(int n, GenPlan* p);
size_t gen_smem_bytes(int n, int elem_bytes);
int gen_max_n(int elem_bytes);

struct GenArgs {
  const GenPlan* plan;
  const void* tw;  // W_n^m, m in [0, n), vec2 of the precision
  int n, nc, ncp;
  cudaStream_t stream;
  cudaEvent_t* ev;  // nullable
};

// Poisson solve f -> u (device, n^3 real) via the half-spectrum workspace spec.
cudaError_t gen_poisson_f64(const GenArgs& a, const void* f, void* u, void* spec);
cudaError_t gen_poisson_f32(const GenArgs& a, const void* f, void* u, void* spec);
constexpr int kGenLaunches = 5;
// The generic z passes alone (rows' r2c into the generic layout / c2r back).
cudaError_t gen_z_r2c_f64(const GenArgs& a, const void* f, void* spec);
cudaError_t gen_z_r2c_f32(const GenArgs& a, const void* f, void* spec);
cudaError_t gen_z_c2r_f64(const GenArgs& a, const void* spec, void* u);
cudaError_t gen_z_c2r_f32(const GenArgs& a, const void* spec, void* u);

// Radix-R split path (R = 3: n = 3M, M a power of two in [16, 512]; R = 5: n = 5M,
// M in [16, 256]) onto the power-of-two passes (poisson_split3.cuh).
constexpr int kSplit3Launches = 7;
struct Split3Args {
  const void* f;
  void* u;
  void* S;          // generic-layout half spectrum (n*n rows of ncp)
  void* Q;          // nine chunks of Layout(M, M) rows of ncp
  const void* tw;   // W_n^m
  const void* stw;  // stage-twiddle tables of an n' = 2M plan (M-point lines: which = 0)
  const void* stwz; // stage-twiddle tables of an n' = M plan (M/2-point lines: the split z passes)
  int n, R, M, nc, ncp;
  cudaStream_t stream;
  cudaEvent_t* ev;  // nullable; kSplit3Launches + 1 events
  TmaCache* tma;
  int sm_count;
  const GenPlan* gplan;
};
// The split radix for n (3 or 5), or 0 when n is not R * 2^k in range.
inline int split_radix(int n) {
  for (int R : {3, 5}) {
    if (n % R) continue;
    const int M = n / R;
    if (M >= 16 && M <= (R == 3 ? 512 : 256) && (M & (M - 1)) == 0) return R;
  }
  return 0;
}
cudaError_t launch_split3_f64(const Split3Args& a);
cudaError_t launch_split3_f32(const Split3Args& a);
// dft3_forward: real g (n^3) -> complex spec (n^3, interleaved).  dft3_inverse:
// complex spec -> real g = Re(backward)/n^3 using `work` (n^3 complex) as scratch.
cudaError_t gen_dft3_forward_f64(const GenArgs& a, const void* g, void* spec);
cudaError_t gen_dft3_inverse_f64(const GenArgs& a, const void* spec, void* g, void* work);
cudaError_t gen_dft3_forward_f32(const GenArgs& a, const void* g, void* spec);
cudaError_t gen_dft3_inverse_f32(const GenArgs& a, const void* spec, void* g, void* work);

}  // namespace arena_fft
