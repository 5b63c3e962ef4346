// stage_twiddles.cu — host construction of the per-stage twiddle tables the
// line engine reads (fft_engine.cuh: tab_s[r*NS + j] = W_{NS*R}^{j r}),
// computed in 80-bit long double and rounded once.
#include <cmath>
#include <cstring>

#include "fft_engine.cuh"
#include "launchers.h"

namespace arena_fft {

namespace {
constexpr int kEs[5] = {2, 4, 8, 16, 32};

int line_len(int n, int which) { return which ? n : n / 2; }
int clampE(int E, int N) { return E < N ? E : N; }
size_t table_entries(int N, int E) { return N >= 2 ? size_t(stage_tw_total(N, clampE(E, N))) : 0; }
}  // namespace

size_t stw_entries(int n) {
  size_t tot = 0;
  for (int which = 0; which < 2; ++which)
    for (int E : kEs) tot += table_entries(line_len(n, which), E);
  return tot;
}

size_t stw_offset(int n, int which, int E) {
  size_t off = 0;
  for (int w = 0; w < 2; ++w)
    for (int e : kEs) {
      if (w == which && clampE(e, line_len(n, w)) == clampE(E, line_len(n, w))) return off;
      off += table_entries(line_len(n, w), e);
    }
  return off;
}

void stw_fill_host(int n, int precision_bits, void* host) {
  const long double two_pi = 6.283185307179586476925286766559005768L;
  size_t idx = 0;
  for (int which = 0; which < 2; ++which)
    for (int e0 : kEs) {
      const int N = line_len(n, which);
      if (N < 2) continue;
      const int E = clampE(e0, N);
      for (int s = 1; s < num_stages(N, E); ++s) {
        const int R = 1 << stage_log2(N, E, s), NS = stage_ns(N, E, s);
        for (int r = 0; r < R; ++r)
          for (int j = 0; j < NS; ++j, ++idx) {
            const long double a = two_pi * (long double)((long long)j * r) / (long double)(NS * R);
            const long double c = cosl(a), sn = -sinl(a);
            if (precision_bits == 64) {
              double v[2] = {double(c), double(sn)};
              memcpy(static_cast<char*>(host) + idx * sizeof v, v, sizeof v);
            } else {
              float v[2] = {float(c), float(sn)};
              memcpy(static_cast<char*>(host) + idx * sizeof v, v, sizeof v);
            }
          }
      }
    }
}

}  // namespace arena_fft
