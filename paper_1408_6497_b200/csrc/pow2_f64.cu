// fp64 instantiation of the power-of-two path (the reference's precision).
#include "pow2_launch.cuh"

namespace arena_fft {
cudaError_t launch_pow2_f64(const Pow2Args& a) { return launch_pow2<double>(a); }
}  // namespace arena_fft
