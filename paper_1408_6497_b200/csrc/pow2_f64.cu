// fp64 instantiation of the power-of-two path (the reference's precision).
#include "pow2_launch.cuh"

namespace arena_fft {
cudaError_t launch_pow2_f64(const Pow2Args& a) { return launch_pow2<double>(a); }
bool pow2_config_f64(int n, KernelGeom* g) { return pow2_config<double>(n, g); }
}  // namespace arena_fft
