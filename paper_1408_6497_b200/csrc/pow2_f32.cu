// fp32 instantiation of the power-of-two path (BASELINE config 5 precision trade-off).
#include "pow2_launch.cuh"

namespace arena_fft {
cudaError_t launch_pow2_f32(const Pow2Args& a) { return launch_pow2<float>(a); }
bool pow2_config_f32(int n, KernelGeom* g) { return pow2_config<float>(n, g); }
}  // namespace arena_fft
