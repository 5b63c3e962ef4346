// fp64 instantiation of the power-of-two path (the reference's precision).
#include "pow2_launch.cuh"

namespace arena_fft {
cudaError_t launch_pow2_f64(const Pow2Args& a) { return launch_pow2<double>(a); }
cudaError_t launch_split3_f64(const Split3Args& a) { return launch_split3<double>(a); }
bool pow2_config_f64(int n, KernelGeom* g) { return pow2_config<double>(n, g); }
bool pow2_fused_ok_f64(int n) {
  switch (n) {
    case 256: return FusedCfg<double, 256>::OK;
    case 512: return FusedCfg<double, 512>::OK;
    case 1024: return FusedCfg<double, 1024>::OK;
    case 2048: return FusedCfg<double, 2048>::OK;
    default: return false;
  }
}
cudaError_t pencil_phase_f64(const PencilArgs& a, int phase) { return pencil_phase<double>(a, phase); }
}  // namespace arena_fft
