// fp32 instantiation of the power-of-two path (BASELINE config 5 precision trade-off).
#include "pow2_launch.cuh"

namespace arena_fft {
cudaError_t launch_pow2_f32(const Pow2Args& a) { return launch_pow2<float>(a); }
cudaError_t launch_split3_f32(const Split3Args& a) { return launch_split3<float>(a); }
bool pow2_config_f32(int n, KernelGeom* g) { return pow2_config<float>(n, g); }
bool pow2_fused_ok_f32(int n) {
  switch (n) {
    case 256: return FusedCfg<float, 256>::OK;
    case 512: return FusedCfg<float, 512>::OK;
    case 1024: return FusedCfg<float, 1024>::OK;
    case 2048: return FusedCfg<float, 2048>::OK;
    default: return false;
  }
}
cudaError_t pencil_phase_f32(const PencilArgs& a, int phase) { return pencil_phase<float>(a, phase); }
}  // namespace arena_fft
