// filter_step_real.cu -- K1 instantiations, real-symmetric variants (ids 100..105).
#include "filter_step_launch.cuh"

namespace chfsi {

cudaError_t launch_filter_real(int id, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                               const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream) {
#define LC(BM, BNC, WM, WNC, ST) launch_cfg<BM, BNC, WM, WNC, ST, kReal>(tmA, tmB, tmA3, tmB3, p, stream)
  switch (id) {
    case 102:
      return LC(128, 32, 32, 16, 5);
    case 103:
      return LC(192, 64, 32, 32, 3);
    case 104:
      return LC(128, 64, 32, 16, 4);
    case 105:
      return LC(128, 48, 32, 16, 5);
#ifdef CHFSI_K1_AB
    case 100:
      return LC(128, 96, 32, 32, 3);
    case 101:
      return LC(128, 64, 32, 32, 4);
#endif
    default:
      return cudaErrorInvalidValue;
  }
#undef LC
}

}  // namespace chfsi
