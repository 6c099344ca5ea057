// filter_step_real.cu -- K1 instantiations, real-symmetric variants (ids 100..105, 132..135).
#include "filter_step_launch.cuh"

namespace chfsi {

cudaError_t launch_filter_real(int id, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                               const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream) {
#define LC(BM, BNC, WM, WNC, ST) launch_cfg<BM, BNC, WM, WNC, ST, kReal>(tmA, tmB, tmA3, tmB3, p, stream)
  switch (id) {
    case 104:
      return LC(128, 64, 32, 16, 4);
    case 132:  // 8 consumer warps + a producer warpgroup
      return launch_cfg<128, 32, 32, 16, 5, kReal, 1, 1, 2, 4>(tmA, tmB, tmA3, tmB3, p, stream);
    case 133:  // 12 consumer warps + a producer warpgroup
      return launch_cfg<192, 64, 32, 32, 3, kReal, 1, 1, 2, 4>(tmA, tmB, tmA3, tmB3, p, stream);
    case 135:  // 12 consumer warps + a producer warpgroup
      return launch_cfg<128, 48, 32, 16, 5, kReal, 1, 1, 2, 4>(tmA, tmB, tmA3, tmB3, p, stream);
#ifdef CHFSI_K1_AB
    case 102:  // 132 without the producer warpgroup (A/B)
      return LC(128, 32, 32, 16, 5);
    case 103:  // 133 without the producer warpgroup (A/B)
      return LC(192, 64, 32, 32, 3);
    case 105:  // 135 without the producer warpgroup (A/B)
      return LC(128, 48, 32, 16, 5);
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
