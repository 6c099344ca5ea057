// filter_step_z3.cu -- K1 instantiations, complex Gauss 3M variants (ids >= 200).
#include "filter_step_launch.cuh"

namespace chfsi {

cudaError_t launch_filter_z3(int id, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                             const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream) {
#define LC(BM, BNC, WM, WNC, ST) launch_cfg<BM, BNC, WM, WNC, ST, kZ3M>(tmA, tmB, tmA3, tmB3, p, stream)
  switch (id) {
    case 200:  // the workhorse: 12 consumer warps + a producer warpgroup
      return launch_cfg<128, 48, 32, 16, 3, kZ3M, 1, 1, 2, 4>(tmA, tmB, tmA3, tmB3, p, stream);
    case 207:
      return LC(64, 64, 16, 16, 4);
    case 208:
      return LC(128, 32, 32, 8, 3);
#ifdef CHFSI_K1_AB
    case 239:  // z200 without the producer warpgroup (thread 0 produces; the round-1 workhorse)
      return LC(128, 48, 32, 16, 3);
    case 201:
      return LC(128, 32, 32, 16, 3);
    case 202:
      return LC(128, 16, 32, 8, 3);
    case 203:
      return LC(64, 64, 32, 16, 4);
    case 204:
      return LC(192, 32, 32, 16, 2);
    case 209:
      return LC(128, 48, 32, 16, 2);
    case 210:
      return launch_cfg<128, 48, 32, 16, 3, kZ3M, 2>(tmA, tmB, tmA3, tmB3, p, stream);
    case 220:
      return launch_cfg<128, 48, 32, 16, 6, kZ3M, 1, 1, 1>(tmA, tmB, tmA3, tmB3, p, stream);
    case 227:
      return launch_cfg<64, 64, 16, 16, 8, kZ3M, 1, 1, 1>(tmA, tmB, tmA3, tmB3, p, stream);
    case 206:
      return launch_cfg<64, 48, 32, 16, 2, kZ3M, 1, 2>(tmA, tmB, tmA3, tmB3, p, stream);
#endif
    default:
      return cudaErrorInvalidValue;
  }
#undef LC
}

}  // namespace chfsi
