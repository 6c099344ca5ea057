// filter_step_z4.cu -- K1 instantiations, complex 4M real-embedding variants (ids 0..15).
#include "filter_step_launch.cuh"

namespace chfsi {

cudaError_t launch_filter_z4(int id, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                             const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream) {
#define LC(BM, BNC, WM, WNC, ST) launch_cfg<BM, BNC, WM, WNC, ST, kZ4M>(tmA, tmB, tmA3, tmB3, p, stream)
  switch (id) {
    case 1:
      return LC(64, 64, 32, 16, 6);
    case 3:
      return LC(64, 32, 32, 16, 8);
    case 5:
      return LC(128, 16, 16, 16, 6);
    case 6:
      return LC(128, 32, 32, 8, 5);
    case 7:
      return LC(128, 48, 32, 16, 4);
    case 9:
      return LC(256, 32, 64, 16, 3);
    case 10:
      return LC(256, 4, 32, 4, 3);
    case 11:
      return LC(128, 8, 32, 4, 6);
    case 12:
      return LC(128, 12, 32, 4, 6);
    case 13:
      return LC(256, 8, 32, 4, 3);
    case 14:
      return LC(256, 12, 64, 4, 3);
#ifdef CHFSI_K1_AB
    case 0:
      return LC(128, 32, 32, 16, 5);
    case 2:
      return LC(128, 64, 32, 32, 4);
    case 4:
      return LC(128, 64, 32, 16, 4);
    case 8:
      return LC(128, 64, 64, 16, 4);
    case 15:
      return LC(256, 8, 64, 4, 3);
#endif
    default:
      return cudaErrorInvalidValue;
  }
#undef LC
}

}  // namespace chfsi
