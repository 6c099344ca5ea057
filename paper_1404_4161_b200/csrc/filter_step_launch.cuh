// filter_step_launch.cuh -- the launcher template of K1 (one instantiation per tile variant). The
// instantiations are spread over filter_step_{z3,z4,real}.cu so they compile in parallel.
#pragma once
#include <atomic>

#include "filter_step.cuh"

namespace chfsi {

template <int BM, int BNC, int WM, int WNC, int STAGES, int MODE = kZ4M, int CL = 1, int OCC = 1, int KH = 2,
          int PW = 0>
inline cudaError_t launch_cfg(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                       const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream) {
  using Cfg = FilterCfg<BM, BNC, WM, WNC, STAGES, MODE, CL, KH, PW>;
  auto kern = filter_step_kernel<BM, BNC, WM, WNC, STAGES, MODE, CL, OCC, KH, PW>;
  // the opt-in shared-memory size is a per-device function attribute: set it once per device (contexts
  // on several host threads may launch the same instantiation concurrently)
  static std::atomic<uint64_t> attr_devices{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_devices.load(std::memory_order_acquire) & bit)) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    if (e != cudaSuccess) return e;
    if constexpr (PW > 0) {  // the producer warpgroup hands its registers to the consumers (setmaxnreg): the
      // launch allocation must be the one the kernel's arithmetic assumed, or the consumers' increase blocks
      cudaFuncAttributes fa;
      e = cudaFuncGetAttributes(&fa, kern);
      if (e != cudaSuccess) return e;
      if (fa.numRegs != (65536 / Cfg::kThreads) / 8 * 8) return cudaErrorInvalidConfiguration;
    }
    attr_devices.fetch_or(bit, std::memory_order_release);
  }
  if constexpr (CL == 1) {
    kern<<<p.grid, Cfg::kThreads, Cfg::kSmemBytes, stream>>>(tmA, tmB, tmA3, tmB3, p);
    return cudaGetLastError();
  } else {  // p.grid counts clusters
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.grid * CL));
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmA3, tmB3, p);
  }
}

// per-family dispatch (filter_step_{z3,z4,real}.cu): cudaErrorInvalidValue for an id not built
cudaError_t launch_filter_z3(int id, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                             const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream);
cudaError_t launch_filter_z4(int id, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                             const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream);
cudaError_t launch_filter_real(int id, const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                               const CUtensorMap& tmB3, const StepParams& p, cudaStream_t stream);

}  // namespace chfsi
