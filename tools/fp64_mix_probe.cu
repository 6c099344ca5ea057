// Does DFMA (FP64 CUDA-core FMA) add throughput on top of DMMA (FP64 tensor core) on B200 (sm_100a)?
// Register-only loops: (1) every warp interleaves NA DMMA.8x8x4 and NF DFMA per iteration; (2) warp
// specialisation: warps 0..W/2-1 run DMMA only, the rest DFMA only. Prints total FP64 TF/s.
// If the sum stays at the DMMA peak the two share the FP64 datapath and a hybrid K1 cannot go past it.
#include <cstdio>
#include <cuda_runtime.h>

template <int NA, int NF>
__global__ void mix_loop(double* out, int iters, int split) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NA > 0 ? NA : 1][2], f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (NA > 0 ? NA : 1); ++i) c[i][0] = c[i][1] = 0;
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = i;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool do_mma = !split || warp < nw / 2, do_fma = !split || warp >= nw / 2;
  for (int it = 0; it < iters; ++it) {
    if (do_mma) {
#pragma unroll
      for (int i = 0; i < NA; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    if (do_fma) {
#pragma unroll
      for (int i = 0; i < NF; ++i) f[i] = fma(a, f[i], b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NA; ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < NF; ++i) s += f[i];
  if (s == 12345.0) out[0] = s;
}

template <int NA, int NF>
void run(const char* name, double* d, int sms, int warps, int split) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  dim3 grid(sms * 2), block(32 * warps);
  mix_loop<NA, NF><<<grid, block>>>(d, 10, split);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    mix_loop<NA, NF><<<grid, block>>>(d, iters, split);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    if (cudaGetLastError() != cudaSuccess) {
      printf("{\"probe\": \"%s\", \"error\": \"launch failed\"}\n", name);
      return;
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double wm = split ? warps / 2 : warps, wf = split ? warps - warps / 2 : warps;
  const double fl_mma = 2.0 * 256.0 * NA * iters * (double)grid.x * wm;
  const double fl_fma = 2.0 * 32.0 * NF * iters * (double)grid.x * wf;
  printf("{\"probe\": \"%s\", \"dmma_per_iter\": %d, \"dfma_per_iter\": %d, \"warps\": %d, \"split\": %d, "
         "\"ms\": %.3f, \"dmma_tflops\": %.2f, \"dfma_tflops\": %.2f, \"total_tflops\": %.2f}\n",
         name, NA, NF, warps, split, best, fl_mma / best / 1e9, fl_fma / best / 1e9, (fl_mma + fl_fma) / best / 1e9);
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int sms = p.multiProcessorCount;
  run<16, 0>("dmma_only", d, sms, 8, 0);
  run<0, 16>("dfma_only", d, sms, 8, 0);
  run<16, 16>("interleaved", d, sms, 8, 0);
  run<16, 32>("interleaved", d, sms, 8, 0);
  run<16, 64>("interleaved", d, sms, 8, 0);
  run<16, 128>("interleaved", d, sms, 8, 0);
  run<8, 16>("interleaved", d, sms, 8, 0);
  run<16, 16>("warp_split", d, sms, 8, 1);
  run<16, 16>("warp_split", d, sms, 16, 1);
  run<16, 64>("warp_split", d, sms, 8, 1);
  return 0;
}
