// FP64 peak probe for B200 (sm_100a): register-only DMMA (mma.sync m8n8k4 f64) and DFMA loops.
// Used once to establish the FP64 roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

template <int NACC>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d; cudaMalloc(&d, 8);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %zu, \"regs_per_sm\": %d}\n",
         p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.regsPerMultiprocessor);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16}) {
    for (int rep = 0; rep < 3; ++rep) {
      int iters = 20000;
      dim3 grid(sms * 2), block(32 * warps);
      dmma_loop<16><<<grid, block>>>(d, 10);
      cudaEventRecord(e0);
      dmma_loop<16><<<grid, block>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256.0 * 16 * iters * (double)grid.x * warps;
      printf("{\"probe\": \"dmma_m8n8k4\", \"warps_per_cta\": %d, \"ctas\": %d, \"tflops\": %.2f}\n", warps, grid.x, flops / ms / 1e9);
    }
  }
  for (int warps : {8, 16, 32}) {
    for (int rep = 0; rep < 3; ++rep) {
      int iters = 20000;
      dim3 grid(sms * 2), block(32 * warps);
      dfma_loop<16><<<grid, block>>>(d, 10);
      cudaEventRecord(e0);
      dfma_loop<16><<<grid, block>>>(d, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * iters * (double)grid.x * warps * 32;
      printf("{\"probe\": \"dfma\", \"warps_per_cta\": %d, \"ctas\": %d, \"tflops\": %.2f}\n", warps, grid.x, flops / ms / 1e9);
    }
  }
  // sustained DMMA for ~4 s to see clocks under FP64 load
  {
    dim3 grid(sms * 2), block(32 * 8);
    cudaEventRecord(e0);
    for (int r = 0; r < 40; ++r) dmma_loop<16><<<grid, block>>>(d, 20000);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 40 * 2.0 * 256.0 * 16 * 20000 * (double)grid.x * 8;
    printf("{\"probe\": \"dmma_sustained\", \"seconds\": %.2f, \"tflops\": %.2f}\n", ms / 1e3, flops / ms / 1e9);
  }
  return 0;
}
