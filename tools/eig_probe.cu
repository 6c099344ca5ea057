// eig_probe.cu -- times the k x k Hermitian eigensolve of Rayleigh-Ritz on the device: cuSOLVER ZHEEVD
// (divide and conquer, the default) against ZHEEVJ (Jacobi) on matrices shaped like the projected G of
// a ChFSI loop after the first (nearly diagonal: Ritz values on the diagonal + small coupling), and on a
// dense random Hermitian matrix (the first loop). Build: nvcc -O2 -arch=sm_100a tools/eig_probe.cu
// -lcusolver -o tools/eig_probe; run: tools/eig_probe k [coupling]
#include <cuComplex.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

int main(int argc, char** argv) {
  const int k = argc > 1 ? atoi(argv[1]) : 624;
  const double coupling = argc > 2 ? atof(argv[2]) : 1e-6;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd;
  std::vector<cuDoubleComplex> G((size_t)k * k);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i <= j; ++i) {
      cuDoubleComplex v = make_cuDoubleComplex(coupling * nd(rng), i == j ? 0.0 : coupling * nd(rng));
      if (i == j) v.x += -2.0 + 2.0 * j / k;  // Ritz values
      G[(size_t)j * k + i] = v;
      G[(size_t)i * k + j] = cuConj(v);
    }
  cusolverDnHandle_t h;
  cusolverDnCreate(&h);
  cuDoubleComplex *dA, *dG, *work;
  double* dW;
  int* info;
  cudaMalloc(&dA, sizeof(cuDoubleComplex) * k * k);
  cudaMalloc(&dG, sizeof(cuDoubleComplex) * k * k);
  cudaMalloc(&dW, sizeof(double) * k);
  cudaMalloc(&info, sizeof(int));
  cudaMemcpy(dG, G.data(), sizeof(cuDoubleComplex) * k * k, cudaMemcpyHostToDevice);
  int lwd = 0, lwj = 0;
  syevjInfo_t params;
  cusolverDnCreateSyevjInfo(&params);
  cusolverDnXsyevjSetTolerance(params, 1e-15);
  cusolverDnXsyevjSetMaxSweeps(params, 15);
  cusolverDnZheevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, k, dA, k, dW, &lwd);
  cusolverDnZheevj_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, k, dA, k, dW, &lwj, params);
  cudaMalloc(&work, sizeof(cuDoubleComplex) * (lwd > lwj ? lwd : lwj));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // 64-bit generic API (cusolverDnXsyevd) with the same matrix
  cusolverDnParams_t xp;
  cusolverDnCreateParams(&xp);
  size_t xdev = 0, xhost = 0;
  cusolverDnXsyevd_bufferSize(h, xp, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, k, CUDA_C_64F, dA, k, CUDA_R_64F,
                              dW, CUDA_C_64F, &xdev, &xhost);
  void* xwork = nullptr;
  cudaMalloc(&xwork, xdev > 0 ? xdev : 1);
  std::vector<char> hwork(xhost > 0 ? xhost : 1);
  for (int alg = 0; alg < 3; ++alg) {
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaMemcpy(dA, dG, sizeof(cuDoubleComplex) * k * k, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      if (alg == 0)
        cusolverDnZheevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, k, dA, k, dW, work, lwd, info);
      else if (alg == 1)
        cusolverDnZheevj(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, k, dA, k, dW, work, lwj, info, params);
      else
        cusolverDnXsyevd(h, xp, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, k, CUDA_C_64F, dA, k, CUDA_R_64F, dW,
                         CUDA_C_64F, xwork, xdev, hwork.data(), xhost, info);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    int hinfo = 0;
    cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost);
    int sweeps = 0;
    double res = 0;
    if (alg == 1) {
      cusolverDnXsyevjGetSweeps(h, params, &sweeps);
      cusolverDnXsyevjGetResidual(h, params, &res);
    }
    printf("{\"k\": %d, \"coupling\": %g, \"alg\": \"%s\", \"ms\": %.3f, \"info\": %d, \"sweeps\": %d, \"residual\": %.3g}\n",
           k, coupling, alg == 0 ? "zheevd" : alg == 1 ? "zheevj" : "Xsyevd", best, hinfo, sweeps, res);
  }
  return 0;
}
