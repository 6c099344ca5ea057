// blas_traits.cuh -- scalar traits over the library calls of the supporting steps (cuBLAS / cuSOLVER):
// complex Hermitian (cuDoubleComplex, the north-star path) or real symmetric (double, SURVEY 8(f)
// NEXT-3), plus the status-marshalling macros shared by supporting.cu and eig_refine.cu.
#pragma once
#include <cublas_v2.h>
#include <cuComplex.h>
#include <cusolverDn.h>

#include <string>

#include "ctx.cuh"

namespace chfsi {

#define CUBLAS_TRY(ctx, call)                                                   \
  do {                                                                          \
    cublasStatus_t _s = (call);                                                 \
    if (_s != CUBLAS_STATUS_SUCCESS) {                                          \
      set_err(ctx, std::string(#call) + ": cuBLAS status " + std::to_string((int)_s)); \
      return CHFSI_ERR_CUDA;                                                    \
    }                                                                           \
  } while (0)
#define CUSOLVER_TRY(ctx, call)                                                 \
  do {                                                                          \
    cusolverStatus_t _s = (call);                                               \
    if (_s != CUSOLVER_STATUS_SUCCESS) {                                        \
      set_err(ctx, std::string(#call) + ": cuSOLVER status " + std::to_string((int)_s)); \
      return CHFSI_ERR_CUDA;                                                    \
    }                                                                           \
  } while (0)
#define TRY(x)                   \
  do {                           \
    chfsi_status _st = (x);      \
    if (_st != CHFSI_OK) return _st; \
  } while (0)

// D is the element type of the library's small kernels.
template <typename T>
struct Sc;
template <>
struct Sc<cuDoubleComplex> {
  using T = cuDoubleComplex;
  using D = double2;
  static constexpr int elem = 2;
  static constexpr cublasOperation_t opH = CUBLAS_OP_C;
  static T one() { return {1.0, 0.0}; }
  static T zero() { return {0.0, 0.0}; }
  static T mone() { return {-1.0, 0.0}; }
  // the n k^2-class products of QR / Rayleigh-Ritz: cuBLAS ZGEMM, or its Gauss 3M form (ZGEMM3M) when the
  // context runs the filter in 3M (the same arithmetic, 25 % fewer real multiplications)
  static cublasStatus_t gemm(chfsi_ctx ctx, cublasOperation_t a, cublasOperation_t b, int m, int n, int k,
                             const T* al, const T* A, int lda, const T* B, int ldb, const T* be, T* C, int ldc) {
    if (ctx->zmul == 3) return cublasZgemm3m(ctx->cublas, a, b, m, n, k, al, A, lda, B, ldb, be, C, ldc);
    return cublasZgemm(ctx->cublas, a, b, m, n, k, al, A, lda, B, ldb, be, C, ldc);
  }
  static cublasStatus_t gemv(cublasHandle_t h, cublasOperation_t a, int m, int n, const T* al, const T* A, int lda,
                             const T* x, const T* be, T* y) {
    return cublasZgemv(h, a, m, n, al, A, lda, x, 1, be, y, 1);
  }
  static cublasStatus_t trsm_ru(cublasHandle_t h, int m, int n, const T* R, int ldr, T* Y, int ldy) {
    const T o = one();
    return cublasZtrsm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, n, &o, R, ldr,
                       Y, ldy);
  }
  static cusolverStatus_t potrf_bs(cusolverDnHandle_t h, int n, T* A, int lda, int* lw) {
    return cusolverDnZpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, n, A, lda, lw);
  }
  static cusolverStatus_t potrf(cusolverDnHandle_t h, int n, T* A, int lda, T* w, int lw, int* info) {
    return cusolverDnZpotrf(h, CUBLAS_FILL_MODE_UPPER, n, A, lda, w, lw, info);
  }
  static cusolverStatus_t heevd_bs(cusolverDnHandle_t h, int n, T* A, int lda, double* W, int* lw) {
    return cusolverDnZheevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A, lda, W, lw);
  }
  static cusolverStatus_t heevd(cusolverDnHandle_t h, int n, T* A, int lda, double* W, T* w, int lw, int* info) {
    return cusolverDnZheevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A, lda, W, w, lw, info);
  }
  static cusolverStatus_t geqrf_bs(cusolverDnHandle_t h, int m, int n, T* A, int lda, int* lw) {
    return cusolverDnZgeqrf_bufferSize(h, m, n, A, lda, lw);
  }
  static cusolverStatus_t geqrf(cusolverDnHandle_t h, int m, int n, T* A, int lda, T* tau, T* w, int lw, int* info) {
    return cusolverDnZgeqrf(h, m, n, A, lda, tau, w, lw, info);
  }
  static cusolverStatus_t orgqr_bs(cusolverDnHandle_t h, int m, int n, T* A, int lda, const T* tau, int* lw) {
    return cusolverDnZungqr_bufferSize(h, m, n, n, A, lda, tau, lw);
  }
  static cusolverStatus_t orgqr(cusolverDnHandle_t h, int m, int n, T* A, int lda, const T* tau, T* w, int lw,
                                int* info) {
    return cusolverDnZungqr(h, m, n, n, A, lda, tau, w, lw, info);
  }
  // upper triangle of C = A^H A (n x n; A is k x n)
  static cublasStatus_t herk_c(cublasHandle_t h, int n, int k, const T* A, int lda, T* C, int ldc) {
    const double o = 1.0, z = 0.0;
    return cublasZherk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, n, k, &o, A, lda, &z, C, ldc);
  }
  // upper triangle of C = A^H B for a product known to be Hermitian (A, B k x n)
  static cublasStatus_t herkx_c(cublasHandle_t h, int n, int k, const T* A, int lda, const T* B, int ldb, T* C,
                                int ldc) {
    const T o = one();
    const double z = 0.0;
    return cublasZherkx(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_C, n, k, &o, A, lda, B, ldb, &z, C, ldc);
  }
  static double re(const T& x) { return x.x; }
};
template <>
struct Sc<double> {
  using T = double;
  using D = double;
  static constexpr int elem = 1;
  static constexpr cublasOperation_t opH = CUBLAS_OP_T;
  static T one() { return 1.0; }
  static T zero() { return 0.0; }
  static T mone() { return -1.0; }
  static cublasStatus_t gemm(chfsi_ctx ctx, cublasOperation_t a, cublasOperation_t b, int m, int n, int k,
                             const T* al, const T* A, int lda, const T* B, int ldb, const T* be, T* C, int ldc) {
    return cublasDgemm(ctx->cublas, a, b, m, n, k, al, A, lda, B, ldb, be, C, ldc);
  }
  static cublasStatus_t gemv(cublasHandle_t h, cublasOperation_t a, int m, int n, const T* al, const T* A, int lda,
                             const T* x, const T* be, T* y) {
    return cublasDgemv(h, a, m, n, al, A, lda, x, 1, be, y, 1);
  }
  static cublasStatus_t trsm_ru(cublasHandle_t h, int m, int n, const T* R, int ldr, T* Y, int ldy) {
    const T o = one();
    return cublasDtrsm(h, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, m, n, &o, R, ldr,
                       Y, ldy);
  }
  static cusolverStatus_t potrf_bs(cusolverDnHandle_t h, int n, T* A, int lda, int* lw) {
    return cusolverDnDpotrf_bufferSize(h, CUBLAS_FILL_MODE_UPPER, n, A, lda, lw);
  }
  static cusolverStatus_t potrf(cusolverDnHandle_t h, int n, T* A, int lda, T* w, int lw, int* info) {
    return cusolverDnDpotrf(h, CUBLAS_FILL_MODE_UPPER, n, A, lda, w, lw, info);
  }
  static cusolverStatus_t heevd_bs(cusolverDnHandle_t h, int n, T* A, int lda, double* W, int* lw) {
    return cusolverDnDsyevd_bufferSize(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A, lda, W, lw);
  }
  static cusolverStatus_t heevd(cusolverDnHandle_t h, int n, T* A, int lda, double* W, T* w, int lw, int* info) {
    return cusolverDnDsyevd(h, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, n, A, lda, W, w, lw, info);
  }
  static cusolverStatus_t geqrf_bs(cusolverDnHandle_t h, int m, int n, T* A, int lda, int* lw) {
    return cusolverDnDgeqrf_bufferSize(h, m, n, A, lda, lw);
  }
  static cusolverStatus_t geqrf(cusolverDnHandle_t h, int m, int n, T* A, int lda, T* tau, T* w, int lw, int* info) {
    return cusolverDnDgeqrf(h, m, n, A, lda, tau, w, lw, info);
  }
  static cusolverStatus_t orgqr_bs(cusolverDnHandle_t h, int m, int n, T* A, int lda, const T* tau, int* lw) {
    return cusolverDnDorgqr_bufferSize(h, m, n, n, A, lda, tau, lw);
  }
  static cusolverStatus_t orgqr(cusolverDnHandle_t h, int m, int n, T* A, int lda, const T* tau, T* w, int lw,
                                int* info) {
    return cusolverDnDorgqr(h, m, n, n, A, lda, tau, w, lw, info);
  }
  static cublasStatus_t herk_c(cublasHandle_t h, int n, int k, const T* A, int lda, T* C, int ldc) {
    const double o = 1.0, z = 0.0;
    return cublasDsyrk(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, n, k, &o, A, lda, &z, C, ldc);
  }
  static cublasStatus_t herkx_c(cublasHandle_t h, int n, int k, const T* A, int lda, const T* B, int ldb, T* C,
                                int ldc) {
    const double o = 1.0, z = 0.0;
    return cublasDsyrkx(h, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T, n, k, &o, A, lda, B, ldb, &z, C, ldc);
  }
  static double re(const T& x) { return x; }
};


}  // namespace chfsi
