// generalized.cu -- the generalised front / back end: Cholesky of B,
// H = L^{-1} A L^{-H}, and the back-transformation c = L^{-H} y. The n^3 steps are plain library
// calls (cuSOLVER ZPOTRF, cuBLAS ZTRSM); the Hermitisation is the library's own kernel.
#include <algorithm>

#include "ctx.cuh"
#include "small_kernels.cuh"

using namespace chfsi;

static const cuDoubleComplex kOne = {1.0, 0.0};

extern "C" {

chfsi_status chfsi_reduce_generalized(chfsi_ctx ctx, int64_t n, void* A, int64_t lda, void* B, int64_t ldb) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || !A || !B || lda < n || ldb < n || ctx->nranks != 1 || n > INT32_MAX) {
    set_err(ctx, "chfsi_reduce_generalized: bad arguments (single rank only)");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  cuDoubleComplex* a = static_cast<cuDoubleComplex*>(A);
  cuDoubleComplex* b = static_cast<cuDoubleComplex*>(B);
  int lw = 0;
  if (cusolverDnZpotrf_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, (int)n, b, (int)ldb, &lw) !=
      CUSOLVER_STATUS_SUCCESS) {
    set_err(ctx, "cusolverDnZpotrf_bufferSize failed");
    return CHFSI_ERR_CUDA;
  }
  chfsi_status st = ensure(ctx, ctx->solver_ws, sizeof(cuDoubleComplex) * (size_t)std::max(lw, 1));
  if (!st) st = ensure(ctx, ctx->devinfo, 64);
  if (st) return st;
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  if (cusolverDnZpotrf(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, (int)n, b, (int)ldb,
                       static_cast<cuDoubleComplex*>(ctx->solver_ws.ptr), lw, info) != CUSOLVER_STATUS_SUCCESS) {
    set_err(ctx, "cusolverDnZpotrf failed");
    return CHFSI_ERR_CUDA;
  }
  int hinfo = 0;
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) {
    set_err(ctx, "chfsi_reduce_generalized: B is not positive definite (pivot " + std::to_string(hinfo - 1) + ")");
    return CHFSI_ERR_ARG;
  }
  // A <- L^{-1} A, then A <- A L^{-H}
  if (cublasZtrsm(ctx->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, (int)n,
                  (int)n, &kOne, b, (int)ldb, a, (int)lda) != CUBLAS_STATUS_SUCCESS ||
      cublasZtrsm(ctx->cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, (int)n,
                  (int)n, &kOne, b, (int)ldb, a, (int)lda) != CUBLAS_STATUS_SUCCESS) {
    set_err(ctx, "cublasZtrsm failed");
    return CHFSI_ERR_CUDA;
  }
  CHFSI_CUDA_TRY(ctx, launch_hermitize(n, static_cast<double2*>(A), lda, ctx->stream));
  ctx->launches++;
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return CHFSI_OK;
}

chfsi_status chfsi_back_transform(chfsi_ctx ctx, int64_t n, const void* L, int64_t ldl, void* X, int64_t ldx,
                                  int64_t k) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || k < 0 || !L || (k > 0 && !X) || ldl < n || ldx < n || ctx->nranks != 1) {
    set_err(ctx, "chfsi_back_transform: bad arguments (single rank only)");
    return CHFSI_ERR_ARG;
  }
  if (k == 0) return CHFSI_OK;
  cudaSetDevice(ctx->device);
  if (cublasZtrsm(ctx->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, (int)n,
                  (int)k, &kOne, static_cast<const cuDoubleComplex*>(L), (int)ldl, static_cast<cuDoubleComplex*>(X),
                  (int)ldx) != CUBLAS_STATUS_SUCCESS) {
    set_err(ctx, "cublasZtrsm failed");
    return CHFSI_ERR_CUDA;
  }
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return CHFSI_OK;
}

}  // extern "C"
