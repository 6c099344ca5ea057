// generalized.cu -- the generalised front / back end: Cholesky of B,
// H = L^{-1} A L^{-H}, and the back-transformation c = L^{-H} y. The n^3 steps are plain library
// calls (cuSOLVER ZPOTRF, cuBLAS ZTRSM / ZGEMM); the Hermitisation is the library's own kernel. The
// row-panel forms (p >= 1) factor B on the ranks' column slabs (right-looking panels, broadcast over the
// communicator), gather L and A and compute each rank's columns of H with O(n^2 n_loc) work.
#include <algorithm>
#include <string>
#include <vector>

#include "ctx.cuh"
#include "small_kernels.cuh"

using namespace chfsi;

#define TRY(x)                       \
  do {                               \
    chfsi_status _st = (x);          \
    if (_st != CHFSI_OK) return _st; \
  } while (0)

static const cuDoubleComplex kOne = {1.0, 0.0};
static const cuDoubleComplex kZero = {0.0, 0.0};

namespace {

// X (n x nloc) <- columns row0 .. row0 + nloc - 1 of the identity
__global__ void unit_cols_kernel(int64_t n, int64_t nloc, int64_t row0, double2* X, int64_t ldx) {
  for (int64_t j = blockIdx.y; j < nloc; j += gridDim.y)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      X[j * ldx + i] = make_double2(i == row0 + j ? 1.0 : 0.0, 0.0);
}

// Hp[:, j] <- column row0 + j of (W + W^H) / 2, W the gathered n x n matrix: the (i, c) entry computed
// here and the (c, i) entry computed by the rank that owns column i are exact conjugates (the same
// two operands, added in either order), so the assembled H is Hermitian bit for bit (R13)
__global__ void hermitize_panel_kernel(int64_t n, int64_t nloc, int64_t row0, const double2* __restrict__ W,
                                       int64_t ldw, double2* Hp, int64_t ldh) {
  for (int64_t j = blockIdx.y; j < nloc; j += gridDim.y) {
    const int64_t c = row0 + j;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const double2 a = W[c * ldw + i], b = W[i * ldw + c];
      Hp[j * ldh + i] = i == c ? make_double2(a.x, 0.0) : make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
    }
  }
}

// grid over (rows, columns): <= 64 row blocks of 256 threads, <= 65535 column blocks (grid-stride beyond)
dim3 col_grid(int64_t n, int64_t cols) {
  return dim3((unsigned)std::min<int64_t>((n + 255) / 256, 64), (unsigned)std::min<int64_t>(cols, 65535));
}

// W (n x n, ld n) <- the p column slabs S_q (n x nloc) of all ranks: this rank's slab is copied into its
// column range, then one in-place allgather
chfsi_status gather_slabs(chfsi_ctx ctx, int64_t n, int64_t nloc, const void* S, int64_t lds, double2* W) {
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(W + n * nloc * ctx->rank, 16 * n, S, 16 * lds, 16 * n, nloc,
                                        cudaMemcpyDeviceToDevice, ctx->stream));
  return comm_allgather_inplace(ctx, reinterpret_cast<double*>(W), (size_t)2 * n * nloc);
}

// B = L L^H factored on the column slabs (rank q owns global columns [q nloc, (q+1) nloc)): right-looking,
// in panels of <= kPanel columns that never straddle a slab. The owner factors the panel's diagonal block
// (ZPOTRF) and solves the rows below it (ZTRSM), the panel (rows j0..n-1) is broadcast, and every rank
// updates its own trailing columns (ZGEMM). Lp (n x nloc, ld n) in: this rank's slab of B; out: its slab
// of L in the lower triangle (the strict upper part is unspecified). *bad <- the first failing global
// pivot + 1 of this rank's panels, or 0.
constexpr int64_t kPanel = 256;

chfsi_status cholesky_slabs(chfsi_ctx ctx, int64_t n, int64_t nloc, cuDoubleComplex* Lp, int64_t* bad) {
  const int64_t q0 = nloc * ctx->rank;  // this rank's first global column
  *bad = 0;
  TRY(ensure(ctx, ctx->w1, 16 * (size_t)n * (size_t)std::min(kPanel, nloc)));
  TRY(ensure(ctx, ctx->devinfo, 64));
  cuDoubleComplex* P = static_cast<cuDoubleComplex*>(ctx->w1.ptr);
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  static const cuDoubleComplex kMone = {-1.0, 0.0};
  for (int64_t j0 = 0; j0 < n;) {
    const int64_t owner = j0 / nloc, slab_end = (owner + 1) * nloc;
    const int64_t jb = std::min(kPanel, slab_end - j0);
    const int64_t below = n - j0 - jb;
    if (owner == ctx->rank) {
      cuDoubleComplex* D = Lp + (j0 - q0) * n + j0;  // diagonal block, ld n
      int lw = 0;
      if (cusolverDnZpotrf_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, (int)jb, D, (int)n, &lw) !=
          CUSOLVER_STATUS_SUCCESS) {
        set_err(ctx, "cusolverDnZpotrf_bufferSize failed");
        return CHFSI_ERR_CUDA;
      }
      TRY(ensure(ctx, ctx->solver_ws, sizeof(cuDoubleComplex) * (size_t)std::max(lw, 1)));
      if (cusolverDnZpotrf(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, (int)jb, D, (int)n,
                           static_cast<cuDoubleComplex*>(ctx->solver_ws.ptr), lw, info) != CUSOLVER_STATUS_SUCCESS ||
          (below > 0 && cublasZtrsm(ctx->cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C,
                                    CUBLAS_DIAG_NON_UNIT, (int)below, (int)jb, &kOne, D, (int)n, D + jb, (int)n) !=
                            CUBLAS_STATUS_SUCCESS)) {
        set_err(ctx, "distributed Cholesky: cuSOLVER / cuBLAS failed");
        return CHFSI_ERR_CUDA;
      }
      int hinfo = 0;
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      if (hinfo > 0 && *bad == 0) *bad = j0 + hinfo;
      // the panel's rows j0..n-1, packed (ld n - j0)
      CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(P, 16 * (n - j0), D, 16 * n, 16 * (n - j0), jb, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
    }
    TRY(comm_bcast(ctx, reinterpret_cast<double*>(P), (size_t)2 * (n - j0) * jb, (int)owner));
    // trailing update of this rank's columns c >= j0 + jb, rows c0..n-1 (the lower part and the slab's
    // diagonal blocks): L[c0:, cols] -= P[c0 - j0:, :] P[cols - j0, :]^H
    const int64_t c0 = std::max(j0 + jb, q0), c1 = q0 + nloc;
    if (c0 < c1 && c0 < n) {
      const cuDoubleComplex* Pr = P + (c0 - j0);
      if (cublasZgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_C, (int)(n - c0), (int)(c1 - c0), (int)jb, &kMone, Pr,
                      (int)(n - j0), Pr, (int)(n - j0), &kOne, Lp + (c0 - q0) * n + c0, (int)n) != CUBLAS_STATUS_SUCCESS) {
        set_err(ctx, "distributed Cholesky: cublasZgemm failed");
        return CHFSI_ERR_CUDA;
      }
    }
    j0 += jb;
  }
  return CHFSI_OK;
}

bool panel_args_ok(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc) {
  return n >= 1 && n <= INT32_MAX && nloc >= 1 && nloc * ctx->nranks == n && row0 == nloc * ctx->rank;
}

}  // namespace

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

chfsi_status chfsi_reduce_generalized_panel(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, void* Ap,
                                            int64_t lda, const void* Bp, int64_t ldb, void* L, int64_t ldl) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (!panel_args_ok(ctx, n, row0, nloc) || !Ap || !Bp || !L || lda < n || ldb < n || ldl < n) {
    set_err(ctx, "chfsi_reduce_generalized_panel: bad arguments");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  chfsi_status st = ensure(ctx, ctx->gw, 16 * (size_t)n * n);
  if (!st) st = ensure(ctx, ctx->gx, 16 * (size_t)n * nloc);
  if (!st) st = ensure(ctx, ctx->devinfo, 64);
  if (!st) st = ensure(ctx, ctx->small2, sizeof(double) * (size_t)std::max(8, ctx->nranks));
  if (st) return st;
  double2* W = static_cast<double2*>(ctx->gw.ptr);
  cuDoubleComplex* w = static_cast<cuDoubleComplex*>(ctx->gw.ptr);
  cuDoubleComplex* X = static_cast<cuDoubleComplex*>(ctx->gx.ptr);
  cuDoubleComplex* l = static_cast<cuDoubleComplex*>(L);
  cuDoubleComplex* a = static_cast<cuDoubleComplex*>(Ap);
  const int ni = (int)n, nl = (int)nloc;
  // B = L L^H. p > 1: factored on the slabs (cholesky_slabs: every rank factors and updates its own
  // columns, ZPOTRF work shared) and gathered, so every rank holds the same bits of L; p = 1: one ZPOTRF.
  double* dflag = static_cast<double*>(ctx->small2.ptr);
  double hflag = 0.0;
  if (ctx->nranks > 1) {
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(X, 16 * n, Bp, 16 * ldb, 16 * n, nloc, cudaMemcpyDeviceToDevice,
                                          ctx->stream));
    int64_t bad = 0;
    TRY(cholesky_slabs(ctx, n, nloc, X, &bad));
    // every rank learns every rank's verdict (the collectives stay matched): slot r holds rank r's first
    // failing pivot + 1; the smallest non-zero one is reported
    std::vector<double> flags(ctx->nranks, 0.0);
    flags[ctx->rank] = (double)bad;
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(dflag, flags.data(), sizeof(double) * flags.size(), cudaMemcpyHostToDevice,
                                        ctx->stream));
    TRY(comm_allreduce_sum(ctx, dflag, flags.size()));
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(flags.data(), dflag, sizeof(double) * flags.size(), cudaMemcpyDeviceToHost,
                                        ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    for (double f : flags)
      if (f != 0.0 && (hflag == 0.0 || f < hflag)) hflag = f;
    if (hflag != 0.0) {
      set_err(ctx, "chfsi_reduce_generalized_panel: B is not positive definite (pivot " +
                       std::to_string((long long)hflag - 1) + ")");
      return CHFSI_ERR_ARG;
    }
    TRY(gather_slabs(ctx, n, nloc, X, n, W));
  } else {
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(W, 16 * n, Bp, 16 * ldb, 16 * n, n, cudaMemcpyDeviceToDevice, ctx->stream));
  }
  if (ctx->nranks == 1) {
    int lw = 0;
    if (cusolverDnZpotrf_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, w, ni, &lw) != CUSOLVER_STATUS_SUCCESS) {
      set_err(ctx, "cusolverDnZpotrf_bufferSize failed");
      return CHFSI_ERR_CUDA;
    }
    TRY(ensure(ctx, ctx->solver_ws, sizeof(cuDoubleComplex) * (size_t)std::max(lw, 1)));
    int* info = static_cast<int*>(ctx->devinfo.ptr);
    if (cusolverDnZpotrf(ctx->cusolver, CUBLAS_FILL_MODE_LOWER, ni, w, ni,
                         static_cast<cuDoubleComplex*>(ctx->solver_ws.ptr), lw, info) != CUSOLVER_STATUS_SUCCESS) {
      set_err(ctx, "cusolverDnZpotrf failed");
      return CHFSI_ERR_CUDA;
    }
    int hinfo = 0;
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    hflag = (double)hinfo;
  }
  if (ctx->nranks == 1 && hflag != 0.0) {
    set_err(ctx, "chfsi_reduce_generalized_panel: B is not positive definite (pivot " +
                     std::to_string((long long)hflag - 1) + ")");
    return CHFSI_ERR_ARG;
  }
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(L, 16 * ldl, W, 16 * n, 16 * n, n, cudaMemcpyDeviceToDevice, ctx->stream));
  // this rank's columns of H = L^{-1} A L^{-H}: X = L^{-H} E_cols, then L^{-1} (A X)
  unit_cols_kernel<<<col_grid(n, nloc), 256, 0, ctx->stream>>>(n, nloc, row0, reinterpret_cast<double2*>(X), n);
  CHFSI_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches++;
  TRY(gather_slabs(ctx, n, nloc, Ap, lda, W));  // the whole A
  if (cublasZtrsm(ctx->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, ni, nl,
                  &kOne, l, (int)ldl, X, ni) != CUBLAS_STATUS_SUCCESS ||
      cublasZgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, ni, nl, ni, &kOne, w, ni, X, ni, &kZero, a, (int)lda) !=
          CUBLAS_STATUS_SUCCESS ||
      cublasZtrsm(ctx->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, ni, nl,
                  &kOne, l, (int)ldl, a, (int)lda) != CUBLAS_STATUS_SUCCESS) {
    set_err(ctx, "chfsi_reduce_generalized_panel: cuBLAS failed");
    return CHFSI_ERR_CUDA;
  }
  // exact Hermitian storage across the ranks' slabs (R13): gather the unsymmetrised H, average with H^H
  TRY(gather_slabs(ctx, n, nloc, Ap, lda, W));
  hermitize_panel_kernel<<<col_grid(n, nloc), 256, 0, ctx->stream>>>(n, nloc, row0, W, n, static_cast<double2*>(Ap),
                                                                     lda);
  CHFSI_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches++;
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return CHFSI_OK;
}

chfsi_status chfsi_back_transform_panel(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* L,
                                        int64_t ldl, void* X, int64_t ldx, int64_t k) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (!panel_args_ok(ctx, n, row0, nloc) || !L || ldl < n || k < 0 || k > n || (k > 0 && !X) || ldx < nloc) {
    set_err(ctx, "chfsi_back_transform_panel: bad arguments");
    return CHFSI_ERR_ARG;
  }
  if (k == 0) return CHFSI_OK;
  cudaSetDevice(ctx->device);
  chfsi_status st = ensure(ctx, ctx->gw, 16 * (size_t)n * k);
  if (!st) st = ensure(ctx, ctx->gx, 16 * (size_t)n * k);
  if (st) return st;
  double2* P = static_cast<double2*>(ctx->gx.ptr);  // packed [rank][nloc x k]
  double2* Y = static_cast<double2*>(ctx->gw.ptr);  // all n rows, ld n
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(P + nloc * k * ctx->rank, 16 * nloc, X, 16 * ldx, 16 * nloc, k,
                                        cudaMemcpyDeviceToDevice, ctx->stream));
  TRY(comm_allgather_inplace(ctx, reinterpret_cast<double*>(P), (size_t)2 * nloc * k));
  for (int q = 0; q < ctx->nranks; ++q)
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Y + nloc * q, 16 * n, P + nloc * k * q, 16 * nloc, 16 * nloc, k,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
  // c = L^{-H} y: every rank solves the whole block (n^2 k, like one filter step) and keeps its rows
  if (cublasZtrsm(ctx->cublas, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_C, CUBLAS_DIAG_NON_UNIT, (int)n,
                  (int)k, &kOne, static_cast<const cuDoubleComplex*>(L), (int)ldl,
                  reinterpret_cast<cuDoubleComplex*>(Y), (int)n) != CUBLAS_STATUS_SUCCESS) {
    set_err(ctx, "cublasZtrsm failed");
    return CHFSI_ERR_CUDA;
  }
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(X, 16 * ldx, Y + row0, 16 * n, 16 * nloc, k, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  return CHFSI_OK;
}

}  // extern "C"
