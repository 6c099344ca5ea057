// supporting.cu -- the supporting ChFSI steps on the device (Alg 1):
//   Lanczos spectral bounds (line 3), QR of the filtered block (line 6; P:581-584:
//   CGS2 against the locked block + CholeskyQR2, Householder fallback), Rayleigh-Ritz (lines 7-9;
//   P:584-589) with residuals (line 10; R8) computed from (HQ)W without a second n^2 k product.
// n^2 k contractions (H Q) run on the K1 kernel; n k^2 / k^3 pieces are plain library calls
// (cuBLAS ZGEMM/ZTRSM, cuSOLVER ZPOTRF/ZHEEVD/ZGEQRF/ZUNGQR); small reductions are the library's
// own kernels (small_kernels.cu). Every k x k reduction across ranks is an NCCL allreduce.
#include <algorithm>
#include <cmath>
#include <vector>

#include "ctx.cuh"
#include "small_kernels.cuh"
#include "supporting.cuh"

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

static const cuDoubleComplex kOne = {1.0, 0.0}, kZero = {0.0, 0.0}, kMinusOne = {-1.0, 0.0};

static inline cuDoubleComplex* zc(void* p) { return static_cast<cuDoubleComplex*>(p); }
static inline const cuDoubleComplex* zc(const void* p) { return static_cast<const cuDoubleComplex*>(p); }

// C (m x n, ldc) = A^H B with A (K x m), B (K x n) local rows, summed over ranks
static chfsi_status gram(chfsi_ctx ctx, int64_t K, int64_t m, int64_t n, const void* A, int64_t lda, const void* B,
                         int64_t ldb, void* C, int64_t ldc) {
  CUBLAS_TRY(ctx, cublasZgemm(ctx->cublas, CUBLAS_OP_C, CUBLAS_OP_N, (int)m, (int)n, (int)K, &kOne, zc(A), (int)lda,
                              zc(B), (int)ldb, &kZero, zc(C), (int)ldc));
  if (ctx->nranks > 1) {
    if (ldc != m) {
      set_err(ctx, "gram: allreduce needs packed C");
      return CHFSI_ERR_ARG;
    }
    TRY(comm_allreduce_sum(ctx, static_cast<double*>(C), (size_t)2 * m * n));
  }
  return CHFSI_OK;
}

// ---------------------------------------------------------------------------------------------
// Lanczos (R17): full reorthogonalisation (classical Gram-Schmidt, two passes) on this rank's rows.
static void tridiag_extremes(const std::vector<double>& al, const std::vector<double>& be, int m, double* tmin,
                             double* tmax) {
  // Sturm-sequence bisection for the smallest and the largest eigenvalue of T (m x m)
  double lo = al[0], hi = al[0];
  for (int i = 0; i < m; ++i) {
    const double rad = (i > 0 ? std::fabs(be[i - 1]) : 0.0) + (i + 1 < m ? std::fabs(be[i]) : 0.0);
    lo = std::min(lo, al[i] - rad);
    hi = std::max(hi, al[i] + rad);
  }
  auto count_below = [&](double x) {
    int cnt = 0;
    double d = 1.0;
    for (int i = 0; i < m; ++i) {
      d = (al[i] - x) - (i > 0 ? be[i - 1] * be[i - 1] / d : 0.0);
      if (d == 0.0) d = -1e-300;
      if (d < 0) ++cnt;
    }
    return cnt;
  };
  for (int which = 0; which < 2; ++which) {
    const int target = which == 0 ? 1 : m;
    double a = lo, b = hi;
    for (int it = 0; it < 200; ++it) {
      const double x = 0.5 * (a + b);
      if (x <= a || x >= b) break;
      if (count_below(x) >= target)
        b = x;
      else
        a = x;
    }
    (which == 0 ? *tmin : *tmax) = b;
  }
}

chfsi_status lanczos_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                          int32_t steps, uint64_t seed, double* theta_min, double* theta_max, double* upper) {
  if (steps > n) steps = (int32_t)n;
  const int p = ctx->nranks;
  const int64_t ldv = nloc;
  TRY(ensure(ctx, ctx->lz, sizeof(double) * 2 * ((size_t)ldv * (steps + 1) + (size_t)n + (size_t)nloc)));
  TRY(ensure(ctx, ctx->small3, sizeof(double) * 2 * (size_t)(steps + 8)));
  double2* V = static_cast<double2*>(ctx->lz.ptr);
  double2* vfull = V + (size_t)ldv * (steps + 1);
  double2* w = vfull + n;
  double2* coef = static_cast<double2*>(ctx->small3.ptr);
  double* nrm = reinterpret_cast<double*>(coef + steps + 2);
  std::vector<double> al(steps), be(steps);
  std::vector<double2> hcoef(steps + 2);
  for (int restart = 0; restart <= 3; ++restart) {
    CHFSI_CUDA_TRY(ctx, launch_random_block(nloc, 1, row0, seed, (4ull << 16) | (uint64_t)restart, 0, V, ldv,
                                            ctx->stream));
    ctx->launches++;
    double h = 0;
    CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, 1, V, ldv, nrm, ctx->stream));
    ctx->launches++;
    TRY(comm_allreduce_sum(ctx, nrm, 1));
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    CHFSI_CUDA_TRY(ctx, launch_scale(nloc, V, 1.0 / std::sqrt(h), ctx->stream));
    ctx->launches++;
    double hest = 0;
    bool broke = false;
    int j = 0;
    for (; j < steps; ++j) {
      double2* vj = V + (size_t)j * ldv;
      const double2* vin = vj;
      if (p > 1) {
        CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(vfull + (size_t)nloc * ctx->rank, vj, 16 * nloc, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
        TRY(comm_allgather_inplace(ctx, reinterpret_cast<double*>(vfull), (size_t)2 * nloc));
        vin = vfull;
      }
      CHFSI_CUDA_TRY(ctx, launch_hemv(n, nloc, static_cast<const double2*>(Hp), ldh, vin, w, ctx->stream));
      ctx->launches++;
      for (int pass = 0; pass < 2; ++pass) {
        CUBLAS_TRY(ctx, cublasZgemv(ctx->cublas, CUBLAS_OP_C, (int)nloc, j + 1, &kOne, zc(V), (int)ldv, zc(w), 1,
                                    &kZero, zc(coef), 1));
        TRY(comm_allreduce_sum(ctx, reinterpret_cast<double*>(coef), (size_t)2 * (j + 1)));
        if (pass == 0) {
          CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(hcoef.data(), coef, 16 * (j + 1), cudaMemcpyDeviceToHost, ctx->stream));
        }
        CUBLAS_TRY(ctx, cublasZgemv(ctx->cublas, CUBLAS_OP_N, (int)nloc, j + 1, &kMinusOne, zc(V), (int)ldv, zc(coef),
                                    1, &kOne, zc(w), 1));
      }
      CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, 1, w, nloc, nrm, ctx->stream));
      ctx->launches++;
      TRY(comm_allreduce_sum(ctx, nrm, 1));
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&h, nrm, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      al[j] = hcoef[j].x;  // alpha_j = Re(v_j^H H v_j)
      be[j] = std::sqrt(h);
      hest = std::max(hest, std::fabs(al[j]) + be[j] + (j > 0 ? be[j - 1] : 0.0));
      if (j + 1 < steps) {
        if (be[j] < 1e-14 * hest) {
          broke = true;
          break;
        }
        double2* vn = V + (size_t)(j + 1) * ldv;
        CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(vn, w, 16 * nloc, cudaMemcpyDeviceToDevice, ctx->stream));
        CHFSI_CUDA_TRY(ctx, launch_scale(nloc, vn, 1.0 / be[j], ctx->stream));
        ctx->launches++;
      }
    }
    if (broke) continue;
    tridiag_extremes(al, be, steps, theta_min, theta_max);
    *upper = *theta_max + be[steps - 1];
    return CHFSI_OK;
  }
  set_err(ctx, "chfsi_lanczos_bounds: breakdown after 3 restarts");
  return CHFSI_ERR_NOCONV;
}

// ---------------------------------------------------------------------------------------------
// Householder QR of Y (nloc x ka) with a positive real R diagonal; p > 1 gathers the block.
static chfsi_status householder(chfsi_ctx ctx, int64_t n, int64_t nloc, void* Y, int64_t ldy, int64_t ka) {
  const int p = ctx->nranks;
  void* A = Y;
  int64_t lda = ldy, m = nloc;
  if (p > 1) {
    TRY(ensure(ctx, ctx->R0, sizeof(double) * 2 * (size_t)n * ka));
    TRY(ensure(ctx, ctx->w4, sizeof(double) * 2 * (size_t)n * ka));
    double* R = static_cast<double*>(ctx->R0.ptr);
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(R + (size_t)2 * nloc * ka * ctx->rank, 16 * nloc, Y, 16 * ldy, 16 * nloc, ka,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
    TRY(comm_allgather_inplace(ctx, R, (size_t)2 * nloc * ka));
    double* F = static_cast<double*>(ctx->w4.ptr);
    for (int q = 0; q < p; ++q)
      CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(F + (size_t)2 * nloc * q, 16 * n, R + (size_t)2 * nloc * ka * q, 16 * nloc,
                                            16 * nloc, ka, cudaMemcpyDeviceToDevice, ctx->stream));
    A = F;
    lda = n;
    m = n;
  }
  TRY(ensure(ctx, ctx->small2, sizeof(double) * 2 * (size_t)ka * (ka + 1)));
  TRY(ensure(ctx, ctx->devinfo, 64));
  cuDoubleComplex* tau = zc(ctx->small2.ptr);
  cuDoubleComplex* Rd = tau + ka;  // copy of R (ka x ka)
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  int lw1 = 0, lw2 = 0;
  CUSOLVER_TRY(ctx, cusolverDnZgeqrf_bufferSize(ctx->cusolver, (int)m, (int)ka, zc(A), (int)lda, &lw1));
  CUSOLVER_TRY(ctx, cusolverDnZungqr_bufferSize(ctx->cusolver, (int)m, (int)ka, (int)ka, zc(A), (int)lda, tau, &lw2));
  const int lw = std::max(lw1, lw2);
  TRY(ensure(ctx, ctx->solver_ws, sizeof(cuDoubleComplex) * (size_t)std::max(lw, 1)));
  CUSOLVER_TRY(ctx, cusolverDnZgeqrf(ctx->cusolver, (int)m, (int)ka, zc(A), (int)lda, tau, zc(ctx->solver_ws.ptr), lw,
                                     info));
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Rd, 16 * ka, A, 16 * lda, 16 * ka, ka, cudaMemcpyDeviceToDevice, ctx->stream));
  CUSOLVER_TRY(ctx, cusolverDnZungqr(ctx->cusolver, (int)m, (int)ka, (int)ka, zc(A), (int)lda, tau,
                                     zc(ctx->solver_ws.ptr), lw, info));
  CHFSI_CUDA_TRY(ctx, launch_col_phase(m, ka, static_cast<double2*>(A), lda, reinterpret_cast<double2*>(Rd), ka,
                                       ctx->stream));
  ctx->launches++;
  if (p > 1) {
    const double* F = static_cast<const double*>(A);
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Y, 16 * ldy, F + (size_t)2 * nloc * ctx->rank, 16 * n, 16 * nloc, ka,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
  }
  int hinfo = 0;
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) {
    set_err(ctx, "Householder fallback failed (info " + std::to_string(hinfo) + ")");
    return CHFSI_ERR_QR;
  }
  return CHFSI_OK;
}

chfsi_status qr_impl(chfsi_ctx ctx, int64_t n, int64_t nloc, const void* XL, int64_t ldxl, int64_t nl, void* Y,
                     int64_t ldy, int64_t ka, int32_t* used_fallback) {
  if (used_fallback) *used_fallback = 0;
  if (ka == 0) return CHFSI_OK;
  TRY(ensure(ctx, ctx->small1, sizeof(double) * 2 * (size_t)std::max<int64_t>(ka, nl) * ka + 64));
  TRY(ensure(ctx, ctx->devinfo, 64));
  cuDoubleComplex* S = zc(ctx->small1.ptr);
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  // CGS2 against the locked block (R15: the locked columns are not modified)
  if (nl > 0) {
    for (int pass = 0; pass < 2; ++pass) {
      TRY(gram(ctx, nloc, nl, ka, XL, ldxl, Y, ldy, S, nl));
      CUBLAS_TRY(ctx, cublasZgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)nloc, (int)ka, (int)nl, &kMinusOne,
                                  zc(XL), (int)ldxl, S, (int)nl, &kOne, zc(Y), (int)ldy));
    }
  }
  // CholeskyQR2: S = Y^H Y = R^H R, Y <- Y R^{-1}, twice
  bool ok = true;
  int lw = 0;
  CUSOLVER_TRY(ctx, cusolverDnZpotrf_bufferSize(ctx->cusolver, CUBLAS_FILL_MODE_UPPER, (int)ka, S, (int)ka, &lw));
  TRY(ensure(ctx, ctx->solver_ws, sizeof(cuDoubleComplex) * (size_t)std::max(lw, 1)));
  for (int pass = 0; pass < 2 && ok; ++pass) {
    TRY(gram(ctx, nloc, ka, ka, Y, ldy, Y, ldy, S, ka));
    CUSOLVER_TRY(ctx, cusolverDnZpotrf(ctx->cusolver, CUBLAS_FILL_MODE_UPPER, (int)ka, S, (int)ka,
                                       zc(ctx->solver_ws.ptr), lw, info));
    int hinfo = 0;
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    if (hinfo != 0) {
      ok = false;
      break;
    }
    CUBLAS_TRY(ctx, cublasZtrsm(ctx->cublas, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                                CUBLAS_DIAG_NON_UNIT, (int)nloc, (int)ka, &kOne, S, (int)ka, zc(Y), (int)ldy));
  }
  if (ok) {  // orthogonality check ||Q^H Q - I||_max <= 1e-12
    TRY(gram(ctx, nloc, ka, ka, Y, ldy, Y, ldy, S, ka));
    double* e = reinterpret_cast<double*>(info + 4);
    CHFSI_CUDA_TRY(ctx, launch_orth_err(ka, reinterpret_cast<double2*>(S), ka, e, ctx->stream));
    ctx->launches++;
    double he = 0;
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&he, e, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    ok = he <= 1e-12;
  }
  if (!ok) {
    if (used_fallback) *used_fallback = 1;
    TRY(householder(ctx, n, nloc, Y, ldy, ka));
  }
  return CHFSI_OK;
}

// ---------------------------------------------------------------------------------------------
// Rayleigh-Ritz with residuals. Q (nloc x ka) in/out. mu (host, ascending), resid (host, nullable).
chfsi_status rr_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh, void* Q,
                     int64_t ldq, int64_t ka, double normH, double* mu, double* resid) {
  if (ka == 0) return CHFSI_OK;
  const size_t blk = sizeof(double) * 2 * (size_t)nloc * ka;
  TRY(ensure(ctx, ctx->w1, blk));
  TRY(ensure(ctx, ctx->w2, blk));
  TRY(ensure(ctx, ctx->w3, blk));
  TRY(ensure(ctx, ctx->small1, sizeof(double) * 2 * (size_t)ka * ka + 64));
  TRY(ensure(ctx, ctx->small2, sizeof(double) * (size_t)(4 * ka + 64)));
  TRY(ensure(ctx, ctx->devinfo, 64));
  cuDoubleComplex* W = zc(ctx->w1.ptr);  // H Q
  cuDoubleComplex* Yr = zc(ctx->w2.ptr);  // Q V
  cuDoubleComplex* HY = zc(ctx->w3.ptr);  // (H Q) V
  cuDoubleComplex* G = zc(ctx->small1.ptr);
  double* dmu = static_cast<double*>(ctx->small2.ptr);
  double* dr = dmu + ka;
  double* dn = dr + ka;
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  TRY(hmul_impl(ctx, n, row0, nloc, Hp, ldh, Q, ldq, ka, W, nloc));
  TRY(gram(ctx, nloc, ka, ka, Q, ldq, W, nloc, G, ka));
  CHFSI_CUDA_TRY(ctx, launch_hermitize(ka, reinterpret_cast<double2*>(G), ka, ctx->stream));
  ctx->launches++;
  // small dense eigensolve: once, on rank 0, broadcast (identical bits on every rank)
  if (ctx->rank == 0) {
    int lw = 0;
    CUSOLVER_TRY(ctx, cusolverDnZheevd_bufferSize(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER,
                                                  (int)ka, G, (int)ka, dmu, &lw));
    TRY(ensure(ctx, ctx->solver_ws, sizeof(cuDoubleComplex) * (size_t)std::max(lw, 1)));
    CUSOLVER_TRY(ctx, cusolverDnZheevd(ctx->cusolver, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_UPPER, (int)ka, G,
                                       (int)ka, dmu, zc(ctx->solver_ws.ptr), lw, info));
  }
  TRY(comm_bcast(ctx, reinterpret_cast<double*>(G), (size_t)2 * ka * ka, 0));
  TRY(comm_bcast(ctx, dmu, (size_t)ka, 0));
  CUBLAS_TRY(ctx, cublasZgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)nloc, (int)ka, (int)ka, &kOne, zc(Q),
                              (int)ldq, G, (int)ka, &kZero, Yr, (int)nloc));
  if (resid) {
    CUBLAS_TRY(ctx, cublasZgemm(ctx->cublas, CUBLAS_OP_N, CUBLAS_OP_N, (int)nloc, (int)ka, (int)ka, &kOne, W,
                                (int)nloc, G, (int)ka, &kZero, HY, (int)nloc));
    CHFSI_CUDA_TRY(ctx, launch_resid2(nloc, ka, reinterpret_cast<double2*>(HY), nloc, reinterpret_cast<double2*>(Yr),
                                      nloc, dmu, dr, ctx->stream));
    CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, ka, reinterpret_cast<double2*>(Yr), nloc, dn, ctx->stream));
    ctx->launches += 2;
    TRY(comm_allreduce_sum(ctx, dr, (size_t)2 * ka));  // dr and dn are contiguous
  }
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Q, 16 * ldq, Yr, 16 * nloc, 16 * nloc, ka, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
  std::vector<double> h(3 * ka);
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), dmu, sizeof(double) * (resid ? 3 * ka : ka), cudaMemcpyDeviceToHost,
                                      ctx->stream));
  int hinfo = 0;
  if (ctx->rank == 0)
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) {
    set_err(ctx, "zheevd failed (info " + std::to_string(hinfo) + ")");
    return CHFSI_ERR_CUDA;
  }
  for (int64_t j = 0; j < ka; ++j) {
    mu[j] = h[j];
    if (resid) resid[j] = std::sqrt(h[ka + j]) / (std::sqrt(h[2 * ka + j]) * normH);
  }
  return CHFSI_OK;
}

}  // namespace chfsi

using namespace chfsi;

extern "C" {

chfsi_status chfsi_lanczos_bounds(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                                  int32_t steps, uint64_t seed, double* theta_min, double* theta_max,
                                  double* upper_bound) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || nloc < 1 || row0 < 0 || row0 + nloc > n || ldh < n || !Hp || steps < 1 || !theta_min || !theta_max ||
      !upper_bound || (ctx->nranks > 1 && (nloc * ctx->nranks != n || row0 != nloc * ctx->rank))) {
    set_err(ctx, "chfsi_lanczos_bounds: bad arguments");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  return lanczos_impl(ctx, n, row0, nloc, Hp, ldh, steps, seed, theta_min, theta_max, upper_bound);
}

chfsi_status chfsi_qr(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, void* Y, int64_t ldy, int64_t k,
                      int64_t nlocked, int32_t* used_fallback) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || nloc < 1 || row0 < 0 || row0 + nloc > n || ldy < nloc || k < 0 || k > n || nlocked < 0 ||
      nlocked > k || (k > 0 && !Y) || (ctx->nranks > 1 && (nloc * ctx->nranks != n || row0 != nloc * ctx->rank))) {
    set_err(ctx, "chfsi_qr: bad arguments");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  double2* y = static_cast<double2*>(Y);
  return qr_impl(ctx, n, nloc, y, ldy, nlocked, y + (size_t)ldy * nlocked, ldy, k - nlocked, used_fallback);
}

chfsi_status chfsi_rayleigh_ritz(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                                 void* Q, int64_t ldq, int64_t k, double normH, double* ritz, double* resid) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || nloc < 1 || row0 < 0 || row0 + nloc > n || ldh < n || ldq < nloc || k < 0 || k > n ||
      (k > 0 && (!Hp || !Q || !ritz)) || (resid && !(normH > 0)) ||
      (ctx->nranks > 1 && (nloc * ctx->nranks != n || row0 != nloc * ctx->rank))) {
    set_err(ctx, "chfsi_rayleigh_ritz: bad arguments");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  return rr_impl(ctx, n, row0, nloc, Hp, ldh, Q, ldq, k, normH, ritz, resid);
}

}  // extern "C"
