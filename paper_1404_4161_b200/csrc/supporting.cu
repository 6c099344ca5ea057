// supporting.cu -- the supporting ChFSI steps on the device (Alg 1):
//   Lanczos spectral bounds (line 3), QR of the filtered block (line 6; P:581-584:
//   CGS2 against the locked block + CholeskyQR2, Householder fallback), Rayleigh-Ritz (lines 7-9;
//   P:584-589) with residuals (line 10; R8) computed from (HQ)W without a second n^2 k product.
// n^2 k contractions (H Q) run on the K1 kernel; n k^2 / k^3 pieces are plain library calls
// (cuBLAS ZGEMM/ZTRSM, cuSOLVER ZPOTRF/ZHEEVD/ZGEQRF/ZUNGQR); small reductions are the library's
// own kernels (small_kernels.cu). Every k x k reduction across ranks is an NCCL allreduce.
#include <cstdio>
#include <algorithm>
#include <cmath>
#include <vector>

#include "blas_traits.cuh"
#include "ctx.cuh"
#include "small_kernels.cuh"
#include "supporting.cuh"

namespace chfsi {

// C (m x n, ldc) = A^H B with A (K x m), B (K x n) local rows, summed over ranks
template <typename T>
static chfsi_status gram(chfsi_ctx ctx, int64_t K, int64_t m, int64_t n, const void* A, int64_t lda, const void* B,
                         int64_t ldb, void* C, int64_t ldc) {
  using S = Sc<T>;
  const T one = S::one(), zero = S::zero();
  CUBLAS_TRY(ctx, S::gemm(ctx, S::opH, CUBLAS_OP_N, (int)m, (int)n, (int)K, &one, static_cast<const T*>(A),
                          (int)lda, static_cast<const T*>(B), (int)ldb, &zero, static_cast<T*>(C), (int)ldc));
  if (ctx->nranks > 1) {
    if (ldc != m) {
      set_err(ctx, "gram: allreduce needs packed C");
      return CHFSI_ERR_ARG;
    }
    TRY(comm_allreduce_sum(ctx, static_cast<double*>(C), (size_t)S::elem * m * n));
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

template <typename T>
chfsi_status lanczos_t(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh, int32_t steps,
                       uint64_t seed, double* theta_min, double* theta_max, double* upper) {
  using S = Sc<T>;
  using D = typename S::D;
  const T one = S::one(), zero = S::zero(), mone = S::mone();
  if (steps > n) steps = (int32_t)n;
  const int p = ctx->nranks;
  const int64_t ldv = nloc;
  TRY(ensure(ctx, ctx->lz, sizeof(D) * ((size_t)ldv * (steps + 1) + (size_t)n + (size_t)nloc) + 64));
  TRY(ensure(ctx, ctx->small3, sizeof(double) * (2 * (size_t)(steps + 8) + 2 * (size_t)steps + 8)));
  D* V = static_cast<D*>(ctx->lz.ptr);
  D* vfull = V + (size_t)ldv * (steps + 1);
  D* w = vfull + n;
  const void** hslot = reinterpret_cast<const void**>(w + nloc);  // the panel pointer of the graph path
  D* coef = static_cast<D*>(ctx->small3.ptr);
  double* nrm = static_cast<double*>(ctx->small3.ptr) + 2 * (steps + 2);
  double* dalpha = nrm + 8;             // alpha_j, beta_j of every step stay on the device until the end
  double* dbeta = dalpha + steps;
  std::vector<double> al(steps), be(steps);
  // the steps run without host round trips: beta_j = ||w||, v_{j+1} = w / beta_j and alpha_j are formed
  // on the device; the breakdown test (beta_j < 1e-14 ||T||_est) runs on the host afterwards, and a
  // breakdown discards the (then meaningless) later steps and restarts
  auto issue_steps = [&](const void* const* hpp) -> chfsi_status {
    for (int j = 0; j < steps; ++j) {
      D* vj = V + (size_t)j * ldv;
      const D* vin = vj;
      if (p > 1) {
        CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(vfull + (size_t)nloc * ctx->rank, vj, sizeof(D) * nloc,
                                            cudaMemcpyDeviceToDevice, ctx->stream));
        TRY(comm_allgather_inplace(ctx, reinterpret_cast<double*>(vfull), (size_t)S::elem * nloc));
        vin = vfull;
      }
      CHFSI_CUDA_TRY(ctx, launch_hemv(n, nloc, static_cast<const D*>(Hp), ldh, vin, w, ctx->stream, hpp));
      ctx->launches++;
      for (int pass = 0; pass < 2; ++pass) {
        CUBLAS_TRY(ctx, S::gemv(ctx->cublas, S::opH, (int)nloc, j + 1, &one, reinterpret_cast<const T*>(V), (int)ldv,
                                reinterpret_cast<const T*>(w), &zero, reinterpret_cast<T*>(coef)));
        TRY(comm_allreduce_sum(ctx, reinterpret_cast<double*>(coef), (size_t)S::elem * (j + 1)));
        if (pass == 0)  // alpha_j = Re(v_j^H H v_j) from the first pass
          CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(dalpha + j, coef + j, sizeof(double), cudaMemcpyDeviceToDevice,
                                              ctx->stream));
        CUBLAS_TRY(ctx, S::gemv(ctx->cublas, CUBLAS_OP_N, (int)nloc, j + 1, &mone, reinterpret_cast<const T*>(V),
                                (int)ldv, reinterpret_cast<const T*>(coef), &one, reinterpret_cast<T*>(w)));
      }
      CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, 1, w, nloc, nrm, ctx->stream));
      ctx->launches++;
      TRY(comm_allreduce_sum(ctx, nrm, 1));
      D* vn = j + 1 < steps ? V + (size_t)(j + 1) * ldv : nullptr;
      CHFSI_CUDA_TRY(ctx, launch_lanczos_next(nloc, w, vn, nrm, nullptr, dbeta + j, nullptr, ctx->stream));
      ctx->launches++;
    }
    return CHFSI_OK;
  };
  // One rank: the 25 steps (~7 small launches each) are launch-bound at small n, so they run as a CUDA
  // graph captured once per shape / workspace and replayed for every problem, the panel read through
  // hslot. Several ranks keep direct launches (their collectives order against the other ranks).
  static const bool graphs_env = !(getenv("CHFSI_GRAPHS") && getenv("CHFSI_GRAPHS")[0] == '0');
  bool use_graph = p == 1 && graphs_env && !ctx->lz_graph_off;
  if (use_graph) {
    const std::vector<int64_t> key = {n, nloc, ldh, steps, (int64_t)S::elem, (int64_t)(intptr_t)V,
                                      (int64_t)(intptr_t)coef, (int64_t)(intptr_t)ctx->cublas};
    if (!ctx->lz_exec || ctx->lz_key != key) {
      if (ctx->lz_exec) {
        cudaGraphExecDestroy(ctx->lz_exec);
        ctx->lz_exec = nullptr;
      }
      cudaGraph_t graph = nullptr;
      const int64_t launches0 = ctx->launches;
      // capture on a library-owned stream (the context's may be the legacy default stream, which cannot
      // be captured): the steps are recorded, not run, so no ordering with the context stream is needed
      bool ok = ctx->cap_stream || cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking) == cudaSuccess;
      cudaStream_t home = ctx->stream;
      if (ok) {
        ctx->stream = ctx->cap_stream;
        ok = cublasSetStream(ctx->cublas, ctx->cap_stream) == CUBLAS_STATUS_SUCCESS &&
             cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
          const chfsi_status st = issue_steps(reinterpret_cast<const void* const*>(hslot));
          ok = cudaStreamEndCapture(ctx->cap_stream, &graph) == cudaSuccess && st == CHFSI_OK;
        }
        ctx->stream = home;
        cublasSetStream(ctx->cublas, home);
      }
      if (ok) ok = cudaGraphInstantiate(&ctx->lz_exec, graph, 0) == cudaSuccess;
      if (graph) cudaGraphDestroy(graph);
      if (!ok) {  // e.g. a library call that cannot be captured: launch directly from now on
        const cudaError_t ce = cudaGetLastError();
        if (getenv("CHFSI_GRAPHS_DEBUG"))
          fprintf(stderr, "chfsi: Lanczos graph capture failed (%s; %s); direct launches\n", cudaGetErrorString(ce),
                  ctx->err.c_str());
        if (ctx->lz_exec) cudaGraphExecDestroy(ctx->lz_exec);
        ctx->lz_exec = nullptr;
        ctx->lz_graph_off = true;
        use_graph = false;
        ctx->err.clear();
      } else {
        ctx->lz_key = key;
        if (getenv("CHFSI_GRAPHS_DEBUG")) fprintf(stderr, "chfsi: Lanczos steps captured (n %lld, %d steps)\n", (long long)n, steps);
      }
      ctx->launches = launches0;  // captured, not launched
    }
  }
  for (int restart = 0; restart <= 3; ++restart) {
    CHFSI_CUDA_TRY(ctx, launch_random_block(nloc, 1, row0, seed, (4ull << 16) | (uint64_t)restart, 0, V, ldv,
                                            ctx->stream));
    ctx->launches++;
    CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, 1, V, ldv, nrm, ctx->stream));
    ctx->launches++;
    TRY(comm_allreduce_sum(ctx, nrm, 1));
    CHFSI_CUDA_TRY(ctx, launch_scale_rnorm(nloc, V, nrm, ctx->stream));  // v_0 / ||v_0||, on the device
    ctx->launches++;
    if (use_graph) {
      CHFSI_CUDA_TRY(ctx, launch_store_ptr(hslot, Hp, ctx->stream));
      CHFSI_CUDA_TRY(ctx, cudaGraphLaunch(ctx->lz_exec, ctx->stream));
      ctx->launches += 1 + 3 * (int64_t)steps;  // store + the graph's own kernels (hemv, colnorm, next per step)
    } else {
      TRY(issue_steps(nullptr));
    }
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(al.data(), dalpha, sizeof(double) * steps, cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(be.data(), dbeta, sizeof(double) * steps, cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    double hest = 0;
    bool broke = false;
    for (int j = 0; j < steps; ++j) {
      hest = std::max(hest, std::fabs(al[j]) + be[j] + (j > 0 ? be[j - 1] : 0.0));
      if (j + 1 < steps && be[j] < 1e-14 * hest) {
        broke = true;
        break;
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
// Householder QR of Y (nloc x ka) with a positive real R diagonal; p > 1 gathers the block (every rank
// factors the same gathered block, so every rank gets the same R). rdiag (host, nullable) <- |R_jj|.
template <typename T>
static chfsi_status householder(chfsi_ctx ctx, int64_t n, int64_t nloc, void* Y, int64_t ldy, int64_t ka,
                                std::vector<double>* rdiag) {
  using S = Sc<T>;
  using D = typename S::D;
  const size_t eb = sizeof(T);
  const int p = ctx->nranks;
  void* A = Y;
  int64_t lda = ldy, m = nloc;
  if (p > 1) {
    TRY(ensure(ctx, ctx->R0, eb * (size_t)n * ka));
    TRY(ensure(ctx, ctx->w4, eb * (size_t)n * ka));
    double* R = static_cast<double*>(ctx->R0.ptr);
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(R + (size_t)S::elem * nloc * ka * ctx->rank, eb * nloc, Y, eb * ldy,
                                          eb * nloc, ka, cudaMemcpyDeviceToDevice, ctx->stream));
    TRY(comm_allgather_inplace(ctx, R, (size_t)S::elem * nloc * ka));
    double* F = static_cast<double*>(ctx->w4.ptr);
    for (int q = 0; q < p; ++q)
      CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(F + (size_t)S::elem * nloc * q, eb * n, R + (size_t)S::elem * nloc * ka * q,
                                            eb * nloc, eb * nloc, ka, cudaMemcpyDeviceToDevice, ctx->stream));
    A = F;
    lda = n;
    m = n;
  }
  TRY(ensure(ctx, ctx->small2, eb * (size_t)ka * (ka + 1)));
  TRY(ensure(ctx, ctx->devinfo, 64));
  T* tau = static_cast<T*>(ctx->small2.ptr);
  T* Rd = tau + ka;  // copy of R (ka x ka)
  T* At = static_cast<T*>(A);
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  int lw1 = 0, lw2 = 0;
  CUSOLVER_TRY(ctx, S::geqrf_bs(ctx->cusolver, (int)m, (int)ka, At, (int)lda, &lw1));
  CUSOLVER_TRY(ctx, S::orgqr_bs(ctx->cusolver, (int)m, (int)ka, At, (int)lda, tau, &lw2));
  const int lw = std::max(lw1, lw2);
  TRY(ensure(ctx, ctx->solver_ws, eb * (size_t)std::max(lw, 1)));
  CUSOLVER_TRY(ctx, S::geqrf(ctx->cusolver, (int)m, (int)ka, At, (int)lda, tau, static_cast<T*>(ctx->solver_ws.ptr), lw,
                             info));
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Rd, eb * ka, A, eb * lda, eb * ka, ka, cudaMemcpyDeviceToDevice, ctx->stream));
  std::vector<T> hdiag(rdiag ? ka : 0);
  if (rdiag)  // the diagonal of R: stride ka + 1 elements
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(hdiag.data(), eb, Rd, eb * (ka + 1), eb, ka, cudaMemcpyDeviceToHost,
                                          ctx->stream));
  CUSOLVER_TRY(ctx, S::orgqr(ctx->cusolver, (int)m, (int)ka, At, (int)lda, tau, static_cast<T*>(ctx->solver_ws.ptr), lw,
                             info));
  CHFSI_CUDA_TRY(ctx, launch_col_phase(m, ka, static_cast<D*>(A), lda, reinterpret_cast<D*>(Rd), ka, ctx->stream));
  ctx->launches++;
  if (p > 1) {
    const double* F = static_cast<const double*>(A);
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Y, eb * ldy, F + (size_t)S::elem * nloc * ctx->rank, eb * n, eb * nloc, ka,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
  }
  int hinfo = 0;
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (hinfo != 0) {
    set_err(ctx, "Householder fallback failed (info " + std::to_string(hinfo) + ")");
    return CHFSI_ERR_QR;
  }
  if (rdiag) {
    rdiag->resize(ka);
    for (int64_t j = 0; j < ka; ++j) {
      if constexpr (S::elem == 2)
        (*rdiag)[j] = std::hypot(hdiag[j].x, hdiag[j].y);
      else
        (*rdiag)[j] = std::fabs(hdiag[j]);
    }
  }
  return CHFSI_OK;
}

// Alg 1 l6 with the rank-deficiency rule R23, mirroring ora_orthonormalize:
//   nu_j = ||y_j|| (input); repeat { Y <- CGS2(Y vs X_L); QR(Y); D = {j : |R_jj| <= 1e-12 nu_j};
//   if D is empty stop; y_j <- R22 vector (seed + round, stream (6 << 16) | (nl + j)) for j in D }.
// The QR is CholeskyQR2 (R14) unless a projected column is already below 1e-12 nu_j (it then lies in
// span(X_L) and CholeskyQR's R_jj could not resolve it); a failed Cholesky pivot or ||Q^H Q - I||_max
// > 1e-12 falls back to Householder, whose |R_jj| decide D (CholeskyQR2 only ever succeeds on blocks
// with condition numbers far below 1e12, which have no such column).
template <typename T>
chfsi_status qr_t(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* XL, int64_t ldxl, int64_t nl,
                  void* Y, int64_t ldy, int64_t ka, uint64_t seed, int32_t* used_fallback, int32_t* replaced) {
  using S = Sc<T>;
  using D = typename S::D;
  const T one = S::one(), mone = S::mone();
  if (used_fallback) *used_fallback = 0;
  if (replaced) *replaced = 0;
  if (ka == 0) return CHFSI_OK;
  TRY(ensure(ctx, ctx->small1, sizeof(T) * (size_t)std::max<int64_t>(ka, nl) * ka + 64));
  TRY(ensure(ctx, ctx->devinfo, 64));
  TRY(ensure(ctx, ctx->qrn, sizeof(double) * (size_t)(ka + 8)));
  T* G = static_cast<T*>(ctx->small1.ptr);
  T* Yt = static_cast<T*>(Y);
  D* Yd = static_cast<D*>(Y);
  const T* Xt = static_cast<const T*>(XL);
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  double* dnrm = static_cast<double*>(ctx->qrn.ptr);
  const size_t eb = sizeof(T);
  // R23: input column norms nu_j^2 (before the projection against the locked block)
  std::vector<double> nu2(ka), mu2(ka);
  CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, ka, Yd, ldy, dnrm, ctx->stream));
  ctx->launches++;
  TRY(comm_allreduce_sum(ctx, dnrm, (size_t)ka));
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(nu2.data(), dnrm, sizeof(double) * ka, cudaMemcpyDeviceToHost, ctx->stream));
  int lw = 0;
  CUSOLVER_TRY(ctx, S::potrf_bs(ctx->cusolver, (int)ka, G, (int)ka, &lw));
  TRY(ensure(ctx, ctx->solver_ws, sizeof(T) * (size_t)std::max(lw, 1)));
  for (int round = 0;; ++round) {
    // CGS2 against the locked block (R15: the locked columns are not modified)
    if (nl > 0) {
      for (int pass = 0; pass < 2; ++pass) {
        TRY(gram<T>(ctx, nloc, nl, ka, XL, ldxl, Y, ldy, G, nl));
        CUBLAS_TRY(ctx, S::gemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, (int)nloc, (int)ka, (int)nl, &mone, Xt, (int)ldxl, G,
                                (int)nl, &one, Yt, (int)ldy));
      }
    }
    bool ok = true;
    if (nl > 0) {  // a column numerically inside span(X_L) goes straight to the Householder detection
      CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, ka, Yd, ldy, dnrm, ctx->stream));
      ctx->launches++;
      TRY(comm_allreduce_sum(ctx, dnrm, (size_t)ka));
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(mu2.data(), dnrm, sizeof(double) * ka, cudaMemcpyDeviceToHost, ctx->stream));
      CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      for (int64_t j = 0; j < ka; ++j)
        if (std::sqrt(mu2[j]) <= 1e-12 * std::sqrt(nu2[j])) ok = false;
    }
    // the projected block, kept for a Householder / replacement restart (CholeskyQR2 overwrites Y)
    TRY(ensure(ctx, ctx->qsave, eb * (size_t)nloc * ka));
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(ctx->qsave.ptr, eb * nloc, Y, eb * ldy, eb * nloc, ka,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
    // CholeskyQR2: S = Y^H Y = R^H R, Y <- Y R^{-1}, twice. diag(R) = diag(R_2) diag(R_1) estimates the
    // Householder |R_jj| to about eps ||y_j|| (a dependent column gets R_1jj ~ sqrt(eps) ||y_j|| from the
    // rounding of the Gram matrix and R_2jj ~ sqrt(eps) from the noise it leaves), so a column with
    // diag(R)_jj <= 1e-10 nu_j -- 100x above R23's 1e-12 -- is sent to the Householder decision
    std::vector<T> rd[2];
    for (int pass = 0; pass < 2 && ok; ++pass) {
      TRY(gram<T>(ctx, nloc, ka, ka, Y, ldy, Y, ldy, G, ka));
      CUSOLVER_TRY(ctx, S::potrf(ctx->cusolver, (int)ka, G, (int)ka, static_cast<T*>(ctx->solver_ws.ptr), lw, info));
      rd[pass].resize(ka);
      CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(rd[pass].data(), eb, G, eb * (ka + 1), eb, ka, cudaMemcpyDeviceToHost,
                                            ctx->stream));
      int hinfo = 0;
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
      CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      if (hinfo != 0) {
        ok = false;
        break;
      }
      CUBLAS_TRY(ctx, S::trsm_ru(ctx->cublas, (int)nloc, (int)ka, G, (int)ka, Yt, (int)ldy));
    }
    for (int64_t j = 0; j < ka && ok; ++j)
      if (std::fabs(S::re(rd[0][j])) * std::fabs(S::re(rd[1][j])) <= 1e-10 * std::sqrt(nu2[j])) ok = false;
    if (ok) {  // orthogonality check ||Q^H Q - I||_max <= 1e-12
      TRY(gram<T>(ctx, nloc, ka, ka, Y, ldy, Y, ldy, G, ka));
      double* e = reinterpret_cast<double*>(info + 4);
      CHFSI_CUDA_TRY(ctx, launch_orth_err(ka, reinterpret_cast<const D*>(G), ka, e, ctx->stream));
      ctx->launches++;
      double he = 0;
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&he, e, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      ok = he <= 1e-12;
    }
    if (ok) return CHFSI_OK;
    // Householder QR of the projected block; its |R_jj| decide the dependent columns, and a replacement
    // round restarts from the same projected block as the oracle
    if (used_fallback) *used_fallback = 1;
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Y, eb * ldy, ctx->qsave.ptr, eb * nloc, eb * nloc, ka,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
    std::vector<double> rdiag;
    TRY(householder<T>(ctx, n, nloc, Y, ldy, ka, &rdiag));
    std::vector<int64_t> defic;
    for (int64_t j = 0; j < ka; ++j)
      if (rdiag[j] <= 1e-12 * std::sqrt(nu2[j])) defic.push_back(j);
    if (defic.empty()) return CHFSI_OK;
    if (round == 3) {
      set_err(ctx, "QR: " + std::to_string(defic.size()) + " column(s) still rank deficient after 3 replacement rounds");
      return CHFSI_ERR_QR;
    }
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Y, eb * ldy, ctx->qsave.ptr, eb * nloc, eb * nloc, ka,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
    for (size_t i = 0; i < defic.size(); ++i) {
      D* col = Yd + (size_t)defic[i] * ldy;
      CHFSI_CUDA_TRY(ctx, launch_random_block(nloc, 1, row0, seed + (uint64_t)round, (6ull << 16) | (uint64_t)(nl + defic[i]),
                                              0, col, ldy, ctx->stream));
      CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, 1, col, ldy, dnrm + (i % 8), ctx->stream));
      ctx->launches += 2;
      if (i % 8 == 7 || i + 1 == defic.size()) {  // the replaced columns' nu_j^2, 8 at a time
        const size_t cnt = i % 8 + 1;
        double h8[8];
        TRY(comm_allreduce_sum(ctx, dnrm, cnt));
        CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(h8, dnrm, sizeof(double) * cnt, cudaMemcpyDeviceToHost, ctx->stream));
        CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
        for (size_t q = 0; q < cnt; ++q) nu2[defic[i + 1 - cnt + q]] = h8[q];
      }
    }
    if (replaced) *replaced += (int32_t)defic.size();
  }
}

// ---------------------------------------------------------------------------------------------
// Rayleigh-Ritz with residuals. Q (nloc x ka) in/out. mu (host, ascending), resid (host, nullable).
template <typename T>
chfsi_status rr_t(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh, void* Q,
                  int64_t ldq, int64_t ka, double normH, double* mu, double* resid) {
  using S = Sc<T>;
  using D = typename S::D;
  const T one = S::one(), zero = S::zero();
  const size_t eb = sizeof(T);
  if (ka == 0) return CHFSI_OK;
  const size_t blk = eb * (size_t)nloc * ka;
  TRY(ensure(ctx, ctx->w1, blk));
  TRY(ensure(ctx, ctx->w2, blk));
  TRY(ensure(ctx, ctx->w3, blk));
  TRY(ensure(ctx, ctx->small1, eb * (size_t)ka * ka + 64));
  TRY(ensure(ctx, ctx->small2, sizeof(double) * (size_t)(4 * ka + 64)));
  TRY(ensure(ctx, ctx->devinfo, 64));
  T* W = static_cast<T*>(ctx->w1.ptr);   // H Q
  T* Yr = static_cast<T*>(ctx->w2.ptr);  // Q V
  T* HY = static_cast<T*>(ctx->w3.ptr);  // (H Q) V
  T* G = static_cast<T*>(ctx->small1.ptr);
  const T* Qt = static_cast<const T*>(Q);
  double* dmu = static_cast<double*>(ctx->small2.ptr);
  double* dr = dmu + ka;
  double* dn = dr + ka;
  int* info = static_cast<int*>(ctx->devinfo.ptr);
  TRY(hmul_impl(ctx, n, row0, nloc, Hp, ldh, Q, ldq, ka, W, nloc, S::elem));
  TRY(gram<T>(ctx, nloc, ka, ka, Q, ldq, W, nloc, G, ka));
  CHFSI_CUDA_TRY(ctx, launch_hermitize(ka, reinterpret_cast<D*>(G), ka, ctx->stream));
  ctx->launches++;
  // diagnostics (CHFSI_RR_LOG): how far the projected matrix is from diagonal (relative Frobenius mass of
  // the off-diagonal part), the quantity a Jacobi-type eigensolver would have to remove
  static const bool rr_log = getenv("CHFSI_RR_LOG") != nullptr;
  static const char* rr_dump = getenv("CHFSI_RR_DUMP");  // directory: every projected matrix as raw column-major
  if (rr_dump && ctx->rank == 0) {
    static int dump_no = 0;
    std::vector<T> hg((size_t)ka * ka);
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(hg.data(), G, sizeof(T) * hg.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    const std::string path = std::string(rr_dump) + "/g_" + std::to_string(dump_no++) + "_k" + std::to_string(ka) + ".bin";
    if (FILE* f = fopen(path.c_str(), "wb")) {
      fwrite(hg.data(), sizeof(T), hg.size(), f);
      fclose(f);
    }
  }
  if (rr_log && ctx->rank == 0) {
    std::vector<T> hg((size_t)ka * ka);
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(hg.data(), G, sizeof(T) * hg.size(), cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    double off = 0, tot = 0, offmax = 0;
    for (int64_t j = 0; j < ka; ++j)
      for (int64_t i = 0; i < ka; ++i) {
        const T& g = hg[(size_t)j * ka + i];
        double a2;
        if constexpr (S::elem == 2) a2 = g.x * g.x + g.y * g.y; else a2 = g * g;
        tot += a2;
        if (i != j) off += a2, offmax = std::max(offmax, std::sqrt(a2));
      }
    fprintf(stderr, "rr k %lld offdiag_rel %.3e offdiag_max %.3e\n", (long long)ka, std::sqrt(off / tot), offmax);
  }
  // small dense eigensolve: once, on rank 0, broadcast (identical bits on every rank)
  CHFSI_CUDA_TRY(ctx, cudaMemsetAsync(info, 0, sizeof(double), ctx->stream));
  if (ctx->rank == 0) {
    for (auto& ev : ctx->eig_ev)
      if (!ev) CHFSI_CUDA_TRY(ctx, cudaEventCreate(&ev));
    CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->eig_ev[0], ctx->stream));
    // the nearly diagonal G of a problem's later loops: Jacobi-type refinement (eig_refine.cu); otherwise
    // (or when it declines) the dense ZHEEVD
    bool refined = false;
    int steps = 0;
    if (ctx->eig_mode == 0) TRY(eig_refine<T>(ctx, ka, G, dmu, &refined, &steps));
    if (refined) {
      ctx->eig_refined++;
    } else {
      int lw = 0;
      CUSOLVER_TRY(ctx, S::heevd_bs(ctx->cusolver, (int)ka, G, (int)ka, dmu, &lw));
      TRY(ensure(ctx, ctx->solver_ws, eb * (size_t)std::max(lw, 1)));
      CUSOLVER_TRY(ctx, S::heevd(ctx->cusolver, (int)ka, G, (int)ka, dmu, static_cast<T*>(ctx->solver_ws.ptr), lw, info));
      ctx->eig_dense++;
    }
    CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->eig_ev[1], ctx->stream));
  }
  TRY(comm_bcast(ctx, reinterpret_cast<double*>(G), (size_t)S::elem * ka * ka, 0));
  TRY(comm_bcast(ctx, dmu, (size_t)ka, 0));
  // rank 0's info travels with the result (8 bytes), so every rank takes the same error branch
  TRY(comm_bcast(ctx, reinterpret_cast<double*>(info), 1, 0));
  CUBLAS_TRY(ctx, S::gemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, (int)nloc, (int)ka, (int)ka, &one, Qt, (int)ldq, G,
                          (int)ka, &zero, Yr, (int)nloc));
  if (resid) {
    CUBLAS_TRY(ctx, S::gemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, (int)nloc, (int)ka, (int)ka, &one, W, (int)nloc, G,
                            (int)ka, &zero, HY, (int)nloc));
    CHFSI_CUDA_TRY(ctx, launch_resid2(nloc, ka, reinterpret_cast<const D*>(HY), nloc, reinterpret_cast<const D*>(Yr),
                                      nloc, dmu, dr, ctx->stream));
    CHFSI_CUDA_TRY(ctx, launch_colnorm2(nloc, ka, reinterpret_cast<const D*>(Yr), nloc, dn, ctx->stream));
    ctx->launches += 2;
    TRY(comm_allreduce_sum(ctx, dr, (size_t)2 * ka));  // dr and dn are contiguous
  }
  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Q, eb * ldq, Yr, eb * nloc, eb * nloc, ka, cudaMemcpyDeviceToDevice,
                                        ctx->stream));
  std::vector<double> h(3 * ka);
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(h.data(), dmu, sizeof(double) * (resid ? 3 * ka : ka), cudaMemcpyDeviceToHost,
                                      ctx->stream));
  int hinfo = 0;
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->rank == 0) {
    float ms = 0;
    CHFSI_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->eig_ev[0], ctx->eig_ev[1]));
    ctx->eig_seconds += 1e-3 * ms;
  }
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

// explicit instantiations + the complex entry points used by the C-ABI and the solver
template chfsi_status lanczos_t<cuDoubleComplex>(chfsi_ctx, int64_t, int64_t, int64_t, const void*, int64_t, int32_t,
                                                 uint64_t, double*, double*, double*);
template chfsi_status lanczos_t<double>(chfsi_ctx, int64_t, int64_t, int64_t, const void*, int64_t, int32_t, uint64_t,
                                        double*, double*, double*);
template chfsi_status qr_t<cuDoubleComplex>(chfsi_ctx, int64_t, int64_t, int64_t, const void*, int64_t, int64_t, void*,
                                            int64_t, int64_t, uint64_t, int32_t*, int32_t*);
template chfsi_status qr_t<double>(chfsi_ctx, int64_t, int64_t, int64_t, const void*, int64_t, int64_t, void*, int64_t,
                                   int64_t, uint64_t, int32_t*, int32_t*);
template chfsi_status rr_t<cuDoubleComplex>(chfsi_ctx, int64_t, int64_t, int64_t, const void*, int64_t, void*, int64_t,
                                            int64_t, double, double*, double*);
template chfsi_status rr_t<double>(chfsi_ctx, int64_t, int64_t, int64_t, const void*, int64_t, void*, int64_t, int64_t,
                                   double, double*, double*);

chfsi_status lanczos_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                          int32_t steps, uint64_t seed, double* theta_min, double* theta_max, double* upper) {
  return lanczos_t<cuDoubleComplex>(ctx, n, row0, nloc, Hp, ldh, steps, seed, theta_min, theta_max, upper);
}
chfsi_status qr_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* XL, int64_t ldxl, int64_t nl,
                     void* Y, int64_t ldy, int64_t ka, uint64_t seed, int32_t* used_fallback, int32_t* replaced) {
  return qr_t<cuDoubleComplex>(ctx, n, row0, nloc, XL, ldxl, nl, Y, ldy, ka, seed, used_fallback, replaced);
}
chfsi_status rr_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh, void* Q,
                     int64_t ldq, int64_t ka, double normH, double* mu, double* resid) {
  return rr_t<cuDoubleComplex>(ctx, n, row0, nloc, Hp, ldh, Q, ldq, ka, normH, mu, resid);
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
      !upper_bound || (nloc * ctx->nranks != n || row0 != nloc * ctx->rank)) {
    set_err(ctx, "chfsi_lanczos_bounds: bad arguments");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  return lanczos_impl(ctx, n, row0, nloc, Hp, ldh, steps, seed, theta_min, theta_max, upper_bound);
}

chfsi_status chfsi_qr(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, void* Y, int64_t ldy, int64_t k,
                      int64_t nlocked, int32_t* used_fallback) {
  return chfsi_qr_ex(ctx, n, row0, nloc, Y, ldy, k, nlocked, 0, used_fallback, nullptr);
}

chfsi_status chfsi_qr_ex(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, void* Y, int64_t ldy, int64_t k,
                         int64_t nlocked, uint64_t seed, int32_t* used_fallback, int32_t* replaced) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || nloc < 1 || row0 < 0 || row0 + nloc > n || ldy < nloc || k < 0 || k > n || k > 65536 ||
      nlocked < 0 || nlocked > k || (k > 0 && !Y) || (nloc * ctx->nranks != n || row0 != nloc * ctx->rank)) {
    set_err(ctx, "chfsi_qr: bad arguments (k <= 65536 for the R23 replacement streams)");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  double2* y = static_cast<double2*>(Y);
  return qr_impl(ctx, n, row0, nloc, y, ldy, nlocked, y + (size_t)ldy * nlocked, ldy, k - nlocked, seed, used_fallback,
                 replaced);
}

chfsi_status chfsi_rayleigh_ritz(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                                 void* Q, int64_t ldq, int64_t k, double normH, double* ritz, double* resid) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || nloc < 1 || row0 < 0 || row0 + nloc > n || ldh < n || ldq < nloc || k < 0 || k > n ||
      (k > 0 && (!Hp || !Q || !ritz)) || (resid && !(normH > 0)) ||
      (nloc * ctx->nranks != n || row0 != nloc * ctx->rank)) {
    set_err(ctx, "chfsi_rayleigh_ritz: bad arguments");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  return rr_impl(ctx, n, row0, nloc, Hp, ldh, Q, ldq, k, normH, ritz, resid);
}

}  // extern "C"
