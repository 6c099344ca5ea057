// eig_refine.cu -- the k x k eigensolve of Rayleigh-Ritz (Alg 1 lines 7-9; the paper's
// EleMRRR step) for the nearly diagonal projected matrices of ChFSI's later loops.
//
// After a problem's first loop, Q = QR(filtered Ritz vectors) is close to the Ritz basis, so
// G = Q^H H Q is close to diagonal: the off-diagonal couplings are 1e-6 .. 3e-1 of the gaps between the
// diagonal entries (profiles/r02_rr_probe.jsonl). Instead of a dense ZHEEVD (a latency-bound ~9 ms at
// k = 624 on B200), every coupling is removed at once by a Jacobi-type simultaneous first-order
// rotation, iterated to quadratic convergence with the non-orthogonality folded in (the refinement of
// Ogita & Aishima, 2018), started from X = I:
//   S = X^H G X,  M = X^H X,  lam_i = S_ii / M_ii (Rayleigh quotients),
//   E_ij = (S_ij - lam_j M_ij) / (lam_j - lam_i)  (i != j),  E_ii = (1 - M_ii) / 2,  X <- X (I + E).
// The first step (X = I: S = G, M = I) needs no product; every later one is 4 k^3-class cuBLAS calls
// (G X, X^H (G X) and X^H X as Hermitian rank-k updates, X (I + E)). The largest |E_ij| (i != j) decides:
// above kTheta (a coupling comparable to its gap: first order is not enough) or not decreasing -> the
// dense eigensolve; at most kStop -> converged (the update just applied leaves errors ~ |E|^2 << eps).
// Eigenvalues are the Rayleigh quotients of the last step, sorted ascending (stable) with their columns.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include <cstring>

#include "blas_traits.cuh"
#include "small_kernels.cuh"
#include "supporting.cuh"

namespace chfsi {

namespace {

constexpr double kTheta = 0.3;  // largest first-order coupling |E_ij| the refinement accepts
constexpr double kStop = 1e-7;  // converged once every |E_ij| <= kStop (error after the update ~ 1e-14)
constexpr int kMaxSteps = 8;

__device__ __forceinline__ double re_(double2 a) { return a.x; }
__device__ __forceinline__ double re_(double a) { return a; }
__device__ __forceinline__ double abs_(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double abs_(double a) { return fabs(a); }
__device__ __forceinline__ double2 conj_(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double conj_(double a) { return a; }
__device__ __forceinline__ double2 axpy_div(double2 s, double l, double2 m, double d) {  // (s - l m) / d
  return make_double2((s.x - l * m.x) / d, (s.y - l * m.y) / d);
}
__device__ __forceinline__ double axpy_div(double s, double l, double m, double d) { return (s - l * m) / d; }
__device__ __forceinline__ double2 div_(double2 s, double d) { return make_double2(s.x / d, s.y / d); }
__device__ __forceinline__ double div_(double s, double d) { return s / d; }
template <typename D>
__device__ __forceinline__ D real_(double v);
template <>
__device__ __forceinline__ double2 real_<double2>(double v) {
  return make_double2(v, 0.0);
}
template <>
__device__ __forceinline__ double real_<double>(double v) {
  return v;
}
// upper-triangle storage (herk / herkx): element (i, j) of the Hermitian matrix
template <typename D>
__device__ __forceinline__ D herm_at(const D* A, int64_t ld, int64_t i, int64_t j) {
  return i <= j ? A[j * ld + i] : conj_(A[i * ld + j]);
}

__device__ __forceinline__ void max_out(double m, unsigned long long* out) {
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __double_as_longlong(m));  // m >= 0 (or inf): bit order = order
}

// step 1 (X = I): lam_i = G_ii, P = I + E with E_ij = G_ij / (G_jj - G_ii); an exact tie with a non-zero
// coupling gives inf (-> the dense eigensolve)
template <typename D>
__global__ void jr_first_kernel(int64_t k, const D* __restrict__ G, int64_t ldg, D* __restrict__ P, int64_t ldp,
                                double* lam, unsigned long long* emax) {
  double m = 0.0;
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
    const double lj = re_(G[j * ldg + j]);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
      D e;
      if (i == j) {
        e = real_<D>(1.0);
        lam[i] = lj;
      } else {
        const D g = G[j * ldg + i];
        const double a = abs_(g);
        e = a == 0.0 ? real_<D>(0.0) : div_(g, lj - re_(G[i * ldg + i]));
        const double ae = abs_(e);
        m = fmax(m, ae != ae ? INFINITY : ae);  // NaN -> inf (fmax would drop it)
      }
      P[j * ldp + i] = e;
    }
  }
  max_out(m, emax);
}

// step t >= 2 from S = X^H G X and M = X^H X (upper triangles): lam_i = S_ii / M_ii; P = I + E
template <typename D>
__global__ void jr_update_kernel(int64_t k, const D* __restrict__ S, const D* __restrict__ M, int64_t ld,
                                 D* __restrict__ P, int64_t ldp, double* lam, unsigned long long* emax) {
  double m = 0.0;
  for (int64_t j = blockIdx.y; j < k; j += gridDim.y) {
    const double mjj = re_(M[j * ld + j]);
    const double lj = re_(S[j * ld + j]) / mjj;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += (int64_t)gridDim.x * blockDim.x) {
      D e;
      if (i == j) {
        e = real_<D>(1.0 + 0.5 * (1.0 - mjj));
        lam[i] = lj;
      } else {
        const double li = re_(S[i * ld + i]) / re_(M[i * ld + i]);
        e = axpy_div(herm_at(S, ld, i, j), lj, herm_at(M, ld, i, j), lj - li);
        const double ae = abs_(e);
        m = fmax(m, ae != ae ? INFINITY : ae);
      }
      P[j * ldp + i] = e;
    }
  }
  max_out(m, emax);
}

inline dim3 grid2(int64_t k) {
  return dim3((unsigned)((k + 255) / 256), (unsigned)std::min<int64_t>(k, 65535));
}

}  // namespace

template <typename T>
chfsi_status eig_refine(chfsi_ctx ctx, int64_t ka, T* G, double* dmu, bool* done, int* steps) {
  using S = Sc<T>;
  using D = typename S::D;
  *done = false;
  *steps = 0;
  if (ka < 2) return CHFSI_OK;  // the dense path handles the trivial sizes
  const size_t kk = (size_t)ka * ka;
  TRY(ensure(ctx, ctx->eigw, sizeof(T) * 5 * kk + sizeof(double) * (size_t)(ka + 8) + sizeof(int) * (size_t)ka));
  T* Xa = static_cast<T*>(ctx->eigw.ptr);
  T* Xb = Xa + kk;
  T* Tm = Xb + kk;  // G X, then the next step's I + E
  T* Sm = Tm + kk;  // X^H G X (upper)
  T* Mm = Sm + kk;  // X^H X (upper)
  double* lam = reinterpret_cast<double*>(Mm + kk);
  unsigned long long* emax = reinterpret_cast<unsigned long long*>(lam + ka);
  int* perm = reinterpret_cast<int*>(lam + ka + 8);
  const T one = S::one(), zero = S::zero();
  const int k = (int)ka;
  auto read_emax = [&](double* h) -> chfsi_status {
    unsigned long long bits = 0;
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&bits, emax, sizeof(bits), cudaMemcpyDeviceToHost, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    std::memcpy(h, &bits, sizeof(double));
    return CHFSI_OK;
  };
  // step 1: X_1 = I + E_1 straight from G
  CHFSI_CUDA_TRY(ctx, cudaMemsetAsync(emax, 0, sizeof(*emax), ctx->stream));
  jr_first_kernel<D><<<grid2(ka), 256, 0, ctx->stream>>>(ka, reinterpret_cast<const D*>(G), ka,
                                                         reinterpret_cast<D*>(Xa), ka, lam, emax);
  CHFSI_CUDA_TRY(ctx, cudaGetLastError());
  ctx->launches++;
  double e = 0.0, prev = INFINITY;
  TRY(read_emax(&e));
  *steps = 1;
  if (!(e <= kTheta)) return CHFSI_OK;
  T* X = Xa;
  T* Xn = Xb;
  bool conv = e <= kStop;
  prev = e;
  for (int it = 2; it <= kMaxSteps && !conv; ++it) {
    CUBLAS_TRY(ctx, S::gemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, k, k, k, &one, G, k, X, k, &zero, Tm, k));
    CUBLAS_TRY(ctx, S::herkx_c(ctx->cublas, k, k, X, k, Tm, k, Sm, k));
    CUBLAS_TRY(ctx, S::herk_c(ctx->cublas, k, k, X, k, Mm, k));
    CHFSI_CUDA_TRY(ctx, cudaMemsetAsync(emax, 0, sizeof(*emax), ctx->stream));
    jr_update_kernel<D><<<grid2(ka), 256, 0, ctx->stream>>>(ka, reinterpret_cast<const D*>(Sm),
                                                            reinterpret_cast<const D*>(Mm), ka,
                                                            reinterpret_cast<D*>(Tm), ka, lam, emax);
    CHFSI_CUDA_TRY(ctx, cudaGetLastError());
    ctx->launches++;
    TRY(read_emax(&e));
    *steps = it;
    if (!(e <= kTheta) || !(e < prev)) return CHFSI_OK;  // not converging at first order: dense eigensolve
    prev = e;
    CUBLAS_TRY(ctx, S::gemm(ctx, CUBLAS_OP_N, CUBLAS_OP_N, k, k, k, &one, X, k, Tm, k, &zero, Xn, k));
    std::swap(X, Xn);
    conv = e <= kStop;
  }
  if (!conv) return CHFSI_OK;
  // ascending (stable) order of the Rayleigh quotients; G <- the eigenvector columns in that order
  std::vector<double> hl(ka);
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(hl.data(), lam, sizeof(double) * ka, cudaMemcpyDeviceToHost, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  std::vector<int> ord(ka);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return hl[a] < hl[b]; });
  std::vector<double> sorted(ka);
  for (int64_t j = 0; j < ka; ++j) sorted[j] = hl[ord[j]];
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(perm, ord.data(), sizeof(int) * ka, cudaMemcpyHostToDevice, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(dmu, sorted.data(), sizeof(double) * ka, cudaMemcpyHostToDevice, ctx->stream));
  CHFSI_CUDA_TRY(ctx, launch_col_gather(ka, ka, reinterpret_cast<const D*>(X), ka, perm, reinterpret_cast<D*>(G), ka,
                                        ctx->stream));
  ctx->launches++;
  // no synchronisation: a copy from pageable host memory returns once its source has been staged, so
  // ord / sorted may go out of scope; the caller synchronises before it reads the results
  *done = true;
  return CHFSI_OK;
}

template chfsi_status eig_refine<cuDoubleComplex>(chfsi_ctx, int64_t, cuDoubleComplex*, double*, bool*, int*);
template chfsi_status eig_refine<double>(chfsi_ctx, int64_t, double*, double*, bool*, int*);

}  // namespace chfsi
