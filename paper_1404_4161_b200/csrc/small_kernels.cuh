// small_kernels.cuh -- the supporting (non-filter) device kernels of ChFSI: the Lanczos mat-vec (K2,
// HBM-bound), per-column reductions for norms / residuals (K6), Hermitisation (K9), column gathers
// and scalings (K7), and the counter-based random block (R22). All reductions run in a fixed order
// (deterministic, independent of launch timing).
#pragma once
#include "common.cuh"

namespace chfsi {

// w[r] = sum_q conj(Hp[q, r]) v[q] for the nloc local rows r (K2: one warp per row, HBM-bound:
// 16 n nloc bytes per call)
// hpp (nullable): read the panel pointer from this device slot instead of Hp (a captured graph replays
// against whatever panel the slot holds)
cudaError_t launch_hemv(int64_t n, int64_t nloc, const double2* Hp, int64_t ldh, const double2* v, double2* w,
                        cudaStream_t st, const void* const* hpp = nullptr);
// out[j] = sum_r |X[r, j]|^2 (rows x cols)
cudaError_t launch_colnorm2(int64_t rows, int64_t cols, const double2* X, int64_t ldx, double* out, cudaStream_t st);
// out[j] = sum_r |HY[r, j] - mu[j] Y[r, j]|^2 (mu on device)
cudaError_t launch_resid2(int64_t rows, int64_t cols, const double2* HY, int64_t ld1, const double2* Y, int64_t ld2,
                          const double* mu, double* out, cudaStream_t st);
// G <- (G + G^H)/2, imaginary diagonal set to 0
cudaError_t launch_hermitize(int64_t k, double2* G, int64_t ldg, cudaStream_t st);
// dst[:, j] = src[:, idx[j]] for j < cols (idx on device); src and dst must not overlap
cudaError_t launch_col_gather(int64_t rows, int64_t cols, const double2* src, int64_t lds, const int* idx,
                              double2* dst, int64_t ldd, cudaStream_t st);
// Q[:, j] *= phase(R[j, j]) (Householder fallback: make R's diagonal real positive)
cudaError_t launch_col_phase(int64_t rows, int64_t cols, double2* Q, int64_t ldq, const double2* R, int64_t ldr,
                             cudaStream_t st);
// X[r, j] = (2u_{2g} - 1) + i (2u_{2g+1} - 1), g = row0 + r, u from splitmix64(seed ^ (stream_j << 40) ^ idx),
// stream_j = stream_base | j (R22)
cudaError_t launch_random_block(int64_t rows, int64_t cols, int64_t row0, uint64_t seed, uint64_t stream_base,
                                uint64_t stream_stride, double2* X, int64_t ldx, cudaStream_t st);
// x[i] *= s (device scalar s = 1/beta computed on the host)
cudaError_t launch_scale(int64_t rows, double2* x, double s, cudaStream_t st);
// G[i,j] for i<k: make identity minus G, return max |entry| into out[0] via atomicMax on the bit pattern
cudaError_t launch_orth_err(int64_t k, const double2* G, int64_t ldg, double* out, cudaStream_t st);

// 3M filter operands. H3[r * ld3 + c * ldk + o] = Re Hp[q, r] - Im Hp[q, r] for the
// nloc local rows r and K entries q = c * chunk + o (the rank chunks of the contraction, each padded to
// ldk >= chunk with zeros; chunk = ldk = n on one rank). K-major like the interleaved A operand;
// HBM-bound, 24 bytes per entry.
cudaError_t launch_h3_plane(int64_t n, int64_t nloc, const double2* Hp, int64_t ldh, double* H3, int64_t ld3,
                            int64_t chunk, int64_t ldk, cudaStream_t st);
// extended column layout of a B operand: dst + j * cs holds column j of X as rows complex values,
// followed at double offset y3_off by the plane Re X[:, j] + Im X[:, j] (cs, y3_off in doubles)
cudaError_t launch_pack_y3(int64_t rows, int64_t cols, const double2* X, int64_t ldx, double* dst, int64_t cs,
                           int64_t y3_off, cudaStream_t st);

// one Lanczos step finished on the device: beta = sqrt(*nrm2), vn = w / beta (vn nullable), alpha =
// Re(*coef_j) (alpha_out nullable); *beta_out, *alpha_out written (device) -- the host reads all steps'
// scalars once
cudaError_t launch_lanczos_next(int64_t rows, const double2* w, double2* vn, const double* nrm2, const double2* coef_j,
                                double* beta_out, double* alpha_out, cudaStream_t st);
cudaError_t launch_lanczos_next(int64_t rows, const double* w, double* vn, const double* nrm2, const double* coef_j,
                                double* beta_out, double* alpha_out, cudaStream_t st);

// x *= 1 / sqrt(*nrm2) (device scalar; the Lanczos start vector without a host round trip)
cudaError_t launch_scale_rnorm(int64_t rows, double2* x, const double* nrm2, cudaStream_t st);
cudaError_t launch_scale_rnorm(int64_t rows, double* x, const double* nrm2, cudaStream_t st);
// *slot = ptr (stream-ordered)
cudaError_t launch_store_ptr(const void** slot, const void* ptr, cudaStream_t st);

// ---- real-symmetric (NEXT-3) counterparts, same semantics on double data ----
cudaError_t launch_hemv(int64_t n, int64_t nloc, const double* Hp, int64_t ldh, const double* v, double* w,
                        cudaStream_t st, const void* const* hpp = nullptr);
cudaError_t launch_colnorm2(int64_t rows, int64_t cols, const double* X, int64_t ldx, double* out, cudaStream_t st);
cudaError_t launch_resid2(int64_t rows, int64_t cols, const double* HY, int64_t ld1, const double* Y, int64_t ld2,
                          const double* mu, double* out, cudaStream_t st);
cudaError_t launch_hermitize(int64_t k, double* G, int64_t ldg, cudaStream_t st);
cudaError_t launch_col_gather(int64_t rows, int64_t cols, const double* src, int64_t lds, const int* idx, double* dst,
                              int64_t ldd, cudaStream_t st);
// Q[:, j] *= sign(R[j, j])
cudaError_t launch_col_phase(int64_t rows, int64_t cols, double* Q, int64_t ldq, const double* R, int64_t ldr,
                             cudaStream_t st);
// X[r, j] = 2u_{2g} - 1 (the real part of the complex R22 formula)
cudaError_t launch_random_block(int64_t rows, int64_t cols, int64_t row0, uint64_t seed, uint64_t stream_base,
                                uint64_t stream_stride, double* X, int64_t ldx, cudaStream_t st);
cudaError_t launch_scale(int64_t rows, double* x, double s, cudaStream_t st);
cudaError_t launch_orth_err(int64_t k, const double* G, int64_t ldg, double* out, cudaStream_t st);

}  // namespace chfsi
