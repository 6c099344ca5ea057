// supporting.cuh -- internal entry points of the supporting ChFSI steps (supporting.cu), used by the
// public C-ABI wrappers and by the sequence solver (solver.cu).
#pragma once
#include <cuComplex.h>

#include "ctx.cuh"

namespace chfsi {

chfsi_status lanczos_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                          int32_t steps, uint64_t seed, double* theta_min, double* theta_max, double* upper);
// Orthonormalise Y (nloc x ka) against XL (nloc x nl, orthonormal, untouched) and itself, with the
// rank-deficiency rule R23 (replacement vectors: R22, seed + round, stream (6 << 16) | (nl + j)).
// used_fallback / replaced: host, nullable.
chfsi_status qr_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* XL, int64_t ldxl, int64_t nl,
                     void* Y, int64_t ldy, int64_t ka, uint64_t seed, int32_t* used_fallback, int32_t* replaced);
// Rayleigh-Ritz on Q (in/out); mu host[ka] ascending; resid host[ka] nullable (R8).
chfsi_status rr_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh, void* Q,
                     int64_t ldq, int64_t ka, double normH, double* mu, double* resid);

// the same steps templated on the scalar (cuDoubleComplex: Hermitian; double: real symmetric, NEXT-3)
template <typename T>
chfsi_status lanczos_t(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh, int32_t steps,
                       uint64_t seed, double* theta_min, double* theta_max, double* upper);
template <typename T>
chfsi_status qr_t(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* XL, int64_t ldxl, int64_t nl, void* Y,
                  int64_t ldy, int64_t ka, uint64_t seed, int32_t* used_fallback, int32_t* replaced);
template <typename T>
chfsi_status rr_t(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh, void* Q,
                  int64_t ldq, int64_t ka, double normH, double* mu, double* resid);

// k x k Hermitian eigensolve of Rayleigh-Ritz by the Jacobi-type refinement (eig_refine.cu). On success
// (*done = true) G holds the eigenvectors (columns ascending by eigenvalue) and dmu (device) the
// eigenvalues; otherwise G is untouched and the caller runs the dense eigensolve. *steps: steps taken.
template <typename T>
chfsi_status eig_refine(chfsi_ctx ctx, int64_t ka, T* G, double* dmu, bool* done, int* steps);

}  // namespace chfsi
