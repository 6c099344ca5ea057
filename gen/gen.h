/* gen.h -- seeded synthetic INPUT generator shared by the oracle side and the CUDA side.
 *
 * This module holds none of the method's arithmetic (no filter, no QR, no Rayleigh-Ritz):
 * it only manufactures the inputs the paper's workloads are stood in by (DESIGN.md "Input
 * recipe"):
 *   - the spectrum Lambda(n, n_d): dense log-spaced-density bottom in [-2,0], sparse tail in (0,40];
 *   - Q = P_1 ... P_8 (8 Householder reflectors of N(0,1) complex vectors) in compact WY form
 *     Q = I - V T V^H, and H^(1) = Q Lambda Q^H built entrywise (24 complex MACs per entry);
 *   - the GUE perturbation G_l and the sequence step H^(l+1) = H^(l) + delta*40*G_l (BASELINE.json
 *     configs[1..3]);
 *   - a CN(0,1) start basis, and the c4 GUE test matrix.
 * Every entry is a pure function of (seed, stream, index), so any rank can build any column panel
 * bit-identically and the result does not depend on the thread count.
 * Complex data: interleaved complex128 (re, im), column-major, explicit leading dimension.
 */
#ifndef CHFSI_GEN_H
#define CHFSI_GEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define GEN_NREF 8
/* RNG streams: major << 16 | minor */
#define GEN_STREAM(major, minor) ((((uint64_t)(major)) << 16) | (uint64_t)(minor))

uint64_t gen_splitmix64(uint64_t x);
/* u = (splitmix64(seed ^ (stream << 40) ^ idx) >> 11) * 2^-53, an exact double in [0,1). */
double gen_uniform(uint64_t seed, uint64_t stream, uint64_t idx);
/* Box-Muller pair from uniforms 2*idx and 2*idx+1 (host libm; host-only generator). */
void gen_normal2(uint64_t seed, uint64_t stream, uint64_t idx, double* z0, double* z1);

/* lam[0..n-1] ascending: n_d dense values -2 + 2*log10(1 + 9 i/(n_d-1)), then n-n_d tail values
 * 40*(j+1)/(n-n_d). */
void gen_spectrum(int64_t n, int64_t nd, double* lam);

/* Compact-WY factors of Q = P_1...P_8: V (n x 8), T (8 x 8 upper), both col-major complex. */
void gen_wy(int64_t n, uint64_t seed, double* V, double* T);
/* B = V T (n x 8), A = Lambda V (n x 8), D = B (V^H Lambda V) (n x 8). */
void gen_wy_aux(int64_t n, const double* lam, const double* V, const double* T,
                double* B, double* A, double* D);
/* H^(1)[:, c0:c0+ncols] into H (ld >= n). Upper entries by formula, lower mirrored by conj. */
void gen_h1_panel(int64_t n, const double* lam, const double* B, const double* A, const double* D,
                  int64_t c0, int64_t ncols, double* H, int64_t ldh);
/* X[:, t] = Q e_{idx[t]} = e_i - B conj(V[i,:])^T, t = 0..m-1 (exact eigenvectors of H^(1)). */
void gen_eigvecs(int64_t n, const double* V, const double* B, const int64_t* idx, int64_t m,
                 double* X, int64_t ldx);
/* GUE panel: G[r,c] = (x + i y)/sqrt(2n) (r<c), G[r,r] = x/sqrt(n), Hermitian mirror. */
void gen_gue_panel(int64_t n, uint64_t seed, uint64_t stream, int64_t c0, int64_t ncols,
                   double* G, int64_t ldg);
/* H[:, c0:c0+ncols] <- fl(H + fl(scale * G_ell)) with G_ell from stream (2, ell). */
void gen_perturb_panel(int64_t n, uint64_t seed, int32_t ell, double scale, int64_t c0,
                       int64_t ncols, double* H, int64_t ldh);
/* Rows [r0, r0+nrows) of the n x k start basis Y[r,j] = (x + i y)/sqrt(2), stream (3,0). */
void gen_start_basis(int64_t n, int64_t k, uint64_t seed, int64_t r0, int64_t nrows,
                     double* Y, int64_t ldy);

/* Lower-triangular factor with real positive diagonal for a generalised pair with a known spectrum
 * (DESIGN.md 5): M[i,i] = 1 + 0.5 u_i, M[i,j] = scale (x + i y)/sqrt(2n) for i > j (stream (6,0)),
 * zero above the diagonal. B = M M^H is Hermitian positive definite with Cholesky factor M, and
 * A = M H^(1) M^H has the generalised eigenvalues Lambda. */
void gen_lower_factor(int64_t n, uint64_t seed, double scale, double* M, int64_t ldm);

#ifdef __cplusplus
}
#endif
#endif
