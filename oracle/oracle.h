/* oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the CUDA path computes, used only by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs. The product
 * path (paper_1404_4161_b200/) never includes, links or calls anything here, and this file shares no
 * code with it.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / algorithm / equation named at each
 * function); S:n = SPEC.md line n; "R<k>" = the reading of the paper listed in DESIGN.md section 3.
 * Arithmetic: IEEE binary64, explicit re/im complex arithmetic, built with -O2 -fno-fast-math
 * -ffp-contract=off (R18). Complex data is interleaved complex128 (re, im), column-major, explicit
 * leading dimension. Every reduction runs in a fixed order per output element, so results do not
 * depend on the OpenMP thread count.
 *
 * Parity pins (tests/test_oracle_*.py) for each function are listed in DESIGN.md section 4; there is
 * no "parity unpinned" function in this file except the solver trajectory (loop counts, degree
 * vectors), which is unpinned by nature.
 */
#ifndef CHFSI_ORACLE_H
#define CHFSI_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- Chebyshev polynomials (eq:polydef) --------------------------------------------- */
/* C_m(t) = cosh(m acosh t) for t >= 1, (-1)^m cosh(m acosh(-t)) for t <= -1, cos(m acos t) inside. */
long double ora_cheb(int32_t m, long double t);
/* Normalised filter value p_m(lam) = C_m((lam-c)/e) / C_m((lambda1-c)/e). */
long double ora_filter_gain(int32_t m, long double lam, long double lambda1, long double c,
                            long double e);
/* sigma_1 = e/(lambda1-c) (Alg 2 l2); sigma_{i+1} = 1/(2/sigma_1 - sigma_i) (Alg 2 l6).
 * sigma[0..mmax-1] = sigma_1..sigma_mmax. */
void ora_sigma(int32_t mmax, double lambda1, double c, double e, double* sigma);

/* ---- Chebyshev filter (Alg 2) -------------------------------------------------------- */
/* Y (n x k, in: Y_0, out: Y_m) filtered in place; column j with degree deg[j] (ascending, >= 1).
 * H is the full n x n Hermitian matrix; H~ = (H - cI)/e is applied as (H Y - c Y)/e.
 * Reading R1: line 8's trailing term is Y_{i-1}. R2: columns run to k. R3: s = first active column.
 * Returns 0, or 1 on bad arguments, 2 on a non-finite result. matvecs (nullable) += sum(deg). */
int32_t ora_filter(int64_t n, const double* H, int64_t ldh, double* Y, int64_t ldy, int64_t k,
                   const int32_t* deg, double lambda1, double c, double e, int64_t* matvecs);
/* Closed form for diagonal H = diag(d): Y[r,j] *= p_{deg[j]}(d_r) in long double (App. A). */
void ora_filter_diag_closed(int64_t n, const double* d, double* Y, int64_t ldy, int64_t k,
                            const int32_t* deg, double lambda1, double c, double e);
/* Closed form for H = Q diag(lam) Q^H with Q = I - V T V^H (8 reflectors): Y[:,j] <-
 * Q diag(p_{deg[j]}(lam)) Q^H Y[:,j], O(n k 8) work. */
void ora_filter_wy_closed(int64_t n, const double* lam, const double* V, const double* T,
                          double* Y, int64_t ldy, int64_t k, const int32_t* deg, double lambda1,
                          double c, double e);

/* ---- dense building blocks ---------------------------------------------------------------------- */
/* C (m x n) = op(A) op(B), op in {'N','C'} (C = conjugate transpose); inner dimension kk. */
void ora_zgemm(char ta, char tb, int64_t m, int64_t n, int64_t kk, const double* A, int64_t lda,
               const double* B, int64_t ldb, double* C, int64_t ldc);
/* Householder QR ("Householder reflectors based QR"): A (n x k) -> Q (n x k) orthonormal and
 * R (k x k, upper, real positive diagonal; nullable) with A = Q R. Returns the number of columns
 * whose |R_jj| < 1e-12 * ||a_j|| (numerically rank deficient), 0 normally. */
int32_t ora_householder_qr(int64_t n, int64_t k, const double* A, int64_t lda, double* Q,
                           int64_t ldq, double* R, int64_t ldr);
/* Cyclic complex Jacobi eigensolver for a Hermitian n x n A: w ascending (stable by index),
 * V (n x n) eigenvectors, each phase-normalised so its largest-|.| entry is real positive (ties:
 * lowest row). Returns the number of sweeps, or -1 if it did not converge in 60 sweeps. */
int32_t ora_jacobi_eig(int64_t n, const double* A, int64_t lda, double* w, double* V, int64_t ldv);

/* ---- supporting steps of Alg 1 ------------------------------------------------------------------ */
/* Counter-based vector used by the method (Lanczos start, QR replacement), R22:
 * u_t = (splitmix64(seed ^ (stream << 40) ^ t) >> 11) 2^-53, x_i = (2u_{2i}-1) + i (2u_{2i+1}-1). */
void ora_random_vector(int64_t n, uint64_t seed, uint64_t stream, double* x);
/* Lanczos (Alg 1 l3; R17): `steps` iterations with full reorthogonalisation from the
 * normalised ora_random_vector(seed, stream 4<<16 | restart). Outputs theta_min, theta_max of T and
 * beta_up = theta_max + ||f||. Breakdown (beta_j < 1e-14 ||H||_est) restarts, at most 3 times
 * (S:284). Returns 0, or 1 on failure. */
int32_t ora_lanczos(int64_t n, const double* H, int64_t ldh, int32_t steps, uint64_t seed,
                    double* theta_min, double* theta_max, double* beta_up);
/* Rayleigh-Ritz (Alg 1 l7-9): G = Q^H H Q hermitised, G W = W diag(mu), Q <- Q W
 * (phase-normalised W). ritz[k] ascending. */
int32_t ora_rayleigh_ritz(int64_t n, const double* H, int64_t ldh, double* Q, int64_t ldq,
                          int64_t k, double* ritz);
/* resid[j] = ||H x_j - lam_j x_j||_2 / (||x_j||_2 * normH) (R8; eq:resl definition). */
void ora_residuals(int64_t n, const double* H, int64_t ldh, const double* X, int64_t ldx, int64_t k,
                   const double* lam, double normH, double* resid);
/* Rayleigh quotients rho_j = Re(x_j^H H x_j)/(x_j^H x_j) and absolute residuals ||H x_j - rho_j x_j|| /
 * ||x_j|| of the columns of X (n x k), naive (the Kato-Temple / residual checks of SURVEY 8(c) c4). */
void ora_rayleigh_quotients(int64_t n, const double* H, int64_t ldh, const double* X, int64_t ldx, int64_t k,
                            double* rho, double* resid_abs);
/* Degree rule R21: smallest m with C_m(|t|) >= max(res/tol, 1), clamped to [1, cap]; |t| <= 1 -> cap. */
int32_t ora_degree(double res, double tol, double t, int32_t cap);
/* Literal degree bound: ceil(ln(res/tol)/ln rho), clamped to [1, cap]. */
int32_t ora_degree_literal(double res, double tol, double rho, int32_t cap);
/* |rho| = |t| + sqrt(t^2-1) for |t| > 1 (eq:ratio), 1 inside [-1,1] (R5). */
double ora_rho(double t);

/* Alg 1 l6 with the QR rank-deficiency rule R23: the active
 * block Y (n x ka, ld n, in/out) is orthonormalised against the locked block XL (n x nl, ld n; left
 * unchanged) by CGS2 and then by Householder QR; a column j with |R_jj| <= 1e-12 ||y_j(input)|| is
 * replaced by the R22 vector (seed + round, stream (6 << 16) | (nl + j)) and the block is redone
 * (at most 3 rounds). *replaced (nullable) = the number of replacements. Returns 0, or 4 if columns
 * were still deficient after 3 rounds. */
int32_t ora_orthonormalize(int64_t n, const double* XL, int64_t nl, double* Y, int64_t ka, uint64_t seed,
                           int32_t* replaced);

typedef struct {
  int32_t nev, nex, deg0, deg_cap, max_loops, lanczos_steps;
  double tol;
  uint64_t seed;
} ora_opts;

typedef struct {
  int32_t loops, capped, qr_replaced, converged;
  int64_t matvecs_filter, matvecs_total;
  double theta_min, theta_max, beta_up, normH;
} ora_report;

/* ChFSI for one eigenproblem (Alg 1) with the readings R4-R12, R16, R21.
 * X: n x k (k = nev + nex), in: start block (have_prev = 0: arbitrary, e.g. random) or the previous
 * problem's hand-off; out: hand-off block [locked (ascending) | remaining active]. lambda1/lambdak:
 * in (used when have_prev), out (smallest / largest of the final k values). lam[nev], resid[nev]:
 * the converged eigenvalues (ascending) and their residuals; X[:, 0:nev] are their vectors.
 * QR rank deficiency follows R23 (ora_orthonormalize, seed = opts->seed; rep->qr_replaced counts it).
 * Returns 0, 3 if max_loops was hit (partial results), 1 on bad arguments, 4 if R23 failed. */
int32_t ora_chfsi_solve(int64_t n, const double* H, int64_t ldh, const ora_opts* opts, double* X,
                        int64_t ldx, int32_t have_prev, double* lambda1, double* lambdak,
                        double* lam, double* resid, ora_report* rep);

/* ---- generalised front / back end (H = L^{-1} A L^{-H}, B = L L^H) --------------------- */
/* Cholesky B = L L^H (L lower, real positive diagonal; upper part of L set to 0). Returns 0, or j+1 if
 * pivot j is not positive. */
int32_t ora_cholesky(int64_t n, const double* B, int64_t ldb, double* L, int64_t ldl);
/* X (n x k) <- L^{-1} X (adjoint = 0) or L^{-H} X (adjoint = 1), forward / backward substitution. */
void ora_trsm_lower(int64_t n, int64_t k, const double* L, int64_t ldl, double* X, int64_t ldx,
                    int32_t adjoint);
/* H = L^{-1} A L^{-H} (hermitised) and L = chol(B). Returns the Cholesky status. */
int32_t ora_reduce_generalized(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                               double* H, int64_t ldh, double* L, int64_t ldl);

/* Number of eigenvalues of H strictly below sigma (Sylvester's law of inertia): H - sigma I =
 * P L D L^H P^T by the Bunch-Kaufman pivoting strategy (1x1 / 2x2 pivots, alpha = (1 + sqrt 17)/8)
 * on a copy of the lower triangle; the count is the number of negative eigenvalues of the block
 * diagonal D. Pinned against numpy.eigvalsh at n >= 512 (shifts within 1e-8 of an eigenvalue), the
 * generator's exact spectrum, and matrices an unpivoted LDL^H miscounts (tests/test_oracle_linalg.py). */
int64_t ora_count_below(int64_t n, const double* H, int64_t ldh, double sigma);

#ifdef __cplusplus
}
#endif
#endif
