/* chfsi.h -- C-ABI of the B200-native Chebyshev Filtered Subspace Iteration library (libchfsi.so).
 *
 * Paper: Berljafa, Wortmann, Di Napoli, "An Optimized and Scalable Eigensolver for Sequences of
 * Eigenvalue Problems" (arXiv:1404.4161). Citations: P:n = /root/reference/PAPER.md line n (with
 * the section / algorithm / equation it falls in); R<k> = the reading of the paper listed in
 * DESIGN.md section 3.
 *
 * Conventions (all entry points)
 *  - Complex data: interleaved complex128 (double re, double im), column-major, explicit leading
 *    dimension (ld >= rows). Device pointers unless stated "host".
 *  - Distribution (nranks = p >= 1): the rank owns global rows [row0, row0 + nloc) of every n-row
 *    matrix (Y, Q, X). H is passed as its column slab Hp = H[:, row0:row0+nloc] (n x nloc, ldh >= n);
 *    for Hermitian H this is the conjugate of the rank's row panel, and the library applies
 *    (H y)[r] = sum_q conj(Hp[q, r - row0]) y[q] (R13). p == 1: row0 = 0, nloc = n.
 *  - Streams: all device work is enqueued on the context's CUDA stream. A call returns once its
 *    host-visible outputs are valid; device outputs are stream-ordered.
 *  - Ownership: the caller allocates and frees H, Y, Q, X and all host arrays; the library never
 *    frees caller memory. It owns only its workspace (allocated by chfsi_ctx_reserve or on first
 *    use, freed by chfsi_ctx_destroy).
 *  - Errors: every entry point returns a chfsi_status; no exception or abort crosses the ABI. On an
 *    error other than CHFSI_ERR_NOCONV the outputs are unspecified; chfsi_last_error() describes it.
 *  - SPMD (p > 1): every rank calls with identical n, k, degrees, scalars and options.
 *  - There is no CPU fallback: without a usable CUDA device every call returns CHFSI_ERR_CUDA.
 */
#ifndef CHFSI_H
#define CHFSI_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct chfsi_ctx_s* chfsi_ctx;

typedef enum {
  CHFSI_OK = 0,
  CHFSI_ERR_ARG = 1,       /* bad dimension / ld / degree / interval / option */
  CHFSI_ERR_NONFINITE = 2, /* NaN or Inf in a filter output */
  CHFSI_ERR_NOCONV = 3,    /* max_loops reached; outputs hold partial results */
  CHFSI_ERR_QR = 4,        /* CholeskyQR2 and its Householder fallback both failed */
  CHFSI_ERR_CUDA = 5,      /* CUDA / cuBLAS / cuSOLVER failure, or no device */
  CHFSI_ERR_NCCL = 6,      /* NCCL failure or unavailable when nranks > 1 */
  CHFSI_ERR_NOMEM = 7      /* workspace allocation failed */
} chfsi_status;

#define CHFSI_MAX_DEGREE 64

/* Create a context on `device` using `cuda_stream` (a cudaStream_t; NULL = the legacy default
 * stream 0, ordered with the caller's default-stream work). nccl_comm: an ncclComm_t spanning the `nranks` ranks (NULL when nranks == 1). */
chfsi_status chfsi_ctx_create(chfsi_ctx* out, int32_t device, void* cuda_stream, void* nccl_comm,
                              int32_t rank, int32_t nranks);
/* A library-owned NCCL communicator (NVLink / NVSwitch): rank 0 calls chfsi_nccl_unique_id, the caller
 * broadcasts the 128 bytes (e.g. over torch.distributed), then every rank calls chfsi_ctx_create_nccl.
 * The communicator is created with ncclCommInitRank and destroyed with the context. */
chfsi_status chfsi_nccl_unique_id(char id_out[128]);
chfsi_status chfsi_ctx_create_nccl(chfsi_ctx* out, int32_t device, void* cuda_stream, const char id[128],
                                   int32_t rank, int32_t nranks);

/* Emulated ranks: `nranks` contexts in one process, on one device, share a local group whose
 * collectives are device copies ordered by CUDA events and a host barrier (same semantics as the
 * NCCL calls). Drive each rank from its own host thread, each context on its own stream. This runs
 * the nranks > 1 data path (row panels, packed B operands, rank-chunked contraction) on one GPU. */
typedef struct chfsi_local_group_s* chfsi_local_group;
chfsi_status chfsi_local_group_create(chfsi_local_group* out, int32_t nranks);
void chfsi_local_group_destroy(chfsi_local_group group);
chfsi_status chfsi_ctx_create_local(chfsi_ctx* out, int32_t device, void* cuda_stream,
                                    chfsi_local_group group, int32_t rank);

/* Optional: preallocate workspace for problems up to n rows globally, nloc rows per rank and kmax
 * block columns, so no allocation happens inside a timed loop. */
chfsi_status chfsi_ctx_reserve(chfsi_ctx ctx, int64_t n, int64_t nloc, int64_t kmax);
void chfsi_ctx_destroy(chfsi_ctx ctx);
const char* chfsi_last_error(chfsi_ctx ctx);
/* Number of kernels of this library launched on the context since creation (instrumentation). */
int64_t chfsi_kernel_launches(chfsi_ctx ctx);

/* Complex arithmetic of the filter kernel (and of H Q in Rayleigh-Ritz): mults = 3 selects Gauss's
 * 3-multiplication form (default; 6 real flops per complex multiply-add: P1 = sum Re h Re y, P2 = sum
 * Im h Im y, P3 = sum (Re h - Im h)(Re y + Im y); Re = P1 + P2, Im = P3 - P1 + P2 for conj(h) y),
 * mults = 4 the 4M real embedding (8 real flops). Both compute the same p_m(H) Y of Alg 2
 * to rounding; 3M trades a normwise-equivalent error bound (a few ulps more on the imaginary parts)
 * for 25 % fewer tensor-core operations and keeps a (Re H - Im H) plane of the panel (8 bytes per
 * entry) in the context workspace. The environment variable CHFSI_ZMUL=4 selects 4M at context
 * creation. Errors: CHFSI_ERR_ARG for a null ctx or mults not in {3, 4}. */
chfsi_status chfsi_ctx_set_complex_mult(chfsi_ctx ctx, int32_t mults);

/* The k x k Hermitian eigensolve of Rayleigh-Ritz (Alg 1 lines 7-9; the paper uses EleMRRR,
 * P:969-971). mode 0 (default): the projected matrix G = Q^H H Q of a problem's later loops is nearly
 * diagonal, and a Jacobi-type simultaneous refinement from X = I (every first-order rotation
 * E_ij = (S_ij - lam_j M_ij)/(lam_j - lam_i) at once, S = X^H G X, M = X^H X, iterated to quadratic
 * convergence; k^3 cuBLAS products) replaces the dense solve; it declines -- and the dense cuSOLVER
 * ZHEEVD / DSYEVD runs -- when a coupling exceeds 0.3 of its gap or the iteration stops contracting.
 * mode 1: always the dense solve. Results agree to rounding (eigenvalues to ~1e-15 ||G||); reports count
 * the two paths (eig_refined / eig_dense). CHFSI_EIG=dense selects mode 1 at context creation.
 * Errors: CHFSI_ERR_ARG for a null ctx or a mode not in {0, 1}. */
chfsi_status chfsi_ctx_set_eigensolver(chfsi_ctx ctx, int32_t mode);

/* nranks > 1 only, collective (every rank calls it): how the filter's next-step operand is exchanged
 * (BASELINE.json north_star: Y is rebuilt each degree step across the row panels).
 *  mode 0 (default): in-place allgather per column group on a communication stream, overlapped with the
 *          next group's filter kernel (chfsi_ctx_set_pipeline).
 *  mode 1: peer push. The filter kernel's epilogue stores this rank's rows of every still-active column
 *          straight into every rank's next-step operand buffer through NVLink peer pointers (CUDA IPC
 *          mappings between processes; plain pointers between the ranks of a local group), so the
 *          exchange overlaps the MMAs tile by tile; one small barrier (a one-element NCCL allreduce, or
 *          the local group's event barrier) separates consecutive steps.
 * Mode 1 supports up to 8 ranks (one 8-GPU NVSwitch box) and requires the workspace to be reserved first (chfsi_ctx_reserve with the largest n, nloc and
 * block width to be used); the ranks' buffers are then pinned: a later chfsi_ctx_reserve or filter
 * call needing a larger block returns CHFSI_ERR_ARG. The ranks agree on the outcome: if any rank
 * fails to export or map the IPC handles, every rank returns CHFSI_ERR_CUDA with the exchange left at
 * mode 0 (so a caller can fall back collectively). Errors: CHFSI_ERR_ARG (null ctx, bad mode, no
 * reservation), CHFSI_ERR_CUDA (IPC mapping failed on some rank), CHFSI_ERR_NCCL. No-op at
 * nranks == 1. */
chfsi_status chfsi_ctx_set_exchange(chfsi_ctx ctx, int32_t mode);

/* nranks > 1 only: overlap of the per-step exchange with the filter's MMAs (BASELINE.json north_star
 * "Transfers overlap the next panel's MMA"; SURVEY 8(e) "Overlap"). The active columns of every filter
 * step are cut into G contiguous column groups of >= group_cols columns (G <= 16; group_cols = 0: one
 * group, no overlap); group g's in-place allgather runs on a library-owned communication stream while
 * the filter kernel of group g+1 runs on the ctx stream (CUDA-event ordered, no host synchronisation).
 * The contraction order per output element is unchanged, so results agree with G = 1 to rounding of
 * the stream-K partial sums. sm_reserve SMs are left out of the filter kernel's persistent grid for the
 * collective's thread blocks. Defaults: group_cols = 128, sm_reserve = 0. Errors: CHFSI_ERR_ARG for a
 * null ctx, negative values or sm_reserve >= the SM count. Ignored at nranks == 1. */
chfsi_status chfsi_ctx_set_pipeline(chfsi_ctx ctx, int32_t group_cols, int32_t sm_reserve);

/* Chebyshev filter -- Algorithm 2 with the three-term recurrence of eq:3term
 * (P:764-768), reading R1 (line 8's trailing term is Y_{i-1}), R2 (columns run to k), R3 (active
 * start s = #{j : deg[j] <= i} before step i).
 *   Y_1     = (sigma_1/e) (H - cI) Y_0,                            sigma_1 = e/(lambda1 - c)  (l2-3)
 *   Y_{i+1} = (2 sigma_{i+1}/e)(H - cI) Y_i - sigma_{i+1} sigma_i Y_{i-1},
 *             sigma_{i+1} = 1/(2/sigma_1 - sigma_i)                                     (l6, l8)
 * on the active columns only; column j leaves the recurrence after deg[j] steps (l7, l9), so it
 * equals p_{deg[j]}(H) y_j with p_m(t) = C_m((t-c)/e)/C_m((lambda1-c)/e) (App. A of
 * SURVEY.md).
 *   Hp     device, n x nloc column slab of H (see Conventions), ldh >= n. Read only.
 *   Y      device, nloc x k, ldy >= nloc. In: Y_0 (this rank's rows). Out: the filtered block.
 *   deg    host int32[k], ascending, 1 <= deg[j] <= CHFSI_MAX_DEGREE.
 *   lambda1, c, e: the interval [c-e, c+e] = [alpha, beta] to damp and the scaling point lambda1
 *          (gamma); requires e > 0 and lambda1 < c - e.
 *   matvecs host, nullable: receives sum(deg), the number of column mat-vecs with H (global).
 * Errors: CHFSI_ERR_ARG (dims, ld, unsorted / out-of-range degree, e <= 0, lambda1 >= c - e),
 *         CHFSI_ERR_NONFINITE (non-finite output), CHFSI_ERR_CUDA, CHFSI_ERR_NCCL. */
chfsi_status chfsi_filter(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp,
                          int64_t ldh, void* Y, int64_t ldy, int64_t k, const int32_t* deg,
                          double lambda1, double c, double e, int64_t* matvecs);

/* Real-symmetric variant of chfsi_filter (SPEC supports both fields): the
 * same Alg 2 recurrence on real data -- Hp (n x nloc, double, the rank's column slab of the symmetric H),
 * Y (nloc x k, double) -- with a plain real FP64 DMMA GEMM (2 n nloc k_a flop per step instead of 8).
 * Arguments, layout and errors as chfsi_filter. */
chfsi_status chfsi_filter_real(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const double* Hp,
                               int64_t ldh, double* Y, int64_t ldy, int64_t k, const int32_t* deg,
                               double lambda1, double c, double e, int64_t* matvecs);

/* Lanczos spectral bounds -- Alg 1 line 3, reading R17: `steps` iterations
 * with full reorthogonalisation from the normalised counter-based start vector of DESIGN.md R22
 * (seed, stream (4 << 16) | restart); a breakdown restarts with the next stream, at most 3 times.
 *   theta_min, theta_max (host): extreme eigenvalues of the Lanczos tridiagonal T;
 *   upper_bound (host): theta_max + ||f_steps||, the filter's upper interval end beta.
 * Errors: CHFSI_ERR_ARG (steps < 1), CHFSI_ERR_NOCONV (breakdown after 3 restarts), CUDA/NCCL. */
chfsi_status chfsi_lanczos_bounds(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc,
                                  const void* Hp, int64_t ldh, int32_t steps, uint64_t seed,
                                  double* theta_min, double* theta_max, double* upper_bound);

/* QR -- Alg 1 line 6, reading R14/R15: Y[:, nlocked:k] is orthonormalised
 * against Y[:, 0:nlocked] (left bit-identical) by CGS2, then by CholeskyQR2 (S = Y^H Y = R^H R,
 * Y <- Y R^{-1}, twice). If a Cholesky pivot fails or ||Q^H Q - I||_max > 1e-12 the block is
 * re-orthonormalised by Householder QR instead (*used_fallback = 1). Q has R with real positive
 * diagonal (Y_in = Q R).
 * Rank deficiency (reading R23; the paper's "could easily become linearly dependent",
 * P:598-601): an active column j whose Householder |R_jj| (after the projection against the locked
 * block) is <= 1e-12 times its input norm is replaced by the counter-based vector of R22 with seed
 * `seed + round` and stream (6 << 16) | j (j counted from column 0 of Y), and the block is
 * orthonormalised again (at most 3 rounds); [locked | Q] is then orthonormal.
 *   Y  device, nloc x k, ldy >= nloc, in/out; k <= 65536.  used_fallback, replaced host, nullable.
 * chfsi_qr = chfsi_qr_ex with seed 0 and no replacement count.
 * Errors: CHFSI_ERR_ARG, CHFSI_ERR_QR (still deficient after 3 rounds / Householder failed), CUDA/NCCL. */
chfsi_status chfsi_qr(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, void* Y, int64_t ldy,
                      int64_t k, int64_t nlocked, int32_t* used_fallback);
chfsi_status chfsi_qr_ex(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, void* Y, int64_t ldy,
                         int64_t k, int64_t nlocked, uint64_t seed, int32_t* used_fallback,
                         int32_t* replaced);

/* Rayleigh-Ritz -- Alg 1 lines 7-9: G = Q^H H Q (hermitised), G W = W M,
 * Q <- Q W. Q must have orthonormal columns.
 *   Q     device, nloc x k, ldq >= nloc, in/out (Ritz vectors, ascending Ritz values).
 *   ritz  host double[k], ascending.
 *   resid host double[k], nullable: ||H q_j - mu_j q_j||_2 / normH (R8), computed from (HQ)W
 *         without a second n^2 k product.
 * Errors: CHFSI_ERR_ARG (normH <= 0 with resid != NULL), CUDA/NCCL. */
chfsi_status chfsi_rayleigh_ritz(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc,
                                 const void* Hp, int64_t ldh, void* Q, int64_t ldq, int64_t k,
                                 double normH, double* ritz, double* resid);

/* Reduction of the generalised problem A c = lambda B c to standard form -- P:541-545 ("H = L^{-1} A
 * L^{-T} where B = L L^T", complex Hermitian: L^{-1} A L^{-H}; the FLAPW problems of P:330-347):
 *   B  device n x n (ldb >= n), Hermitian positive definite; out: its Cholesky factor L in the lower
 *      triangle (B = L L^H, real positive diagonal); the strict upper triangle is left unspecified.
 *   A  device n x n (lda >= n), Hermitian; out: H = L^{-1} A L^{-H}, stored full and exactly
 *      Hermitian ((H + H^H)/2, R13) -- the input of chfsi_solve_sequence / chfsi_filter.
 * Single rank only (nranks == 1). Errors: CHFSI_ERR_ARG (dims, nranks > 1, B not positive definite:
 * the failing pivot is named in chfsi_last_error), CHFSI_ERR_CUDA. */
chfsi_status chfsi_reduce_generalized(chfsi_ctx ctx, int64_t n, void* A, int64_t lda, void* B,
                                      int64_t ldb);
/* Back-transformation of eigenvectors of H to generalised eigenvectors: X <- L^{-H} X (c = L^{-H} y),
 * L from chfsi_reduce_generalized (lower triangle of the returned B). X device n x k (ldx >= n). The
 * result is B-orthonormal when X is orthonormal. Single rank only. */
chfsi_status chfsi_back_transform(chfsi_ctx ctx, int64_t n, const void* L, int64_t ldl, void* X,
                                  int64_t ldx, int64_t k);
/* Row-panel form of chfsi_reduce_generalized for any nranks >= 1 (collective: every rank
 * calls it with its own panel; nloc * nranks == n, row0 == rank * nloc, as for chfsi_filter).
 * Ap (in/out, device n x nloc, lda >= n): in, the column slab A[:, row0:row0+nloc]; out, the slab
 * Hp = H[:, row0:row0+nloc] of H = L^{-1} A L^{-H}, ready for chfsi_filter / chfsi_solve_sequence with
 * the same (n, row0, nloc). The assembled H is Hermitian bit for bit across the ranks (R13).
 * Bp (in, device n x nloc, ldb >= n): the column slab B[:, row0:row0+nloc] of the Hermitian positive
 * definite B; not modified. L (out, device n x n, ldl >= n, caller-owned): the full Cholesky factor
 * B = L L^H in its lower triangle (identical bits on every rank; the strict upper triangle is
 * unspecified), for chfsi_back_transform_panel.
 * Work: B = L L^H factored on the ranks' column slabs (right-looking panels of <= 256 columns: the
 * panel's owner runs ZPOTRF + ZTRSM, the panel is broadcast, every rank updates its own trailing
 * columns with ZGEMM; p = 1: one ZPOTRF), L and A gathered on every rank (16 n^2 bytes of scratch),
 * then 2 ZTRSM + 1 ZGEMM with nloc right-hand sides per rank. Errors: CHFSI_ERR_ARG (dims / panel,
 * B not positive definite -- returned by every rank, the first failing pivot in chfsi_last_error),
 * CHFSI_ERR_CUDA, CHFSI_ERR_NCCL, CHFSI_ERR_NOMEM. */
chfsi_status chfsi_reduce_generalized_panel(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, void* Ap,
                                            int64_t lda, const void* Bp, int64_t ldb, void* L, int64_t ldl);
/* Row-panel back-transformation, collective: X (in/out, device nloc x k, ldx >= nloc) holds this
 * rank's rows of eigenvectors y of H; on return its rows of c = L^{-H} y. L as returned by
 * chfsi_reduce_generalized_panel (any rank's copy). The k columns are gathered on every rank and solved
 * whole (n^2 k per rank, about one filter step). k <= n. Errors: CHFSI_ERR_ARG, CHFSI_ERR_CUDA,
 * CHFSI_ERR_NCCL, CHFSI_ERR_NOMEM. */
chfsi_status chfsi_back_transform_panel(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* L,
                                        int64_t ldl, void* X, int64_t ldx, int64_t k);

typedef struct {
  int32_t nev, nex;      /* wanted eigenpairs and extra buffer columns, k = nev + nex <= n; nex >= 1
                            (the filter interval starts at the largest of the k current values, R4) */
  int32_t deg0;          /* starting degree of each problem's first loop (R12; default 8) */
  int32_t deg_cap;       /* degree cap (default 40), <= CHFSI_MAX_DEGREE */
  int32_t max_loops;     /* default 50 */
  int32_t lanczos_steps; /* default 25 (R17) */
  double tol;            /* residual tolerance, relative to ||H||_est (R8), e.g. 1e-10 */
  uint64_t seed;         /* Lanczos start-vector seed; problem ell uses seed + ell */
  int32_t random_start;  /* 1: ignore X on input and draw a counter-based start block (R22) */
  /* ablations: */
  int32_t no_reuse;      /* 1: every problem starts from its own random block (R22, seed + ell) instead
                            of the previous problem's eigenvectors -- Fig 2b's "random vectors" arm */
  int32_t fixed_degree;  /* > 0: every vector is filtered with this degree in every loop (no Single
                            Optimisation) -- Fig 5's "-OPT" arm; 0: optimised degrees */
} chfsi_opts;

typedef struct {
  int32_t loops, qr_fallbacks, capped, converged;
  int64_t matvecs_filter, matvecs_total;
  double filter_flops; /* algorithmic: 8 n^2 sum(deg) over all filter calls */
  double t_lanczos, t_filter, t_qr, t_rr, t_resid, t_opt, t_total; /* seconds, CUDA events */
  double theta_min, theta_max, beta_up, normH;
  double t_filter_kernel; /* seconds inside K1 launches of the filter (CUDA events per launch) */
  int64_t filter_launches; /* K1 launches of the filter */
  int32_t qr_replaced;     /* columns replaced by the QR rank-deficiency rule (R23) */
  int32_t reseeded;        /* 1: the previous problem's (lambda_1, lambda_k) did not fit this problem's
                              Lanczos bound (beta <= alpha): re-seeded from QR + Rayleigh-Ritz (R11) */
  int32_t eig_refined;     /* loops whose k x k eigensolve ran as the Jacobi-type refinement */
  int32_t eig_dense;       /* loops whose k x k eigensolve ran as a dense ZHEEVD */
  double t_eig;            /* seconds in the k x k eigensolves (CUDA events) */
} chfsi_report;

/* Callback giving problem ell's column slab (device pointer and its leading dimension). */
typedef chfsi_status (*chfsi_get_h)(void* user, int32_t ell, const void** Hp, int64_t* ldh);

/* ChFSI on a sequence -- Algorithm 1 for ell = 0..nprob-1, the eigenvectors and
 * (lambda_1, lambda_k) of problem ell seeding problem ell+1 (Def 1).
 *   X       device, nloc x (nev+nex), ldx >= nloc. In: the start basis of problem 0 (unless
 *           opts.random_start). Out: the final block of the last problem; its first nev columns are
 *           the eigenvectors, ascending.
 *   lambda  host double[nprob * nev]: eigenvalues of problem ell at lambda[ell*nev + i], ascending.
 *   resid   host double[nprob * nev], nullable: their residuals (R8).
 *   reports host chfsi_report[nprob], nullable.
 * Errors: CHFSI_ERR_ARG, CHFSI_ERR_NOCONV (a problem hit max_loops; the sequence continues and the
 *         partial results are returned), CHFSI_ERR_QR, CUDA/NCCL. */
chfsi_status chfsi_solve_sequence(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc,
                                  int32_t nprob, chfsi_get_h get_h, void* user,
                                  const chfsi_opts* opts, void* X, int64_t ldx, double* lambda,
                                  double* resid, chfsi_report* reports);

/* Real-symmetric ChFSI on a sequence: chfsi_solve_sequence for real
 * symmetric H (double, get_h returns the real column slab) and a real block X (double). Same options,
 * outputs and errors; the filter runs chfsi_filter_real's kernel, the supporting steps their real
 * (DGEMM / DPOTRF / DSYEVD / DGEQRF) counterparts; report filter_flops counts 2 n^2 sum(deg). */
chfsi_status chfsi_solve_sequence_real(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc,
                                       int32_t nprob, chfsi_get_h get_h, void* user,
                                       const chfsi_opts* opts, double* X, int64_t ldx, double* lambda,
                                       double* resid, chfsi_report* reports);

/* Independent sequences: the N_k k-point sequences of one SCF cycle are
 * independent eigenproblem sequences. chfsi_solve_batch solves `count` of them
 * concurrently on one device with `workers` library contexts, each on its own CUDA stream and host
 * thread, taking sequences in order. Each sequence is described as for chfsi_solve_sequence (single
 * rank: row0 = 0, nloc = n); its status is returned in `status`. The call returns the worst status. */
typedef struct {
  int32_t nprob;
  chfsi_get_h get_h;
  void* user;
  void* X;          /* device n x (nev+nex) */
  int64_t ldx;
  double* lambda;   /* host nprob * nev */
  double* resid;    /* host nprob * nev, nullable */
  chfsi_report* reports; /* host [nprob], nullable */
  chfsi_status status;   /* out */
} chfsi_sequence;
chfsi_status chfsi_solve_batch(int32_t device, int32_t workers, int64_t n, const chfsi_opts* opts,
                               chfsi_sequence* seqs, int32_t count);

#ifdef __cplusplus
}
#endif
#endif
