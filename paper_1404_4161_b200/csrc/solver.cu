// solver.cu -- ChFSI for one eigenproblem and for a correlated sequence (Alg 1; Def 1,
// P:75-81), with the readings R4-R12, R16, R21. Host driver: every O(n^2 k) and
// O(n k^2) step runs on the device (filter K1, H Q K1, CholQR2, Rayleigh-Ritz, residuals); the
// host only keeps O(k) bookkeeping (Ritz values, residuals, degrees, lock decisions).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <numeric>
#include <thread>
#include <type_traits>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "ctx.cuh"
#include "small_kernels.cuh"
#include "supporting.cuh"

namespace chfsi {

#define TRY(x)                       \
  do {                               \
    chfsi_status _st = (x);          \
    if (_st != CHFSI_OK) return _st; \
  } while (0)

namespace {

// CUDA-event phase timer: intervals are accumulated when the stream is already synchronised.
struct PhaseTimer {
  std::vector<cudaEvent_t> pool;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  size_t used = 0;
  cudaStream_t st;
  double acc[8] = {0};
  explicit PhaseTimer(cudaStream_t s) : st(s) {}
  ~PhaseTimer() {
    for (; nvtx_depth > 0; --nvtx_depth) nvtxRangePop();  // ranges left open by an error return
    for (auto e : pool) cudaEventDestroy(e);
  }
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
  // NVTX range per phase (header-only NVTX3: free unless a profiler is attached)
  int nvtx_depth = 0;
  std::pair<cudaEvent_t, cudaEvent_t> begin(const char* name) {
    nvtxRangePushA(name);
    ++nvtx_depth;
    cudaEvent_t a = ev(), b = ev();
    cudaEventRecord(a, st);
    return {a, b};
  }
  void end(int phase, std::pair<cudaEvent_t, cudaEvent_t> p) {
    cudaEventRecord(p.second, st);
    pending.push_back({phase, p});
    nvtxRangePop();
    --nvtx_depth;
  }
  void flush() {  // call after a stream synchronisation
    for (auto& q : pending) {
      cudaEventSynchronize(q.second.second);
      float ms = 0;
      cudaEventElapsedTime(&ms, q.second.first, q.second.second);
      acc[q.first] += ms * 1e-3;
    }
    pending.clear();
    used = 0;
  }
};
enum { T_LANCZOS = 0, T_FILTER, T_QR, T_RR, T_RESID, T_OPT, T_TOTAL };

}  // namespace

// One eigenproblem. X (nloc x k) in: start block / hand-off; out: hand-off [locked asc | active].
// E: double2 (complex Hermitian, scalar cuDoubleComplex) or double (real symmetric, NEXT-3)
template <typename E>
static chfsi_status solve_one(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                              const chfsi_opts& o, E* X, int64_t ldx, bool have_prev, double& lam1_io,
                              double& lamk_io, double* lam_out, double* res_out, chfsi_report& rep, uint64_t seed) {
  const int64_t nev = o.nev, k = (int64_t)o.nev + o.nex;
  rep = chfsi_report{};
  const int64_t eig_r0 = ctx->eig_refined, eig_d0 = ctx->eig_dense;
  const double eig_t0 = ctx->eig_seconds;
  PhaseTimer tm(ctx->stream);
  auto t_all = tm.begin("chfsi: eigenproblem");
  const size_t blk = sizeof(double) * 2 * (size_t)nloc * k;
  TRY(ensure(ctx, ctx->ya, blk));
  TRY(ensure(ctx, ctx->xl, blk));
  TRY(ensure(ctx, ctx->tb, blk));
  TRY(ensure(ctx, ctx->idx, sizeof(int) * (size_t)k));
  using Scal = typename std::conditional<std::is_same<E, double>::value, double, cuDoubleComplex>::type;
  constexpr int elem = sizeof(E) / sizeof(double);
  constexpr size_t eb = sizeof(E);
  E* Ya = static_cast<E*>(ctx->ya.ptr);
  E* XL = static_cast<E*>(ctx->xl.ptr);
  E* T = static_cast<E*>(ctx->tb.ptr);
  int* didx = static_cast<int*>(ctx->idx.ptr);
  std::vector<int> hidx(k);
  auto gather = [&](const E* src, const std::vector<int>& cols, E* dst, int64_t ldd) -> chfsi_status {
    if (cols.empty()) return CHFSI_OK;
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(didx, cols.data(), sizeof(int) * cols.size(), cudaMemcpyHostToDevice,
                                        ctx->stream));
    CHFSI_CUDA_TRY(ctx, launch_col_gather(nloc, (int64_t)cols.size(), src, nloc, didx, dst, ldd, ctx->stream));
    ctx->launches++;
    return CHFSI_OK;
  };

  // 3M filter / H Q: the Re H - Im H plane of this problem's panel, built once and reused by every
  // filter step and Rayleigh-Ritz product of the problem (unpinned on every exit path)
  struct PinGuard {
    chfsi_ctx c;
    ~PinGuard() { c->h3_pin = nullptr; }
  } pin_guard{ctx};
  if (elem == 2 && ctx->zmul == 3) {
    TRY(h3_prepare(ctx, Hp, ldh, n, nloc));
    ctx->h3_pin = Hp;
  }

  // Alg 1 l3: Lanczos upper bound beta (R17) and ||H||_est (R8)
  double tmin, tmax, beta;
  auto t0 = tm.begin("chfsi: lanczos");
  TRY(lanczos_t<Scal>(ctx, n, row0, nloc, Hp, ldh, o.lanczos_steps, seed, &tmin, &tmax, &beta));
  tm.end(T_LANCZOS, t0);
  const double normH = std::max(std::fabs(tmin), std::fabs(tmax));
  rep.theta_min = tmin;
  rep.theta_max = tmax;
  rep.beta_up = beta;
  rep.normH = normH;
  rep.matvecs_total += o.lanczos_steps;

  CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(Ya, eb * nloc, X, eb * ldx, eb * nloc, k, cudaMemcpyDeviceToDevice, ctx->stream));
  std::vector<double> mu(k), res(k), lamL, resL;
  double lam1 = lam1_io, alpha = lamk_io;
  // the previous problem's (lambda_1, lambda_k) seed this one unless they do not fit under
  // this problem's upper bound (beta <= alpha: the filter interval would be empty); then, as for a
  // first problem (R11), the start block is orthonormalised and its Ritz values seed (lambda_1, alpha)
  if (have_prev && !(beta > alpha && lam1 < alpha)) {
    have_prev = false;
    rep.reseeded = 1;
  }
  if (!have_prev) {  // R11: start block -> QR -> RR seeds (lambda_1, alpha)
    int32_t fb = 0, nrep = 0;
    auto t1 = tm.begin("chfsi: qr (start)");
    TRY(qr_t<Scal>(ctx, n, row0, nloc, nullptr, nloc, 0, Ya, nloc, k, seed, &fb, &nrep));
    tm.end(T_QR, t1);
    rep.qr_fallbacks += fb;
    rep.qr_replaced += nrep;
    auto t2 = tm.begin("chfsi: rayleigh-ritz (start)");
    TRY(rr_t<Scal>(ctx, n, row0, nloc, Hp, ldh, Ya, nloc, k, normH, mu.data(), nullptr));
    tm.end(T_RR, t2);
    rep.matvecs_total += k;
    lam1 = mu[0];
    alpha = mu[k - 1];
  }
  std::vector<int32_t> m(k, o.fixed_degree > 0 ? o.fixed_degree : o.deg0), ms(k);
  int64_t nl = 0;
  chfsi_status status = CHFSI_ERR_NOCONV;
  while (rep.loops < o.max_loops) {
    const int64_t ka = k - nl;
    const double c = 0.5 * (alpha + beta), e = 0.5 * (beta - alpha);
    // the damped interval [alpha, beta] must be non-empty (Alg 2): Ritz values stay below the
    // Lanczos bound beta in exact arithmetic, so this only trips on a broken input (lambda_1 = alpha, e.g. a
    // k-fold degenerate spectrum, is fine: sigma_1 = -1)
    if (!(e > 0.0) || !std::isfinite(c) || !(lam1 <= alpha)) {
      set_err(ctx, "ChFSI: filter interval collapsed (lambda_1 = " + std::to_string(lam1) + ", alpha = " +
                       std::to_string(alpha) + ", beta = " + std::to_string(beta) + ")");
      status = CHFSI_ERR_NOCONV;
      break;
    }
    // R6: stable ascending sort of the active columns by degree
    std::vector<int> perm(ka);
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return m[a] < m[b]; });
    for (int64_t j = 0; j < ka; ++j) ms[j] = m[perm[j]];
    TRY(gather(Ya, perm, T, nloc));
    // Alg 1 l5: the Chebyshev filter (Alg 2)
    auto t3 = tm.begin("chfsi: filter");
    const double k1s = ctx->k1_seconds;
    const int64_t k1n = ctx->k1_launches;
    TRY(filter_impl(ctx, n, row0, nloc, Hp, ldh, T, nloc, ka, ms.data(), lam1, c, e, true, elem));
    tm.end(T_FILTER, t3);
    rep.t_filter_kernel += ctx->k1_seconds - k1s;
    rep.filter_launches += ctx->k1_launches - k1n;
    int64_t mv = 0;
    for (int64_t j = 0; j < ka; ++j) mv += ms[j];
    rep.matvecs_filter += mv;
    rep.matvecs_total += mv;
    rep.filter_flops += (elem == 2 ? 8.0 : 2.0) * (double)n * (double)n * (double)mv;
    // Alg 1 l6: orthonormalise [locked | filtered] (R14, R15, R23)
    int32_t fb = 0, nrep = 0;
    auto t4 = tm.begin("chfsi: qr");
    TRY(qr_t<Scal>(ctx, n, row0, nloc, XL, nloc, nl, T, nloc, ka, seed, &fb, &nrep));
    tm.end(T_QR, t4);
    rep.qr_fallbacks += fb;
    rep.qr_replaced += nrep;
    // Alg 1 l7-9 (+ residuals, R8): Rayleigh-Ritz on the active block (R16)
    auto t5 = tm.begin("chfsi: rayleigh-ritz");
    TRY(rr_t<Scal>(ctx, n, row0, nloc, Hp, ldh, T, nloc, ka, normH, mu.data(), res.data()));
    tm.end(T_RR, t5);
    rep.matvecs_total += ka;
    rep.loops++;
    // Alg 1 l10 (R7): lock wanted Ritz positions with r <= tol, leftmost in locking order
    auto t6 = tm.begin("chfsi: lock + degrees");
    const int64_t want = nev - nl;
    std::vector<int> lock_cols, keep_cols;
    std::vector<double> mu2, res2;
    for (int64_t j = 0; j < ka; ++j) {
      if (j < want && res[j] <= o.tol) {
        lock_cols.push_back((int)j);
        lamL.push_back(mu[j]);
        resL.push_back(res[j]);
      } else {
        keep_cols.push_back((int)j);
        mu2.push_back(mu[j]);
        res2.push_back(res[j]);
      }
    }
    TRY(gather(T, lock_cols, XL + (size_t)nl * nloc, nloc));
    TRY(gather(T, keep_cols, Ya, nloc));
    nl += (int64_t)lock_cols.size();
    const int64_t na = ka - (int64_t)lock_cols.size();
    // R4: the interval from the current k values (locked + active Ritz)
    double vmin = HUGE_VAL, vmax = -HUGE_VAL;
    for (double v : mu2) vmin = std::min(vmin, v), vmax = std::max(vmax, v);
    for (double v : lamL) vmin = std::min(vmin, v), vmax = std::max(vmax, v);
    lam1 = vmin;
    alpha = vmax;
    for (int64_t j = 0; j < na; ++j) {
      mu[j] = mu2[j];
      res[j] = res2[j];
    }
    if (nl >= nev) {
      status = CHFSI_OK;
      tm.end(T_OPT, t6);
      break;
    }
    // Alg 1 l11 (R21, R5, R9): degrees for the next filter
    if (o.fixed_degree > 0) {  // ablation: no Single Optimisation
      for (int64_t j = 0; j < na; ++j) m[j] = o.fixed_degree;
      tm.end(T_OPT, t6);
      continue;
    }
    const double c2 = 0.5 * (alpha + beta), e2 = 0.5 * (beta - alpha);
    const int64_t want2 = nev - nl;
    int32_t mmax = 1;
    for (int64_t j = 0; j < na && j < want2; ++j) {
      const double t = std::fabs((mu[j] - c2) / e2);
      int32_t d;
      if (t <= 1.0) {
        d = o.deg_cap;
      } else {
        const double ratio = std::max(res[j] / o.tol, 1.0);
        double dm = std::ceil(std::acosh(ratio) / std::acosh(t));
        if (!(dm >= 1.0)) dm = 1.0;
        d = dm > (double)o.deg_cap ? o.deg_cap : (int32_t)dm;
      }
      if (d == o.deg_cap) rep.capped++;
      m[j] = d;
      mmax = std::max(mmax, d);
    }
    for (int64_t j = want2; j < na; ++j) m[j] = mmax;
    tm.end(T_OPT, t6);
  }
  rep.converged = (int32_t)nl;
  // output: locked sorted ascending (stable), then the remaining active columns
  std::vector<int> ord(nl);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return lamL[a] < lamL[b]; });
  if (nl > 0) {
    TRY(gather(XL, ord, T, nloc));
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(X, eb * ldx, T, eb * nloc, eb * nloc, nl, cudaMemcpyDeviceToDevice,
                                          ctx->stream));
  }
  if (k - nl > 0)
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(X + (size_t)nl * ldx, eb * ldx, Ya, eb * nloc, eb * nloc, k - nl,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
  for (int64_t j = 0; j < nev; ++j) {
    if (j < nl) {
      lam_out[j] = lamL[ord[j]];
      if (res_out) res_out[j] = resL[ord[j]];
    } else {  // partial results of a problem that hit max_loops
      lam_out[j] = mu[j - nl];
      if (res_out) res_out[j] = res[j - nl];
    }
  }
  lam1_io = lam1;
  lamk_io = alpha;
  tm.end(T_TOTAL, t_all);
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  tm.flush();
  rep.t_lanczos = tm.acc[T_LANCZOS];
  rep.t_filter = tm.acc[T_FILTER];
  rep.t_qr = tm.acc[T_QR];
  rep.t_rr = tm.acc[T_RR];
  rep.t_opt = tm.acc[T_OPT];
  rep.t_total = tm.acc[T_TOTAL];
  rep.eig_refined = (int32_t)(ctx->eig_refined - eig_r0);
  rep.eig_dense = (int32_t)(ctx->eig_dense - eig_d0);
  rep.t_eig = ctx->eig_seconds - eig_t0;
  if (status == CHFSI_ERR_NOCONV && ctx->err.empty())
    set_err(ctx, "ChFSI: max_loops reached before nev eigenpairs converged");
  return status;
}

}  // namespace chfsi

using namespace chfsi;

template <typename E>
static chfsi_status solve_sequence_t(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, int32_t nprob,
                                     chfsi_get_h get_h, void* user, const chfsi_opts* opts, void* X, int64_t ldx,
                                     double* lambda, double* resid, chfsi_report* reports) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (!opts || !get_h || !X || !lambda || nprob < 0 || n < 1 || nloc < 1 || row0 < 0 || row0 + nloc > n ||
      ldx < nloc) {
    set_err(ctx, "chfsi_solve_sequence: bad arguments");
    return CHFSI_ERR_ARG;
  }
  const chfsi_opts& o = *opts;
  const int64_t k = (int64_t)o.nev + o.nex;
  // nex >= 1: the filter interval starts at the largest of the k current values (R4), so without a
  // buffer vector it would start at the last wanted Ritz value and never separate it from the unwanted
  if (o.nev < 1 || o.nex < 1 || k > n || !(o.tol > 0) || o.deg0 < 1 || o.deg0 > o.deg_cap ||
      o.deg_cap > CHFSI_MAX_DEGREE || o.max_loops < 1 || o.lanczos_steps < 1 || o.fixed_degree < 0 ||
      o.fixed_degree > CHFSI_MAX_DEGREE ||
      (nloc * ctx->nranks != n || row0 != nloc * ctx->rank)) {
    set_err(ctx, "chfsi_solve_sequence: bad options (need nev >= 1, nex >= 1, nev + nex <= n, tol > 0, "
                 "1 <= deg0 <= cap <= 64)");
    return CHFSI_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  E* Xd = static_cast<E*>(X);
  if (o.random_start) {  // R22 block: column j uses stream (3 << 16) | j
    CHFSI_CUDA_TRY(ctx, launch_random_block(nloc, k, row0, o.seed, 3ull << 16, 1, Xd, ldx, ctx->stream));
    ctx->launches++;
  }
  chfsi_status worst = CHFSI_OK;
  double lam1 = 0, lamk = 0;
  for (int32_t ell = 0; ell < nprob; ++ell) {
    const void* Hp = nullptr;
    int64_t ldh = 0;
    if (get_h(user, ell, &Hp, &ldh) != CHFSI_OK || !Hp || ldh < n) {
      set_err(ctx, "chfsi_solve_sequence: get_h failed for problem " + std::to_string(ell));
      return CHFSI_ERR_ARG;
    }
    if (o.no_reuse && ell > 0) {  // ablation: a fresh random block instead of the hand-off
      CHFSI_CUDA_TRY(ctx, launch_random_block(nloc, k, row0, o.seed + (uint64_t)ell, 3ull << 16, 1, Xd, ldx,
                                              ctx->stream));
      ctx->launches++;
    }
    chfsi_report rep{};
    chfsi_status st = solve_one<E>(ctx, n, row0, nloc, Hp, ldh, o, Xd, ldx, ell > 0 && !o.no_reuse, lam1, lamk,
                                lambda + (size_t)ell * o.nev, resid ? resid + (size_t)ell * o.nev : nullptr, rep,
                                o.seed + (uint64_t)ell);
    if (reports) reports[ell] = rep;
    if (st == CHFSI_ERR_NOCONV) {
      worst = CHFSI_ERR_NOCONV;  // the sequence continues with the partial results
      continue;
    }
    if (st != CHFSI_OK) return st;
  }
  if (worst == CHFSI_ERR_NOCONV) set_err(ctx, "ChFSI: at least one problem hit max_loops");
  return worst;
}

extern "C" chfsi_status chfsi_solve_sequence(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, int32_t nprob,
                                             chfsi_get_h get_h, void* user, const chfsi_opts* opts, void* X,
                                             int64_t ldx, double* lambda, double* resid, chfsi_report* reports) {
  return solve_sequence_t<double2>(ctx, n, row0, nloc, nprob, get_h, user, opts, X, ldx, lambda, resid, reports);
}

extern "C" chfsi_status chfsi_solve_sequence_real(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc,
                                                  int32_t nprob, chfsi_get_h get_h, void* user,
                                                  const chfsi_opts* opts, double* X, int64_t ldx, double* lambda,
                                                  double* resid, chfsi_report* reports) {
  return solve_sequence_t<double>(ctx, n, row0, nloc, nprob, get_h, user, opts, X, ldx, lambda, resid, reports);
}

extern "C" chfsi_status chfsi_solve_batch(int32_t device, int32_t workers, int64_t n, const chfsi_opts* opts,
                                          chfsi_sequence* seqs, int32_t count) {
  if (!opts || !seqs || count < 0 || workers < 1 || n < 1) return CHFSI_ERR_ARG;
  if (count == 0) return CHFSI_OK;
  workers = std::min(workers, count);
  std::vector<chfsi_ctx> ctxs(workers, nullptr);
  std::vector<cudaStream_t> streams(workers, nullptr);
  chfsi_status st = CHFSI_OK;
  if (cudaSetDevice(device) != cudaSuccess) return CHFSI_ERR_CUDA;
  for (int w = 0; w < workers && !st; ++w) {
    if (cudaStreamCreateWithFlags(&streams[w], cudaStreamNonBlocking) != cudaSuccess) st = CHFSI_ERR_CUDA;
    if (!st) st = chfsi_ctx_create(&ctxs[w], device, streams[w], nullptr, 0, 1);
  }
  if (!st) {
    std::atomic<int> next{0};
    std::vector<std::thread> th;
    for (int w = 0; w < workers; ++w)
      th.emplace_back([&, w] {
        cudaSetDevice(device);
        for (int s = next++; s < count; s = next++) {
          chfsi_sequence& q = seqs[s];
          q.status = chfsi_solve_sequence(ctxs[w], n, 0, n, q.nprob, q.get_h, q.user, opts, q.X, q.ldx, q.lambda,
                                          q.resid, q.reports);
        }
      });
    for (auto& t : th) t.join();
    for (int s = 0; s < count; ++s)
      if (seqs[s].status != CHFSI_OK && (st == CHFSI_OK || st == CHFSI_ERR_NOCONV)) st = seqs[s].status;
  }
  for (int w = 0; w < workers; ++w) {
    if (ctxs[w]) chfsi_ctx_destroy(ctxs[w]);
    if (streams[w]) cudaStreamDestroy(streams[w]);
  }
  return st;
}
