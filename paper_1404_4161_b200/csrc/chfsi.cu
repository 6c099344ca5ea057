// chfsi.cu -- context management, TMA descriptor encoding, and the Chebyshev filter driver
// (chfsi_filter: Alg 2) plus H*Q for Rayleigh-Ritz, both on the K1 kernel.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "ctx.cuh"
#include "filter_step.cuh"
#include "small_kernels.cuh"

namespace chfsi {

void set_err(chfsi_ctx ctx, const std::string& msg) {
  if (ctx) ctx->err = msg;
}

chfsi_status ensure(chfsi_ctx ctx, DevBuf& b, size_t bytes) {
  if (b.bytes >= bytes) return CHFSI_OK;
  if (b.ptr) {
    cudaStreamSynchronize(ctx->stream);
    cudaFree(b.ptr);
    b.ptr = nullptr;
    b.bytes = 0;
  }
  bytes = std::max<size_t>(bytes, 256);
  if (cudaMalloc(&b.ptr, bytes) != cudaSuccess) {
    cudaGetLastError();
    set_err(ctx, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    return CHFSI_ERR_NOMEM;
  }
  b.bytes = bytes;
  return CHFSI_OK;
}

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

chfsi_status make_tmap_2d(chfsi_ctx ctx, CUtensorMap* m, const void* base, int64_t kreal, int64_t rows,
                          int64_t ld_doubles, int box_rows, int box_inner) {
  auto enc = get_encode();
  if (!enc) {
    set_err(ctx, "cuTensorMapEncodeTiled unavailable");
    return CHFSI_ERR_CUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kreal, (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(ld_doubles * 8)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = box_inner * 8 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_err(ctx, "cuTensorMapEncodeTiled(2d) failed: " + std::to_string((int)r));
    return CHFSI_ERR_CUDA;
  }
  return CHFSI_OK;
}

chfsi_status make_tmap_3d(chfsi_ctx ctx, CUtensorMap* m, const void* base, int64_t kreal, int64_t cols,
                          int64_t chunks, int64_t ld_doubles, int64_t chunk_doubles, int box_cols, int box_inner) {
  auto enc = get_encode();
  if (!enc) {
    set_err(ctx, "cuTensorMapEncodeTiled unavailable");
    return CHFSI_ERR_CUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)kreal, (cuuint64_t)std::max<int64_t>(cols, 1),
                        (cuuint64_t)std::max<int64_t>(chunks, 1)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld_doubles * 8), (cuuint64_t)(std::max<int64_t>(chunk_doubles, ld_doubles) * 8)};
  cuuint32_t box[3] = {(cuuint32_t)box_inner, (cuuint32_t)box_cols, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapSwizzle sw = box_inner * 8 == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_err(ctx, "cuTensorMapEncodeTiled(3d) failed: " + std::to_string((int)r));
    return CHFSI_ERR_CUDA;
  }
  return CHFSI_OK;
}

static inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }


chfsi_status sk_workspace(chfsi_ctx ctx, const TileChoice& t, StepParams& p) {
  const size_t tick_bytes = sizeof(int) * kMaxTailTickets;  // >= tail tiles x cluster ranks (schedule_filter_step)
  const size_t need = tick_bytes + sizeof(double) * filter_partials_doubles(t, ctx->num_sms);
  void* old = ctx->sk.ptr;
  chfsi_status st = ensure(ctx, ctx->sk, need);
  if (st) return st;
  if (ctx->sk.ptr != old) CHFSI_CUDA_TRY(ctx, cudaMemsetAsync(ctx->sk.ptr, 0, tick_bytes, ctx->stream));
  p.tickets = static_cast<int*>(ctx->sk.ptr);
  p.partials = reinterpret_cast<double*>(static_cast<char*>(ctx->sk.ptr) + tick_bytes);
  return CHFSI_OK;
}

// The B operand of one K1 launch: its TMA map, the 3M plane's map, and the column coordinate of the
// first active column.
struct Operand {
  CUtensorMap tm, tm3;
  int32_t b_col0;
};

// Build the B-operand descriptors for one launch over columns [col0, kcols) of `buf`.
//  Column slots hold `rows` elements at a column stride of cs = cw * ld doubles, cw = elem (plain
//  layout) or 3 (3M layout: 2 * ld complex doubles, then the y_r + y_i plane at offset 2 * ld).
//  z3: the launch runs the 3M kernel and also needs the plane's map (a 4M launch on a 3M-layout
//  buffer just skips the planes).
//  p == 1: buf = local state (rows = n), column coordinate = absolute column.
//  p > 1 : buf = packed [rank][kcols - col0][cs] operand (rows = nloc), coordinate = column - col0.
static chfsi_status b_operand(chfsi_ctx ctx, Operand* op, const double* buf, int64_t rows, int64_t ld,
                              int64_t kcols, int64_t col0, int nranks, int box_cols, int elem, int cw, bool z3,
                              int kh = 2) {
  const int64_t cs = cw * ld;
  const int64_t cols = nranks == 1 ? kcols : kcols - col0;
  op->b_col0 = nranks == 1 ? (int32_t)col0 : 0;
  chfsi_status st = make_tmap_3d(ctx, &op->tm, buf, elem * rows, cols, nranks, cs, cs * cols, box_cols);
  if (st || !z3) {
    op->tm3 = op->tm;  // unused outside 3M
    return st;
  }
  return make_tmap_3d(ctx, &op->tm3, buf + 2 * ld, rows, cols, nranks, cs, cs * cols, box_cols, 8 * kh);
}

// The A operand (H panel) through TMA: every box must start on a 16-byte boundary. Complex data always
// does (16-byte elements). Real data is re-strided into a workspace when the panel's leading dimension
// is odd, or when p > 1 and nloc is odd (rank chunk q of the contraction starts at row q nloc): there
// each rank chunk is padded to an even length with zero rows. *kchunk = the K offset (elements) between
// rank chunks, *klen = the K extent of the operand.
static chfsi_status a_operand(chfsi_ctx ctx, const void** Hp, int64_t* ldh, int64_t n, int64_t nloc, int elem,
                              int64_t* kchunk, int64_t* klen) {
  const int p = ctx->nranks;
  *kchunk = nloc;
  *klen = n;
  const bool odd_ld = (elem * *ldh * 8) % 16 != 0;
  const bool odd_chunks = elem == 1 && p > 1 && (nloc % 2) != 0;
  if (!odd_ld && !odd_chunks) return CHFSI_OK;
  const int64_t ldk = odd_chunks ? round_up(nloc, 2) : nloc;
  const int64_t len = odd_chunks ? p * ldk : n;
  const int64_t ld2 = round_up(len, 2);
  chfsi_status st = ensure(ctx, ctx->hpad, sizeof(double) * elem * (size_t)ld2 * nloc);
  if (st) return st;
  double* dst = static_cast<double*>(ctx->hpad.ptr);
  const char* src = static_cast<const char*>(*Hp);
  if (odd_chunks) {
    CHFSI_CUDA_TRY(ctx, cudaMemsetAsync(dst, 0, sizeof(double) * elem * (size_t)ld2 * nloc, ctx->stream));
    for (int q = 0; q < p; ++q)
      CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(dst + (size_t)elem * q * ldk, 8 * elem * ld2, src + 8 * elem * q * nloc,
                                            8 * elem * *ldh, 8 * elem * nloc, nloc, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
  } else {
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(dst, 8 * elem * ld2, src, 8 * elem * *ldh, 8 * elem * n, nloc,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
  }
  *Hp = dst;
  *ldh = ld2;
  *kchunk = ldk;
  *klen = len;
  return CHFSI_OK;
}

// 3M: the plane Re H - Im H of the panel (nloc rows x n, row stride ld3), rebuilt unless the solver
// pinned it for this panel (ctx->h3_pin == Hp for the duration of one eigenproblem).
chfsi_status h3_prepare(chfsi_ctx ctx, const void* Hp, int64_t ldh, int64_t n, int64_t nloc) {
  // K layout of the plane: one rank -> n entries; p ranks -> p chunks of nloc entries, each padded to an
  // even count (TMA boxes of the plane start on 16-byte boundaries for every rank chunk)
  const int p = ctx->nranks;
  const int64_t chunk = p > 1 ? nloc : n, ldk = p > 1 ? round_up(nloc, 2) : n;
  const int64_t klen = p > 1 ? p * ldk : n;
  const int64_t ld3 = round_up(klen, 2);
  chfsi_status st = ensure(ctx, ctx->h3, sizeof(double) * (size_t)ld3 * nloc);
  if (st) return st;
  CHFSI_CUDA_TRY(ctx, launch_h3_plane(n, nloc, static_cast<const double2*>(Hp), ldh, static_cast<double*>(ctx->h3.ptr),
                                      ld3, chunk, ldk, ctx->stream));
  ctx->launches++;
  ctx->h3_ld = ld3;
  ctx->h3_klen = klen;
  ctx->h3_rank_stride = p > 1 ? ldk : 0;
  return CHFSI_OK;
}

static chfsi_status a3_operand(chfsi_ctx ctx, CUtensorMap* m, const void* Hp, int64_t ldh, int64_t n, int64_t nloc,
                               int box_rows, bool* built, int kh = 2) {
  if (!*built) {
    if (ctx->h3_pin != Hp) {
      chfsi_status st = h3_prepare(ctx, Hp, ldh, n, nloc);
      if (st) return st;
    }
    *built = true;
  }
  return make_tmap_2d(ctx, m, ctx->h3.ptr, ctx->h3_klen, nloc, ctx->h3_ld, box_rows, 8 * kh);
}

// Tile variant and arithmetic of one launch. With the 3M column layout available (z3_layout) the
// launch runs 3M or 4M, whichever the step model rates faster: 3M does 25 % fewer tensor flops but
// streams 24 bytes of H per complex entry (interleaved + plane) against 16, so narrow, HBM-bound
// steps run 4M. Below 28 active columns 4M is used regardless (measured at n = 16384: 4M 1.55 ms vs 3M
// 1.77 ms per step at 20 and 24 columns, 3M ahead from 32; profiles/r01_ab_narrow.log);
// CHFSI_Z3_MIN_COLS overrides that threshold.
static TileChoice pick_tile(int elem, bool z3_layout, int64_t nrows, int64_t ncols, int sms, bool* z3k) {
  *z3k = false;
  if (elem == 1) return choose_filter_tile_real(nrows, ncols, sms);
  TileChoice t4 = choose_filter_tile(nrows, ncols, sms);
  if (!z3_layout) return t4;
  static const int64_t min_cols = [] {
    const char* e = getenv("CHFSI_Z3_MIN_COLS");
    return e ? (int64_t)atoll(e) : (int64_t)28;
  }();
  if (ncols < min_cols) return t4;
  TileChoice t3 = choose_filter_tile_z3(nrows, ncols, sms);
  const bool forced3 = getenv("CHFSI_FILTER_VARIANT_Z3") != nullptr;  // test / A-B hook (read per call)
  if (forced3 || t3.cost <= t4.cost) {
    *z3k = true;
    return t3;
  }
  return t4;
}

chfsi_status hmul_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                       const void* Q, int64_t ldq, int64_t k, void* out, int64_t ldo, int elem) {
  (void)row0;
  if (k == 0) return CHFSI_OK;
  const int p = ctx->nranks;
  bool z3 = false;
  TileChoice t = pick_tile(elem, elem == 2 && ctx->zmul == 3, nloc, k, ctx->num_sms, &z3);
  const int cw = z3 ? 3 : elem;
  const size_t eb = 8 * (size_t)elem;
  CUtensorMap tmA, tmA3;
  int64_t kchunk, klen;
  chfsi_status st = a_operand(ctx, &Hp, &ldh, n, nloc, elem, &kchunk, &klen);
  if (st) return st;
  st = make_tmap_2d(ctx, &tmA, Hp, elem * klen, nloc, elem * ldh, t.bm / t.cluster);
  if (st) return st;
  tmA3 = tmA;
  bool h3_built = false;
  if (z3) {
    st = a3_operand(ctx, &tmA3, Hp, ldh, n, nloc, t.bm / t.cluster, &h3_built, t.kh);
    if (st) return st;
  }
  Operand op;
  const double* bsrc = static_cast<const double*>(Q);
  int64_t bld = ldq;
  const int64_t ldp = (elem == 1 || z3) ? round_up(nloc, 2) : nloc;  // packed column stride (per plane)
  if (p > 1) {
    // gather the full-height Q into R0 = [rank][k][cw * ldp]
    st = ensure(ctx, ctx->R0, sizeof(double) * cw * (size_t)ldp * p * (size_t)k);
    if (st) return st;
    double* R = static_cast<double*>(ctx->R0.ptr);
    double* mine = R + (size_t)cw * ldp * k * ctx->rank;
    if (z3) {
      CHFSI_CUDA_TRY(ctx, launch_pack_y3(nloc, k, static_cast<const double2*>(Q), ldq, mine, 3 * ldp, 2 * ldp,
                                         ctx->stream));
      ctx->launches++;
    } else {
      CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(mine, eb * ldp, Q, eb * ldq, eb * nloc, k, cudaMemcpyDeviceToDevice,
                                            ctx->stream));
    }
    st = comm_allgather_inplace(ctx, R, (size_t)cw * ldp * k);
    if (st) return st;
    bsrc = R;
    bld = ldp;
  } else if (z3) {  // Q -> L0 in the 3M column layout
    const int64_t ldl = round_up(nloc, 2);
    st = ensure(ctx, ctx->L0, sizeof(double) * 3 * (size_t)ldl * k);
    if (st) return st;
    CHFSI_CUDA_TRY(ctx, launch_pack_y3(nloc, k, static_cast<const double2*>(Q), ldq, static_cast<double*>(ctx->L0.ptr),
                                       3 * ldl, 2 * ldl, ctx->stream));
    ctx->launches++;
    bsrc = static_cast<const double*>(ctx->L0.ptr);
    bld = ldl;
  } else if ((eb * ldq) % 16 != 0) {  // real data with an odd ld: TMA strides must be multiples of 16 bytes
    const int64_t ldl = round_up(nloc, 2);
    st = ensure(ctx, ctx->L0, eb * (size_t)ldl * k);
    if (st) return st;
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(ctx->L0.ptr, eb * ldl, Q, eb * ldq, eb * nloc, k, cudaMemcpyDeviceToDevice,
                                          ctx->stream));
    bsrc = static_cast<const double*>(ctx->L0.ptr);
    bld = ldl;
  }
  st = b_operand(ctx, &op, bsrc, p == 1 ? n : nloc, bld, k, 0, p, t.bnc, elem, cw, z3, t.kh);
  if (st) return st;
  StepParams sp{};
  sp.nrows = nloc;
  const int64_t kr = p == 1 ? elem * n : elem * nloc;
  const int64_t kbk = 16 * t.kh;  // real K per stage of the variant
  sp.kt_per_rank = (int32_t)((kr + kbk - 1) / kbk);
  sp.num_kt = sp.kt_per_rank * p;
  sp.a_rank_stride = (int32_t)(elem * kchunk);
  sp.a3_rank_stride = (int32_t)round_up(nloc, 2);
  sp.col0 = 0;
  sp.col_end = (int32_t)k;
  sp.fin_end = (int32_t)k;
  sp.b_col0 = op.b_col0;
  sp.flags = 0;
  sp.a = 1.0;
  sp.b = 0.0;
  sp.c = 0.0;
  sp.out = static_cast<double2*>(out);
  sp.ld_out = ldo;
  schedule_filter_step(t, ctx->num_sms, sp);
  st = sk_workspace(ctx, t, sp);
  if (st) return st;
  CHFSI_CUDA_TRY(ctx, launch_filter_step(t, tmA, op.tm, tmA3, op.tm3, sp, ctx->stream));
  ctx->launches++;
  return CHFSI_OK;
}

// Column groups for the p > 1 pipeline: G contiguous ranges [gb[g], gb[g+1]) of the k columns, each
// >= pipe_group_cols wide (G = 1 at p == 1: nothing to overlap).
static std::vector<int64_t> filter_groups(chfsi_ctx ctx, int64_t k) {
  int64_t G = 1;
  if (ctx->nranks > 1 && ctx->exchange == 0 && ctx->pipe_group_cols > 0) G = std::max<int64_t>(1, std::min<int64_t>(k / ctx->pipe_group_cols, 16));
  std::vector<int64_t> gb(G + 1);
  for (int64_t g = 0; g <= G; ++g) gb[g] = g * k / G;
  return gb;
}

static chfsi_status ensure_events(chfsi_ctx ctx, std::vector<cudaEvent_t>& v, size_t count, unsigned flags) {
  while (v.size() < count) {
    cudaEvent_t ev;
    CHFSI_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ev, flags));
    v.push_back(ev);
  }
  return CHFSI_OK;
}

static chfsi_status ensure_comm_stream(chfsi_ctx ctx, size_t groups) {
  if (!ctx->comm_stream) CHFSI_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  if (!ctx->join_ev) CHFSI_CUDA_TRY(ctx, cudaEventCreateWithFlags(&ctx->join_ev, cudaEventDisableTiming));
  chfsi_status st = ensure_events(ctx, ctx->grp_k, groups, cudaEventDisableTiming);
  if (!st) st = ensure_events(ctx, ctx->grp_ag, groups, cudaEventDisableTiming);
  return st;
}

// Alg 2 on this rank's rows. One K1 launch per (step, column group). At p > 1 the packed
// B operand of group g lives at R + cw*ldp*p*gb[g] with layout [rank][ka_g][cw*ldp] (cw = 3 in the 3M
// column layout); the epilogue of step i writes this rank's chunk of step i+1's operand, and an in-place
// allgather on the comm stream completes it while K1 runs on the next group ("Overlap") --
// or, with the peer exchange, the epilogue writes the chunk into every rank's buffer and a barrier
// separates the steps (one group).
chfsi_status filter_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                         void* Y, int64_t ldy, int64_t k, const int32_t* deg, double lambda1, double c, double e,
                         bool check_finite, int elem) {
  (void)row0;
  if (k == 0) return CHFSI_OK;
  const int p = ctx->nranks;
  const int32_t mk = deg[k - 1];
  // sigma schedule (Alg 2 l2, l6) in double on the host, as printed
  std::vector<double> sigma(mk + 1);
  sigma[0] = e / (lambda1 - c);
  for (int i = 1; i < mk; ++i) sigma[i] = 1.0 / (2.0 / sigma[0] - sigma[i - 1]);

  // elem = 2: complex128 (K1 in 3M or 4M form), elem = 1: real symmetric (NEXT-3); sizes in doubles.
  // cw = doubles per row of a column slot: elem, or 3 in the 3M layout [2 ld complex | ld plane]
  const bool z3 = elem == 2 && ctx->zmul == 3;
  const int cw = z3 ? 3 : elem;
  const size_t eb = 8 * (size_t)elem;  // bytes per element
  const int64_t ldl = round_up(nloc, 2);
  chfsi_status st = ensure(ctx, ctx->L0, sizeof(double) * cw * (size_t)ldl * k);
  if (!st) st = ensure(ctx, ctx->L1, sizeof(double) * cw * (size_t)ldl * k);
  if (!st) st = ensure(ctx, ctx->flag, 64);
  const int64_t ldp = (elem == 1 || z3) ? round_up(nloc, 2) : nloc;  // packed column stride (per plane)
  const bool push = p > 1 && ctx->exchange == 1;
  const size_t rbytes = sizeof(double) * cw * (size_t)ldp * p * k;
  if (push && !st && rbytes > ctx->peer_R_bytes) {  // peers hold pointers into R0 / R1: no regrowth
    set_err(ctx, "chfsi_filter: peer exchange needs " + std::to_string(rbytes) +
                     " bytes of packed-operand workspace per buffer; chfsi_ctx_reserve a larger block before "
                     "chfsi_ctx_set_exchange");
    return CHFSI_ERR_ARG;
  }
  if (p > 1 && !st) st = ensure(ctx, ctx->R0, rbytes);
  if (p > 1 && !st) st = ensure(ctx, ctx->R1, rbytes);
  int64_t kchunk = nloc, klen = n;
  if (!st) st = a_operand(ctx, &Hp, &ldh, n, nloc, elem, &kchunk, &klen);
  if (st) return st;
  const std::vector<int64_t> gb = filter_groups(ctx, k);
  const int G = (int)gb.size() - 1;
  if (p > 1) {
    st = ensure_comm_stream(ctx, G);
    if (st) return st;
  }
  const int sms = p > 1 ? std::max(1, ctx->num_sms - std::max(0, (int)ctx->pipe_sm_reserve)) : ctx->num_sms;
  double2* L[2] = {static_cast<double2*>(ctx->L0.ptr), static_cast<double2*>(ctx->L1.ptr)};
  double* R[2] = {static_cast<double*>(ctx->R0.ptr), static_cast<double*>(ctx->R1.ptr)};
  auto region = [&](int b, int g) { return R[b] + (size_t)cw * ldp * p * gb[g]; };  // group g's packed operand
  int* flag = static_cast<int*>(ctx->flag.ptr);
  if (check_finite) CHFSI_CUDA_TRY(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->stream));
  // Y_0 -> L0 (the caller's Y is the output and must never be the B operand)
  if (z3) {
    CHFSI_CUDA_TRY(ctx, launch_pack_y3(nloc, k, static_cast<const double2*>(Y), ldy, reinterpret_cast<double*>(L[0]),
                                       3 * ldl, 2 * ldl, ctx->stream));
    ctx->launches++;
  } else {
    CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(L[0], eb * ldl, Y, eb * ldy, eb * nloc, k, cudaMemcpyDeviceToDevice,
                                          ctx->stream));
  }
  if (p > 1) {  // step 1's full-height operand: this rank's rows of each group, then one allgather per group
    for (int g = 0; g < G; ++g) {
      const int64_t w = gb[g + 1] - gb[g];
      double* mine = region(0, g) + (size_t)cw * ldp * w * ctx->rank;
      const char* ysrc = static_cast<const char*>(Y) + eb * ldy * gb[g];
      if (z3) {
        CHFSI_CUDA_TRY(ctx, launch_pack_y3(nloc, w, reinterpret_cast<const double2*>(ysrc), ldy, mine, 3 * ldp, 2 * ldp,
                                           ctx->stream));
        ctx->launches++;
      } else {
        CHFSI_CUDA_TRY(ctx, cudaMemcpy2DAsync(mine, eb * ldp, ysrc, eb * ldy, eb * nloc, w, cudaMemcpyDeviceToDevice,
                                              ctx->stream));
      }
    }
    CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->join_ev, ctx->stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm_stream, ctx->join_ev, 0));
    for (int g = 0; g < G; ++g) {
      st = comm_allgather_inplace(ctx, region(0, g), (size_t)cw * ldp * (gb[g + 1] - gb[g]), ctx->comm_stream);
      if (st) return st;
      CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->grp_ag[g], ctx->comm_stream));
    }
  }
  CUtensorMap tmA, tmA3;
  int last_bm = -1, last_bm3 = -1;
  bool h3_built = false;
  // CUDA events timing K1 (read back after the final synchronisation): around every launch where it is
  // needed -- the per-launch trace (CHFSI_K1_LOG), the timeline, and p > 1, where exchanges separate the
  // launches -- otherwise one pair around the call's back-to-back launches (an event record between two
  // launches costs ~5 us of GPU time: c1 eigenproblems 1.6 % faster without them,
  // profiles/r02_ab_k1_events.txt); the K1 time then includes the few-us launch gaps
  static const bool k1_log = getenv("CHFSI_K1_LOG") != nullptr;  // per-launch trace (diagnostics)
  st = ensure_events(ctx, ctx->k1_events, (size_t)2 * (mk + 1) * G, cudaEventDefault);
  if (st) return st;
  int nev_used = 0, call_launches = 0;
  std::vector<std::pair<int, int>> launch_log;  // (active columns, variant) per K1 launch
  // timeline (CHFSI_TIMELINE): K1 intervals come from k1_events; exchanges get their own event pairs
  static const char* tl_prefix = getenv("CHFSI_TIMELINE");
  static const int tl_max = getenv("CHFSI_TIMELINE_CALLS") ? atoi(getenv("CHFSI_TIMELINE_CALLS")) : 1;
  static const int tl_skip = getenv("CHFSI_TIMELINE_SKIP") ? atoi(getenv("CHFSI_TIMELINE_SKIP")) : 0;
  if (tl_prefix) ctx->tl_seen++;
  const bool tl = tl_prefix && ctx->tl_seen > tl_skip && ctx->tl_calls < tl_max;
  struct TlRec {
    int kind, g, i, ev;  // kind 0: K1 (ev indexes k1_events), 1: exchange (ev indexes tl_events)
  };
  std::vector<TlRec> tl_log;
  int tl_used = 0;
  const bool per_launch = k1_log || tl || p > 1;
  if (tl) {
    st = ensure_events(ctx, ctx->tl_events, (size_t)2 * (mk + 2) * G + 1, cudaEventDefault);
    if (st) return st;
    CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->tl_events[tl_used++], ctx->stream));  // time origin
  }
  auto tl_pair = [&](int g, int i) -> const cudaEvent_t* {
    if (!tl) return nullptr;
    tl_log.push_back({1, g, i, tl_used});
    tl_used += 2;
    return &ctx->tl_events[tl_used - 2];
  };
  std::vector<char> plane_ok(G, 1);  // group's B operand carries a current 3M plane
  int64_t s = 0;  // active start s_i = #{j : deg[j] <= i}
  for (int i = 0; i < mk; ++i) {
    while (s < k && deg[s] <= i) ++s;
    if (s >= k) break;
    int64_t s_next = s;
    while (s_next < k && deg[s_next] <= i + 1) ++s_next;
    const int cur = i & 1, oth = cur ^ 1;
    for (int g = 0; g < G; ++g) {
      const int64_t c0 = std::max(s, gb[g]), ce = gb[g + 1];
      if (c0 >= ce) continue;  // every column of this group has finished
      const int64_t fin = std::min(std::max(s_next, c0), ce);
      const int64_t ka = ce - c0, ka_next = ce - fin;
      // this launch's arithmetic; a 4M epilogue does not write the y_r + y_i plane, so once a group
      // ran a 4M step its later steps stay 4M
      bool z3k = false;
      TileChoice t = pick_tile(elem, z3 && plane_ok[g], nloc, ka, sms, &z3k);
      if (!z3k) plane_ok[g] = 0;
      const int abox = t.bm / t.cluster;  // A box rows (a CTA pair loads half the tile each)
      if (abox != last_bm) {
        st = make_tmap_2d(ctx, &tmA, Hp, elem * klen, nloc, elem * ldh, abox);
        if (st) return st;
        last_bm = abox;
      }
      if (z3k && abox * 4 + t.kh != last_bm3) {  // the plane box depends on the rows and the stage depth
        st = a3_operand(ctx, &tmA3, Hp, ldh, n, nloc, abox, &h3_built, t.kh);
        if (st) return st;
        last_bm3 = abox * 4 + t.kh;
      }
      Operand op;
      if (p == 1)
        st = b_operand(ctx, &op, reinterpret_cast<const double*>(L[cur]), n, ldl, k, c0, 1, t.bnc, elem, cw, z3k, t.kh);
      else
        st = b_operand(ctx, &op, region(cur, g), nloc, ldp, ce, c0, p, t.bnc, elem, cw, z3k, t.kh);
      if (st) return st;
      StepParams sp{};
      sp.nrows = nloc;
      const int64_t kr = p == 1 ? elem * n : elem * nloc;
      const int64_t kbk = 16 * t.kh;  // real K per stage of the variant
      sp.kt_per_rank = (int32_t)((kr + kbk - 1) / kbk);
      sp.num_kt = sp.kt_per_rank * p;
      sp.a_rank_stride = (int32_t)(elem * kchunk);
      sp.a3_rank_stride = (int32_t)round_up(nloc, 2);
      sp.col0 = (int32_t)c0;
      sp.col_end = (int32_t)ce;
      sp.fin_end = (int32_t)fin;
      sp.b_col0 = op.b_col0;
      if (i == 0) {  // Y_1 = (sigma_1/e)(H - cI) Y_0
        sp.a = sigma[0] / e;
        sp.b = 0.0;
        sp.flags = 1;
      } else {  // Y_{i+1} = (2 sigma_{i+1}/e)(H - cI) Y_i - sigma_{i+1} sigma_i Y_{i-1}
        sp.a = 2.0 * sigma[i] / e;
        sp.b = sigma[i] * sigma[i - 1];
        sp.flags = 3;
      }
      sp.c = c;
      // state column stride in the kernel's units (double2 for complex, double for real); 3M: the
      // plane of column j starts 2 * ldl doubles after it
      const int64_t lds = z3 ? 3 * ldl / 2 : ldl;
      sp.y_cur = L[cur];
      sp.ld_cur = lds;
      sp.y_prev = L[oth];
      sp.ld_prev = lds;
      sp.y_next = L[oth];
      sp.ld_next = lds;
      sp.y3_off = 2 * ldl;
      sp.out = static_cast<double2*>(Y);
      sp.ld_out = ldy;
      if (p > 1 && ka_next > 0) {
        const size_t chunk_off = (size_t)cw * ldp * p * gb[g] + (size_t)cw * ldp * ka_next * ctx->rank;
        if (push) {  // this rank's chunk in every rank's next-step operand (NVLink peer stores)
          for (int q = 0; q < p; ++q)
            sp.r_dst[q] = reinterpret_cast<double2*>((oth ? ctx->peer_R1[q] : ctx->peer_R0[q]) + chunk_off);
          sp.n_rdst = p;
        } else {
          sp.r_dst[0] = reinterpret_cast<double2*>(R[oth] + chunk_off);
          sp.n_rdst = 1;
        }
        sp.ld_r_next = z3 ? 3 * ldp / 2 : ldp;
        sp.y3_off_r = 2 * ldp;
      }
      sp.nonfinite = check_finite ? flag : nullptr;
      schedule_filter_step(t, sms, sp);
      st = sk_workspace(ctx, t, sp);
      if (st) return st;
      // this group's operand for step i is complete once its allgather (comm stream) has landed
      if (p > 1) CHFSI_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->grp_ag[g], 0));
      if (per_launch || call_launches == 0) CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->k1_events[nev_used], ctx->stream));
      CHFSI_CUDA_TRY(ctx, launch_filter_step(t, tmA, op.tm, z3k ? tmA3 : tmA, op.tm3, sp, ctx->stream));
      launch_log.emplace_back((int)ka, t.id);
      if (tl) tl_log.push_back({0, g, i, nev_used});
      ++call_launches;
      if (per_launch) {
        CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->k1_events[nev_used + 1], ctx->stream));
        nev_used += 2;
      }
      ctx->launches++;
      if (push && ka_next > 0) {  // every rank's pushes of step i land before anyone's step i+1
        st = comm_barrier(ctx, ctx->stream);
        if (st) return st;
      } else if (p > 1 && ka_next > 0) {  // complete step i+1's operand of this group behind the next group's K1
        CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->grp_k[g], ctx->stream));
        CHFSI_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->comm_stream, ctx->grp_k[g], 0));
        st = comm_allgather_inplace(ctx, region(oth, g), (size_t)cw * ldp * ka_next, ctx->comm_stream, tl_pair(g, i));
        if (st) return st;
        CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->grp_ag[g], ctx->comm_stream));
      }
    }
  }
  if (!per_launch && call_launches > 0) {  // close the call's single K1 interval
    CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->k1_events[1], ctx->stream));
    nev_used = 2;
  }
  if (p > 1) {  // nothing on the comm stream outlives the call
    CHFSI_CUDA_TRY(ctx, cudaEventRecord(ctx->join_ev, ctx->comm_stream));
    CHFSI_CUDA_TRY(ctx, cudaStreamWaitEvent(ctx->stream, ctx->join_ev, 0));
  }
  int h_nonfinite = 0;  // read with the call's one synchronisation (no extra host round trip)
  if (check_finite)
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&h_nonfinite, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
  if (tl) {  // one JSON line per interval, times in ms from the call's origin event
    ctx->tl_calls++;
    const std::string path = std::string(tl_prefix) + "_rank" + std::to_string(ctx->rank) + ".jsonl";
    if (FILE* f = fopen(path.c_str(), "a")) {
      for (const TlRec& r : tl_log) {
        const cudaEvent_t* e = r.kind == 0 ? &ctx->k1_events[r.ev] : &ctx->tl_events[r.ev];
        float a = 0, b = 0;
        cudaEventElapsedTime(&a, ctx->tl_events[0], e[0]);
        cudaEventElapsedTime(&b, ctx->tl_events[0], e[1]);
        fprintf(f, "{\"call\": %d, \"rank\": %d, \"kind\": \"%s\", \"group\": %d, \"step\": %d, \"t0\": %.4f, \"t1\": %.4f, "
                   "\"sm_reserve\": %d, \"groups\": %d}\n",
                ctx->tl_calls, ctx->rank, r.kind == 0 ? "k1" : "exchange", r.g, r.i, a, b, ctx->pipe_sm_reserve, G);
      }
      fclose(f);
    }
  }
  for (int q = 0; q < nev_used; q += 2) {
    float ms = 0;
    CHFSI_CUDA_TRY(ctx, cudaEventElapsedTime(&ms, ctx->k1_events[q], ctx->k1_events[q + 1]));
    ctx->k1_seconds += ms * 1e-3;
    ctx->k1_launches += per_launch ? 1 : call_launches;
    if (k1_log)
      fprintf(stderr, "k1 rank %d n %lld nloc %lld ka %d variant %d ms %.4f\n", ctx->rank, (long long)n,
              (long long)nloc, launch_log[q / 2].first, launch_log[q / 2].second, ms);
  }
  if (check_finite) {
    int h = h_nonfinite;
    if (p > 1) {  // a non-finite value lives in one rank's rows: every rank takes the same branch
      double hv = h ? 1.0 : 0.0;
      double* dv = reinterpret_cast<double*>(flag) + 1;
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(dv, &hv, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
      st = comm_allreduce_sum(ctx, dv, 1);
      if (st) return st;
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(&hv, dv, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
      CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
      h = hv > 0.0;
    }
    if (h) {
      set_err(ctx, "chfsi_filter: non-finite value in the filtered block");
      return CHFSI_ERR_NONFINITE;
    }
  }
  return CHFSI_OK;
}

}  // namespace chfsi

using namespace chfsi;

// ------------------------------------------------------------------------------------------------
extern "C" {

static chfsi_status ctx_create_impl(chfsi_ctx* out, int32_t device, void* cuda_stream, void* nccl_comm,
                                    chfsi_local_group group, int32_t rank, int32_t nranks,
                                    const char* nccl_id = nullptr) {
  if (!out) return CHFSI_ERR_ARG;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !nccl_comm && !group && !nccl_id))
    return CHFSI_ERR_ARG;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0 || device < 0 || device >= ndev) {
    cudaGetLastError();
    return CHFSI_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) return CHFSI_ERR_CUDA;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return CHFSI_ERR_CUDA;
  if (prop.major != 10) return CHFSI_ERR_CUDA;  // sm_100a build only
  chfsi_ctx ctx = new chfsi_ctx_s();
  ctx->device = device;
  ctx->rank = rank;
  ctx->nranks = nranks;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->nccl_comm = nccl_comm;
  ctx->local_group = group;
  if (const char* zm = getenv("CHFSI_ZMUL")) ctx->zmul = atoi(zm) == 4 ? 4 : 3;
  if (const char* em = getenv("CHFSI_EIG")) ctx->eig_mode = strcmp(em, "dense") == 0 ? 1 : 0;
  if (nccl_id) {
    memcpy(ctx->nccl_id, nccl_id, sizeof(ctx->nccl_id));
    ctx->nccl_id_valid = true;
  }
  // NULL selects the legacy default stream (stream 0), so work is ordered with the caller's default-
  // stream copies; pass an explicit stream for concurrency.
  ctx->stream = static_cast<cudaStream_t>(cuda_stream);
  ctx->own_stream = false;
  if (cublasCreate(&ctx->cublas) != CUBLAS_STATUS_SUCCESS ||
      cublasSetStream(ctx->cublas, ctx->stream) != CUBLAS_STATUS_SUCCESS ||
      cusolverDnCreate(&ctx->cusolver) != CUSOLVER_STATUS_SUCCESS ||
      cusolverDnSetStream(ctx->cusolver, ctx->stream) != CUSOLVER_STATUS_SUCCESS) {
    chfsi_ctx_destroy(ctx);
    return CHFSI_ERR_CUDA;
  }
  chfsi_status st = comm_init(ctx);
  if (st) {
    chfsi_ctx_destroy(ctx);
    return st;
  }
  *out = ctx;
  return CHFSI_OK;
}

chfsi_status chfsi_ctx_create(chfsi_ctx* out, int32_t device, void* cuda_stream, void* nccl_comm, int32_t rank,
                              int32_t nranks) {
  return ctx_create_impl(out, device, cuda_stream, nccl_comm, nullptr, rank, nranks);
}

chfsi_status chfsi_ctx_create_nccl(chfsi_ctx* out, int32_t device, void* cuda_stream, const char id[128],
                                   int32_t rank, int32_t nranks) {
  if (!id) return CHFSI_ERR_ARG;
  return ctx_create_impl(out, device, cuda_stream, nullptr, nullptr, rank, nranks, id);
}

chfsi_status chfsi_ctx_create_local(chfsi_ctx* out, int32_t device, void* cuda_stream, chfsi_local_group group,
                                    int32_t rank) {
  if (!group) return CHFSI_ERR_ARG;
  return ctx_create_impl(out, device, cuda_stream, nullptr, group, rank, group->P);
}

chfsi_status chfsi_ctx_reserve(chfsi_ctx ctx, int64_t n, int64_t nloc, int64_t kmax) {
  if (!ctx || n < 1 || nloc < 1 || kmax < 1 || nloc > n) return CHFSI_ERR_ARG;
  cudaSetDevice(ctx->device);
  if (ctx->exchange == 1 && ctx->nranks > 1 &&
      sizeof(double) * 3 * (size_t)round_up(nloc, 2) * ctx->nranks * kmax > ctx->peer_R_bytes) {
    set_err(ctx, "chfsi_ctx_reserve: the peer exchange is on; reserve before chfsi_ctx_set_exchange");
    return CHFSI_ERR_ARG;  // peers hold pointers into R0 / R1
  }
  const size_t ldl = (size_t)round_up(nloc, 2);
  const size_t blk = sizeof(double) * 3 * ldl * kmax;  // 3M column layout (the widest)
  chfsi_status st = CHFSI_OK;
  if (!st) st = ensure(ctx, ctx->L0, blk);
  if (!st) st = ensure(ctx, ctx->L1, blk);
  if (!st) st = ensure(ctx, ctx->flag, 64);
  if (ctx->nranks > 1) {
    const size_t rb = sizeof(double) * 3 * (size_t)round_up(nloc, 2) * ctx->nranks * kmax;
    if (!st) st = ensure(ctx, ctx->R0, rb);
    if (!st) st = ensure(ctx, ctx->R1, rb);
  }
  if (!st && ctx->zmul == 3)  // the plane, with the rank chunks padded to even lengths at p > 1
    st = ensure(ctx, ctx->h3, sizeof(double) * (size_t)round_up(ctx->nranks * round_up(nloc, 2), 2) * nloc);
  return st;
}

void chfsi_ctx_destroy(chfsi_ctx ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  comm_destroy(ctx);
  DevBuf* bufs[] = {&ctx->h3, &ctx->L0, &ctx->L1, &ctx->R0, &ctx->R1, &ctx->flag, &ctx->sk, &ctx->hpad, &ctx->w1, &ctx->w2, &ctx->w3, &ctx->w4,
                    &ctx->small1, &ctx->small2, &ctx->small3, &ctx->solver_ws, &ctx->devinfo, &ctx->lz,
                    &ctx->ya,    &ctx->xl,     &ctx->tb,     &ctx->idx,    &ctx->gw,     &ctx->gx,
                    &ctx->qsave, &ctx->qrn,   &ctx->eigw};
  for (DevBuf* b : bufs)
    if (b->ptr) cudaFree(b->ptr);
  for (cudaEvent_t ev : ctx->k1_events) cudaEventDestroy(ev);
  for (cudaEvent_t ev : ctx->grp_k) cudaEventDestroy(ev);
  for (cudaEvent_t ev : ctx->grp_ag) cudaEventDestroy(ev);
  for (cudaEvent_t ev : ctx->tl_events) cudaEventDestroy(ev);
  if (ctx->join_ev) cudaEventDestroy(ctx->join_ev);
  if (ctx->lz_exec) cudaGraphExecDestroy(ctx->lz_exec);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  for (cudaEvent_t ev : ctx->eig_ev)
    if (ev) cudaEventDestroy(ev);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->cublas) cublasDestroy(ctx->cublas);
  if (ctx->cusolver) cusolverDnDestroy(ctx->cusolver);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

const char* chfsi_last_error(chfsi_ctx ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int64_t chfsi_kernel_launches(chfsi_ctx ctx) { return ctx ? ctx->launches : 0; }

chfsi_status chfsi_ctx_set_complex_mult(chfsi_ctx ctx, int32_t mults) {
  if (!ctx || (mults != 3 && mults != 4)) return CHFSI_ERR_ARG;
  ctx->zmul = mults;
  return CHFSI_OK;
}

chfsi_status chfsi_ctx_set_eigensolver(chfsi_ctx ctx, int32_t mode) {
  if (!ctx || (mode != 0 && mode != 1)) return CHFSI_ERR_ARG;
  ctx->eig_mode = mode;
  return CHFSI_OK;
}

chfsi_status chfsi_ctx_set_exchange(chfsi_ctx ctx, int32_t mode) {
  if (!ctx || (mode != 0 && mode != 1)) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (ctx->nranks == 1) {
    ctx->exchange = mode;
    return CHFSI_OK;
  }
  if (cudaSetDevice(ctx->device) != cudaSuccess) return CHFSI_ERR_CUDA;
  if (mode == 0) {
    comm_close_peers(ctx);
    ctx->exchange = 0;
    return CHFSI_OK;
  }
  if (ctx->nranks > StepParams::kMaxRdst) {  // one peer pointer per rank travels in the kernel parameters
    set_err(ctx, "chfsi_ctx_set_exchange: the peer push supports at most 8 ranks (one NVLink domain box)");
    return CHFSI_ERR_ARG;
  }
  chfsi_status st = comm_open_peers(ctx);
  if (st) return st;
  ctx->exchange = 1;
  return CHFSI_OK;
}

chfsi_status chfsi_ctx_set_pipeline(chfsi_ctx ctx, int32_t group_cols, int32_t sm_reserve) {
  if (!ctx || group_cols < 0 || sm_reserve < 0 || sm_reserve >= ctx->num_sms) return CHFSI_ERR_ARG;
  ctx->pipe_group_cols = group_cols;
  ctx->pipe_sm_reserve = sm_reserve;
  return CHFSI_OK;
}

static chfsi_status filter_entry(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                                 void* Y, int64_t ldy, int64_t k, const int32_t* deg, double lambda1, double c,
                                 double e, int64_t* matvecs, int elem) {
  if (!ctx) return CHFSI_ERR_ARG;
  ctx->err.clear();
  if (n < 1 || nloc < 1 || nloc > n || row0 < 0 || row0 + nloc > n || ldh < n || ldy < nloc || k < 0 ||
      (k > 0 && (!Hp || !Y || !deg))) {
    set_err(ctx, "chfsi_filter: bad dimensions / leading dimensions / pointers");
    return CHFSI_ERR_ARG;
  }
  if (nloc * ctx->nranks != n || row0 != nloc * ctx->rank) {
    set_err(ctx, "chfsi_filter: row panels must be equal (n = nranks * nloc, row0 = rank * nloc; nranks == 1: nloc = n, row0 = 0)");
    return CHFSI_ERR_ARG;
  }
  if (2 * n > INT32_MAX / 2) {
    set_err(ctx, "chfsi_filter: n too large");
    return CHFSI_ERR_ARG;
  }
  if (!(e > 0.0) || !(lambda1 < c - e) || !std::isfinite(c) || !std::isfinite(e) || !std::isfinite(lambda1)) {
    set_err(ctx, "chfsi_filter: need e > 0 and lambda1 < c - e (the scaling point left of [alpha, beta])");
    return CHFSI_ERR_ARG;
  }
  int64_t mv = 0;
  for (int64_t j = 0; j < k; ++j) {
    if (deg[j] < 1 || deg[j] > CHFSI_MAX_DEGREE || (j > 0 && deg[j] < deg[j - 1])) {
      set_err(ctx, "chfsi_filter: degrees must be ascending in [1, CHFSI_MAX_DEGREE]");
      return CHFSI_ERR_ARG;
    }
    mv += deg[j];
  }
  if (cudaSetDevice(ctx->device) != cudaSuccess) return CHFSI_ERR_CUDA;
  chfsi_status st = filter_impl(ctx, n, row0, nloc, Hp, ldh, Y, ldy, k, deg, lambda1, c, e, true, elem);
  if (st == CHFSI_OK && matvecs) *matvecs = mv;
  return st;
}

chfsi_status chfsi_filter(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                          void* Y, int64_t ldy, int64_t k, const int32_t* deg, double lambda1, double c, double e,
                          int64_t* matvecs) {
  return filter_entry(ctx, n, row0, nloc, Hp, ldh, Y, ldy, k, deg, lambda1, c, e, matvecs, 2);
}

chfsi_status chfsi_filter_real(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const double* Hp, int64_t ldh,
                               double* Y, int64_t ldy, int64_t k, const int32_t* deg, double lambda1, double c,
                               double e, int64_t* matvecs) {
  return filter_entry(ctx, n, row0, nloc, Hp, ldh, Y, ldy, k, deg, lambda1, c, e, matvecs, 1);
}

}  // extern "C"
