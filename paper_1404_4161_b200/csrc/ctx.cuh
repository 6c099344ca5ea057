// ctx.cuh -- the library context behind the chfsi_ctx handle, workspace management, TMA descriptor
// encoding and the communication layer used by every entry point.
#pragma once
#include <cublas_v2.h>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "chfsi.h"
#include "common.cuh"

// Emulated ranks on one device (comm.cu): host barrier + per-rank events.
struct chfsi_local_group_s {
  int P = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  std::vector<const void*> bufs;
  std::vector<cudaEvent_t> ready, done;
  // collectives of the group: copy engines (cudaMemcpyAsync, default) or an SM copy kernel of coll_ctas
  // thread blocks -- the way NCCL moves data, so it competes with the filter kernel for SMs
  // (CHFSI_LG_COLL=kernel, CHFSI_LG_CTAS; the sm_reserve measurement of DESIGN.md 9)
  bool coll_kernel = false;
  int coll_ctas = 16;
  std::vector<void*> R0s, R1s;  // peer push: every rank's packed operand buffers (same device)
  std::vector<size_t> Rbytes;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const long gen = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace chfsi {

// A device buffer owned by the context; grows on demand (never inside a step loop once reserved).
struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
};

struct Comm;  // comm.cu: NCCL (loaded with dlopen) or a single rank

}  // namespace chfsi

struct chfsi_ctx_s {
  int device = 0;
  int rank = 0, nranks = 1;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* nccl_comm = nullptr;
  char nccl_id[128] = {0};     // ncclUniqueId for a library-owned communicator
  bool nccl_id_valid = false;
  chfsi_local_group local_group = nullptr;
  chfsi::Comm* comm = nullptr;
  cublasHandle_t cublas = nullptr;
  cusolverDnHandle_t cusolver = nullptr;
  std::string err;
  int64_t launches = 0;
  // K1 launch timing (CUDA events around every filter-step launch): accumulated seconds, launches
  double k1_seconds = 0;
  int64_t k1_launches = 0;
  std::vector<cudaEvent_t> k1_events;
  // p > 1 filter pipelining (SURVEY 8(e) "Overlap"): the active block is cut into column groups of
  // >= pipe_group_cols columns; group g's allgather (comm_stream) overlaps group g+1's K1 (stream).
  // pipe_sm_reserve SMs are left out of K1's persistent grid for the collective's CTAs.
  // p > 1 exchange of the filter's next-step operand: 0 = in-place allgather per column group on a
  // communication stream; 1 = peer push (K1's epilogue stores this rank's chunk straight into every
  // rank's buffer through peer pointers, then one small barrier per step)
  int32_t exchange = 0;
  std::vector<double*> peer_R0, peer_R1;  // exchange 1: rank q's R0 / R1 as addressed from here
  size_t peer_R_bytes = 0;                // smallest R buffer over the ranks (no regrowth after)
  std::vector<void*> ipc_opened;          // peer mappings to close (cudaIpcCloseMemHandle)
  int32_t pipe_group_cols = 128;
  int32_t pipe_sm_reserve = 0;
  // timeline of the p > 1 filter pipeline (CHFSI_TIMELINE=<prefix>): CUDA-event intervals of every K1
  // launch and every column group's exchange of the first CHFSI_TIMELINE_CALLS (default 1) filter calls,
  // written to <prefix>_rank<r>.jsonl
  std::vector<cudaEvent_t> tl_events;
  int tl_calls = 0, tl_seen = 0;  // calls written / filter calls seen (CHFSI_TIMELINE_SKIP skips the first)
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> grp_k, grp_ag;  // per group: K1 done (stream), allgather done (comm_stream)
  cudaEvent_t join_ev = nullptr;
  // complex filter arithmetic: 3 = Gauss 3M (default), 4 = the 4M real embedding (CHFSI_ZMUL=4 or
  // chfsi_ctx_set_complex_mult); h3 = the Re H - Im H plane of the panel, valid for h3_pin while the
  // solver holds one eigenproblem's H fixed
  int zmul = 3;
  chfsi::DevBuf h3;
  int64_t h3_ld = 0;
  int64_t h3_klen = 0;         // K extent of the plane (n, or p chunks of nloc padded to even)
  int64_t h3_rank_stride = 0;  // K offset between rank chunks of the plane (p > 1)
  const void* h3_pin = nullptr;

  // workspace
  chfsi::DevBuf L0, L1;          // filter local state (nloc x k each)
  chfsi::DevBuf R0, R1;          // p > 1: packed full-height B operands
  chfsi::DevBuf flag;            // int nonfinite flag (+ small scalars)
  chfsi::DevBuf sk;              // K1 stream-K workspace: tickets (zeroed) + partial accumulators
  chfsi::DevBuf hpad;            // real H panel re-strided to an even leading dimension (TMA)
  chfsi::DevBuf w1, w2, w3, w4;  // general nloc x k / k x k scratch for QR / RR / solver
  chfsi::DevBuf small1, small2, small3;
  chfsi::DevBuf solver_ws;       // cuSOLVER workspace
  chfsi::DevBuf devinfo;
  chfsi::DevBuf lz;              // Lanczos basis
  // p == 1: the Lanczos steps as one captured CUDA graph, replayed for every problem (the panel pointer
  // travels through a device slot); re-captured when its shape or workspace changes
  cudaGraphExec_t lz_exec = nullptr;
  std::vector<int64_t> lz_key;
  bool lz_graph_off = false;  // capture failed once (or CHFSI_GRAPHS=0): launch the steps directly
  cudaStream_t cap_stream = nullptr;  // capture happens here (the legacy default stream cannot be captured)
  chfsi::DevBuf ya, xl, tb, idx;  // solver: active block, locked block, filter block, column indices
  chfsi::DevBuf qsave, qrn;      // QR: the projected block (Householder / R23 restart), column norms
  chfsi::DevBuf eigw;            // k x k eigensolve: refinement workspace (eig_refine.cu)
  // Rayleigh-Ritz eigensolver: 0 = Jacobi-type refinement with the dense fallback, 1 = dense (ZHEEVD) only
  int32_t eig_mode = 0;
  int64_t eig_refined = 0, eig_dense = 0;  // eigensolves by each path (rank 0)
  double eig_seconds = 0;                  // their CUDA-event time (rank 0)
  cudaEvent_t eig_ev[2] = {nullptr, nullptr};
  chfsi::DevBuf gw, gx;          // generalised front / back end on row panels: n x n and n x nloc scratch
  chfsi::DevBuf host_pinned_dummy;
  std::vector<char> hbuf;        // host staging
};

namespace chfsi {

chfsi_status ensure(chfsi_ctx ctx, DevBuf& b, size_t bytes);
// K1 stream-K workspace for tile variant `t`: fills p.partials / p.tickets
struct TileChoice;
struct StepParams;
chfsi_status sk_workspace(chfsi_ctx ctx, const TileChoice& t, StepParams& p);
void set_err(chfsi_ctx ctx, const std::string& msg);

// TMA descriptors (FLOAT64, 128B swizzle, OOB -> zero fill)
//  A: real K-major matrix of `rows` rows with `kreal` doubles each, row stride ld_doubles; box (16, box_rows)
//  B: 3-D (kreal, cols, chunks) with column stride ld_doubles and chunk stride chunk_doubles
//  box_inner = 16 doubles (one 128-byte swizzle row) unless given; 8 doubles selects the 64B swizzle
chfsi_status make_tmap_2d(chfsi_ctx ctx, CUtensorMap* m, const void* base, int64_t kreal, int64_t rows,
                          int64_t ld_doubles, int box_rows, int box_inner = 16);
chfsi_status make_tmap_3d(chfsi_ctx ctx, CUtensorMap* m, const void* base, int64_t kreal, int64_t cols,
                          int64_t chunks, int64_t ld_doubles, int64_t chunk_doubles, int box_cols, int box_inner = 16);

// Communication (comm.cu). With nranks == 1 every collective is a no-op / local copy.
chfsi_status comm_init(chfsi_ctx ctx);
void comm_destroy(chfsi_ctx ctx);
// in-place allgather: buf holds nranks chunks of `count` doubles; chunk `rank` is the send part.
// Enqueued on `st` (nullptr: the ctx stream).
// ev_move (nullable, timeline): two events recorded on `st` around the data movement itself (after the
// wait for the peers' data to exist)
chfsi_status comm_allgather_inplace(chfsi_ctx ctx, double* buf, size_t count, cudaStream_t st = nullptr,
                                    const cudaEvent_t* ev_move = nullptr);
chfsi_status comm_allreduce_sum(chfsi_ctx ctx, double* buf, size_t count);
chfsi_status comm_bcast(chfsi_ctx ctx, double* buf, size_t count, int root);
// every rank's work enqueued on `st` before the call is complete before any rank's later work on `st`
// (NCCL: a one-element allreduce; local group: events + host barrier)
chfsi_status comm_barrier(chfsi_ctx ctx, cudaStream_t st);
// collective: make every rank's R0 / R1 addressable from every rank (exchange 1)
chfsi_status comm_open_peers(chfsi_ctx ctx);
void comm_close_peers(chfsi_ctx ctx);

// internal (no status marshalling) versions of the public entry points, used by the solver
chfsi_status filter_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                         void* Y, int64_t ldy, int64_t k, const int32_t* deg, double lambda1, double c, double e,
                         bool check_finite, int elem = 2);
// HQ: out (nloc x k) = H Q for Q (nloc x k, this rank's rows). Uses the K1 kernel, plain epilogue.
// 3M: (re)build the Re H - Im H plane of the panel in ctx->h3
chfsi_status h3_prepare(chfsi_ctx ctx, const void* Hp, int64_t ldh, int64_t n, int64_t nloc);
chfsi_status hmul_impl(chfsi_ctx ctx, int64_t n, int64_t row0, int64_t nloc, const void* Hp, int64_t ldh,
                       const void* Q, int64_t ldq, int64_t k, void* out, int64_t ldo, int elem = 2);

}  // namespace chfsi
