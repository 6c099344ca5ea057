// comm.cu -- communication layer.
//  * NCCL (NVLink 5 / NVSwitch on one B200 box), loaded with dlopen on first use so single-GPU use of
//    libchfsi.so has no NCCL dependency. The communicator is the caller's (e.g. torch's
//    ProcessGroupNCCL comm); the library never creates or destroys it.
//  * A local group: P ranks emulated on one device, one host thread per rank, each with its own
//    stream. Collectives are device copies / a fixed-order reduction ordered by CUDA events and a
//    host barrier -- the same semantics as the NCCL calls (in-place allgather, allreduce, broadcast),
//    so the P > 1 data path (row panels, packed B operands, rank-chunked K loop) runs on a 1-GPU box.
//    No kernel ever waits on another kernel; ordering is host barrier + cudaStreamWaitEvent.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "ctx.cuh"

namespace chfsi {

struct Comm {
  void* lib = nullptr;
  ncclComm_t comm = nullptr;
  bool owns_comm = false;  // created by chfsi_ctx_create_nccl
  chfsi_local_group local = nullptr;
  double* scratch = nullptr;  // local-group allreduce accumulator
  size_t scratch_n = 0;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};

static void* nccl_lib() {
  static void* lib = nullptr;
  if (!lib) {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
      if (!lib) lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
  }
  return lib;
}

chfsi_status comm_init(chfsi_ctx ctx) {
  // a library-owned NCCL communicator is created even for one rank (exercises the NCCL plumbing);
  // the collectives below are no-ops whenever nranks == 1
  if (ctx->nranks == 1 && !ctx->nccl_id_valid) return CHFSI_OK;
  Comm* c = new Comm();
  if (ctx->local_group) {
    c->local = ctx->local_group;
    ctx->comm = c;
    return CHFSI_OK;
  }
  c->lib = nccl_lib();
  if (!c->lib) {
    set_err(ctx, "NCCL (libnccl.so.2) not found");
    delete c;
    return CHFSI_ERR_NCCL;
  }
  c->allgather = reinterpret_cast<decltype(&ncclAllGather)>(dlsym(c->lib, "ncclAllGather"));
  c->allreduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(c->lib, "ncclAllReduce"));
  c->bcast = reinterpret_cast<decltype(&ncclBroadcast)>(dlsym(c->lib, "ncclBroadcast"));
  c->errstr = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(c->lib, "ncclGetErrorString"));
  if (!c->allgather || !c->allreduce || !c->bcast || !c->errstr) {
    set_err(ctx, "NCCL symbols missing");
    delete c;
    return CHFSI_ERR_NCCL;
  }
  if (ctx->nccl_id_valid) {  // library-owned communicator
    auto init = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(c->lib, "ncclCommInitRank"));
    ncclUniqueId id;
    static_assert(sizeof(id) == sizeof(ctx->nccl_id), "ncclUniqueId size");
    memcpy(&id, ctx->nccl_id, sizeof(id));
    ncclResult_t r = init ? init(&c->comm, ctx->nranks, id, ctx->rank) : ncclInternalError;
    if (r != ncclSuccess) {
      set_err(ctx, std::string("ncclCommInitRank: ") + c->errstr(r));
      delete c;
      return CHFSI_ERR_NCCL;
    }
    c->owns_comm = true;
  } else {
    c->comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  }
  ctx->comm = c;
  return CHFSI_OK;
}

void comm_close_peers(chfsi_ctx ctx);

void comm_destroy(chfsi_ctx ctx) {
  comm_close_peers(ctx);
  if (ctx->comm && ctx->comm->scratch) cudaFree(ctx->comm->scratch);
  if (ctx->comm && ctx->comm->owns_comm && ctx->comm->comm) {
    auto destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(ctx->comm->lib, "ncclCommDestroy"));
    if (destroy) destroy(ctx->comm->comm);
  }
  delete ctx->comm;  // the NCCL library handle stays loaded; the communicator belongs to the caller
  ctx->comm = nullptr;
}

static chfsi_status nccl_check(chfsi_ctx ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return CHFSI_OK;
  set_err(ctx, std::string(what) + ": " + ctx->comm->errstr(r));
  return CHFSI_ERR_NCCL;
}

// ---- local group primitives ----
namespace {

__global__ void sum_ranks_kernel(const double* const* src, int P, size_t count, double* dst) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    double s = 0;
    for (int q = 0; q < P; ++q) s += src[q][i];  // fixed rank order: identical bits on every rank
    dst[i] = s;
  }
}

// SM-kernel allgather for the local group: chunk q of every peer's buffer into ours (grid-stride copy)
struct GatherSrc {
  const double* src[8];
};
__global__ void lg_gather_kernel(GatherSrc s, int P, int rank, size_t count, double* dst) {
  const size_t total = count * (size_t)P;
  for (size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (size_t)gridDim.x * blockDim.x) {
    const int q = (int)(t / count);
    if (q == rank) continue;
    dst[t] = s.src[q][t];
  }
}

// publish `buf`, wait until every rank has published and its producer work is ordered before ours
void lg_enter(chfsi_ctx ctx, const void* buf, cudaStream_t st) {
  chfsi_local_group g = ctx->comm->local;
  g->bufs[ctx->rank] = buf;
  cudaEventRecord(g->ready[ctx->rank], st);
  g->barrier();
  for (int q = 0; q < g->P; ++q)
    if (q != ctx->rank) cudaStreamWaitEvent(st, g->ready[q], 0);
}

// every rank's reads of the published buffers are ordered before anyone's later writes
void lg_exit(chfsi_ctx ctx, cudaStream_t st) {
  chfsi_local_group g = ctx->comm->local;
  cudaEventRecord(g->done[ctx->rank], st);
  g->barrier();
  for (int q = 0; q < g->P; ++q)
    if (q != ctx->rank) cudaStreamWaitEvent(st, g->done[q], 0);
  g->barrier();  // nobody re-records its events before all waits above were issued
}

}  // namespace

chfsi_status comm_allgather_inplace(chfsi_ctx ctx, double* buf, size_t count, cudaStream_t st,
                                    const cudaEvent_t* ev_move) {
  if (ctx->nranks == 1 || count == 0) return CHFSI_OK;
  if (!st) st = ctx->stream;
  if (ctx->comm->local) {
    chfsi_local_group g = ctx->comm->local;
    lg_enter(ctx, buf, st);
    if (ev_move) CHFSI_CUDA_TRY(ctx, cudaEventRecord(ev_move[0], st));
    if (g->coll_kernel && g->P <= 8) {
      GatherSrc s{};
      for (int q = 0; q < g->P; ++q) s.src[q] = static_cast<const double*>(g->bufs[q]);
      lg_gather_kernel<<<g->coll_ctas, 512, 0, st>>>(s, g->P, ctx->rank, count, buf);
      CHFSI_CUDA_TRY(ctx, cudaGetLastError());
      ctx->launches++;
    } else {
      for (int q = 0; q < g->P; ++q) {
        if (q == ctx->rank) continue;
        const double* src = static_cast<const double*>(g->bufs[q]) + count * q;
        CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(buf + count * q, src, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
      }
    }
    if (ev_move) CHFSI_CUDA_TRY(ctx, cudaEventRecord(ev_move[1], st));
    lg_exit(ctx, st);
    return CHFSI_OK;
  }
  if (ev_move) CHFSI_CUDA_TRY(ctx, cudaEventRecord(ev_move[0], st));
  chfsi_status r = nccl_check(
      ctx, ctx->comm->allgather(buf + count * ctx->rank, buf, count, ncclDouble, ctx->comm->comm, st), "ncclAllGather");
  if (!r && ev_move) CHFSI_CUDA_TRY(ctx, cudaEventRecord(ev_move[1], st));
  return r;
}

chfsi_status comm_allreduce_sum(chfsi_ctx ctx, double* buf, size_t count) {
  if (ctx->nranks == 1 || count == 0) return CHFSI_OK;
  if (ctx->comm->local) {
    Comm* c = ctx->comm;
    chfsi_local_group g = c->local;
    if (c->scratch_n < count + (size_t)g->P) {
      if (c->scratch) {
        cudaStreamSynchronize(ctx->stream);
        cudaFree(c->scratch);
      }
      CHFSI_CUDA_TRY(ctx, cudaMalloc(&c->scratch, sizeof(double) * (count + (size_t)g->P)));
      c->scratch_n = count + (size_t)g->P;
    }
    lg_enter(ctx, buf, ctx->stream);
    const double** ptrs = reinterpret_cast<const double**>(c->scratch + count);
    std::vector<const double*> hp(g->P);
    for (int q = 0; q < g->P; ++q) hp[q] = static_cast<const double*>(g->bufs[q]);
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(ptrs, hp.data(), sizeof(double*) * g->P, cudaMemcpyHostToDevice, ctx->stream));
    const unsigned blocks = (unsigned)std::min<size_t>((count + 255) / 256, 1024);
    sum_ranks_kernel<<<blocks, 256, 0, ctx->stream>>>(ptrs, g->P, count, c->scratch);
    CHFSI_CUDA_TRY(ctx, cudaGetLastError());
    ctx->launches++;
    lg_exit(ctx, ctx->stream);
    CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(buf, c->scratch, count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    // the pointer table is rewritten by the next call only after this stream's work: order it
    CHFSI_CUDA_TRY(ctx, cudaStreamSynchronize(ctx->stream));
    return CHFSI_OK;
  }
  return nccl_check(ctx, ctx->comm->allreduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm->comm, ctx->stream),
                    "ncclAllReduce");
}

chfsi_status comm_bcast(chfsi_ctx ctx, double* buf, size_t count, int root) {
  if (ctx->nranks == 1 || count == 0) return CHFSI_OK;
  if (ctx->comm->local) {
    chfsi_local_group g = ctx->comm->local;
    lg_enter(ctx, buf, ctx->stream);
    if (ctx->rank != root)
      CHFSI_CUDA_TRY(ctx, cudaMemcpyAsync(buf, g->bufs[root], count * sizeof(double), cudaMemcpyDeviceToDevice,
                                          ctx->stream));
    lg_exit(ctx, ctx->stream);
    return CHFSI_OK;
  }
  return nccl_check(ctx, ctx->comm->bcast(buf, buf, count, ncclDouble, root, ctx->comm->comm, ctx->stream),
                    "ncclBroadcast");
}

chfsi_status comm_barrier(chfsi_ctx ctx, cudaStream_t st) {
  if (ctx->nranks == 1) return CHFSI_OK;
  if (!st) st = ctx->stream;
  if (ctx->comm->local) {
    lg_enter(ctx, nullptr, st);
    lg_exit(ctx, st);
    return CHFSI_OK;
  }
  if (!ctx->comm->scratch) {  // one zeroed word: the barrier reduces zeros (the value is never read)
    CHFSI_CUDA_TRY(ctx, cudaMalloc(&ctx->comm->scratch, sizeof(double) * 8));
    CHFSI_CUDA_TRY(ctx, cudaMemsetAsync(ctx->comm->scratch, 0, sizeof(double) * 8, st));
  }
  return nccl_check(ctx, ctx->comm->allreduce(ctx->comm->scratch, ctx->comm->scratch, 1, ncclDouble, ncclSum,
                                              ctx->comm->comm, st),
                    "ncclAllReduce (barrier)");
}

namespace {
struct PeerInfo {
  cudaIpcMemHandle_t h0, h1;
  uint64_t bytes;
  int32_t device;
  int32_t pad;
};
}  // namespace

chfsi_status comm_open_peers(chfsi_ctx ctx) {
  const int P = ctx->nranks;
  comm_close_peers(ctx);
  ctx->peer_R0.assign(P, nullptr);
  ctx->peer_R1.assign(P, nullptr);
  const size_t mine = std::min(ctx->R0.bytes, ctx->R1.bytes);
  if (!ctx->R0.ptr || !ctx->R1.ptr) {
    set_err(ctx, "peer exchange: reserve the workspace first (chfsi_ctx_reserve)");
    return CHFSI_ERR_ARG;
  }
  if (ctx->comm->local) {  // one process, one device: the group table holds every rank's pointers
    chfsi_local_group g = ctx->comm->local;
    {
      std::lock_guard<std::mutex> lk(g->m);
      if ((int)g->R0s.size() != P) {
        g->R0s.assign(P, nullptr);
        g->R1s.assign(P, nullptr);
        g->Rbytes.assign(P, 0);
      }
      g->R0s[ctx->rank] = ctx->R0.ptr;
      g->R1s[ctx->rank] = ctx->R1.ptr;
      g->Rbytes[ctx->rank] = mine;
    }
    g->barrier();
    size_t mn = mine;
    for (int q = 0; q < P; ++q) {
      ctx->peer_R0[q] = static_cast<double*>(g->R0s[q]);
      ctx->peer_R1[q] = static_cast<double*>(g->R1s[q]);
      mn = std::min(mn, g->Rbytes[q]);
    }
    g->barrier();
    ctx->peer_R_bytes = mn;
    return CHFSI_OK;
  }
  // separate processes: CUDA IPC handles of R0 / R1, gathered over the library's NCCL communicator.
  // Every rank takes part in every collective below whatever fails locally, and the ranks agree on the
  // outcome at the end (a failure count, allreduced), so either all ranks map their peers or all
  // return the same error -- a rank that failed alone would otherwise leave the others in a collective
  PeerInfo me{};
  bool ok = cudaIpcGetMemHandle(&me.h0, ctx->R0.ptr) == cudaSuccess &&
            cudaIpcGetMemHandle(&me.h1, ctx->R1.ptr) == cudaSuccess;
  if (!ok) cudaGetLastError();
  me.bytes = mine;
  me.device = ok ? ctx->device : -1;  // -1: this rank has no handles to offer
  const size_t chunk = (sizeof(PeerInfo) + 7) / 8;  // in doubles
  double* d = nullptr;
  CHFSI_CUDA_TRY(ctx, cudaMalloc(&d, sizeof(double) * (chunk * P + 1)));
  std::vector<PeerInfo> all(P);
  chfsi_status st = CHFSI_OK;
  if (cudaMemcpyAsync(d + chunk * ctx->rank, &me, sizeof(me), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
    st = CHFSI_ERR_CUDA;
  if (!st) st = comm_allgather_inplace(ctx, d, chunk, ctx->stream);
  for (int q = 0; q < P && !st; ++q)
    if (cudaMemcpyAsync(&all[q], d + chunk * q, sizeof(PeerInfo), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess)
      st = CHFSI_ERR_CUDA;
  if (!st && cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = CHFSI_ERR_CUDA;
  if (st) {  // the gather itself failed (a communicator problem every rank sees)
    cudaFree(d);
    set_err(ctx, "peer exchange: gathering the IPC handles failed");
    return st;
  }
  std::string why = ok ? "" : "cudaIpcGetMemHandle failed on this rank";
  size_t mn = mine;
  for (int q = 0; q < P; ++q) {
    mn = std::min<size_t>(mn, all[q].bytes);
    if (q == ctx->rank) {
      ctx->peer_R0[q] = static_cast<double*>(ctx->R0.ptr);
      ctx->peer_R1[q] = static_cast<double*>(ctx->R1.ptr);
      continue;
    }
    if (!ok) continue;
    if (all[q].device < 0) {
      ok = false;
      why = "rank " + std::to_string(q) + " could not export its operand buffers";
      continue;
    }
    int can = 0;
    cudaDeviceCanAccessPeer(&can, ctx->device, all[q].device);
    if (can) {
      cudaError_t e = cudaDeviceEnablePeerAccess(all[q].device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
    }
    void* p0 = nullptr;
    void* p1 = nullptr;
    if (cudaIpcOpenMemHandle(&p0, all[q].h0, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess ||
        cudaIpcOpenMemHandle(&p1, all[q].h1, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      if (p0) cudaIpcCloseMemHandle(p0);
      ok = false;
      why = "cudaIpcOpenMemHandle failed for rank " + std::to_string(q);
      continue;
    }
    ctx->ipc_opened.push_back(p0);
    ctx->ipc_opened.push_back(p1);
    ctx->peer_R0[q] = static_cast<double*>(p0);
    ctx->peer_R1[q] = static_cast<double*>(p1);
  }
  // agreement: the number of ranks that failed (also the barrier after which peers may be written)
  double* fails = d + chunk * P;
  const double mine_fail = ok ? 0.0 : 1.0;
  double total_fail = 0.0;
  st = CHFSI_OK;
  if (cudaMemcpyAsync(fails, &mine_fail, sizeof(double), cudaMemcpyHostToDevice, ctx->stream) != cudaSuccess)
    st = CHFSI_ERR_CUDA;
  if (!st) st = comm_allreduce_sum(ctx, fails, 1);
  if (!st && (cudaMemcpyAsync(&total_fail, fails, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream) != cudaSuccess ||
              cudaStreamSynchronize(ctx->stream) != cudaSuccess))
    st = CHFSI_ERR_CUDA;
  cudaFree(d);
  if (st || total_fail > 0.0) {
    comm_close_peers(ctx);
    set_err(ctx, "peer exchange unavailable: " +
                     (why.empty() ? std::to_string((int)total_fail) + " other rank(s) failed to map their peers" : why));
    return st ? st : CHFSI_ERR_CUDA;
  }
  ctx->peer_R_bytes = mn;
  return CHFSI_OK;
}

void comm_close_peers(chfsi_ctx ctx) {
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  ctx->ipc_opened.clear();
  ctx->peer_R0.clear();
  ctx->peer_R1.clear();
  ctx->peer_R_bytes = 0;
}

}  // namespace chfsi

extern "C" {

chfsi_status chfsi_nccl_unique_id(char id_out[128]) {
  if (!id_out) return CHFSI_ERR_ARG;
  void* lib = chfsi::nccl_lib();
  auto get = lib ? reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(lib, "ncclGetUniqueId")) : nullptr;
  if (!get) return CHFSI_ERR_NCCL;
  ncclUniqueId id;
  if (get(&id) != ncclSuccess) return CHFSI_ERR_NCCL;
  memcpy(id_out, &id, sizeof(id));
  return CHFSI_OK;
}

chfsi_status chfsi_local_group_create(chfsi_local_group* out, int32_t nranks) {
  if (!out || nranks < 1) return CHFSI_ERR_ARG;
  chfsi_local_group g = new chfsi_local_group_s();
  g->P = nranks;
  if (const char* m = getenv("CHFSI_LG_COLL")) g->coll_kernel = strcmp(m, "kernel") == 0;
  if (const char* c = getenv("CHFSI_LG_CTAS")) g->coll_ctas = std::max(1, atoi(c));
  g->bufs.assign(nranks, nullptr);
  g->ready.assign(nranks, nullptr);
  g->done.assign(nranks, nullptr);
  for (int q = 0; q < nranks; ++q) {
    if (cudaEventCreateWithFlags(&g->ready[q], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&g->done[q], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      chfsi_local_group_destroy(g);
      return CHFSI_ERR_CUDA;
    }
  }
  *out = g;
  return CHFSI_OK;
}

void chfsi_local_group_destroy(chfsi_local_group g) {
  if (!g) return;
  for (auto e : g->ready)
    if (e) cudaEventDestroy(e);
  for (auto e : g->done)
    if (e) cudaEventDestroy(e);
  delete g;
}

}  // extern "C"
