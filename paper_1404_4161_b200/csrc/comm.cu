// comm.cu -- communication layer over NCCL (NVLink 5 / NVSwitch on one B200 box). NCCL is loaded
// with dlopen on first use, so single-GPU use of libchfsi.so has no NCCL dependency. The
// communicator is the caller's (e.g. torch's ProcessGroupNCCL comm, or one built from an
// ncclUniqueId broadcast over the torch process group); the library never creates or destroys it.
#include <dlfcn.h>
#include <nccl.h>

#include "ctx.cuh"

namespace chfsi {

struct Comm {
  void* lib = nullptr;
  ncclComm_t comm = nullptr;
  decltype(&ncclAllGather) allgather = nullptr;
  decltype(&ncclAllReduce) allreduce = nullptr;
  decltype(&ncclBroadcast) bcast = nullptr;
  decltype(&ncclGetErrorString) errstr = nullptr;
};

chfsi_status comm_init(chfsi_ctx ctx) {
  if (ctx->nranks == 1) return CHFSI_OK;
  Comm* c = new Comm();
  const char* names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char* nm : names) {
    c->lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!c->lib) c->lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (c->lib) break;
  }
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
  c->comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  ctx->comm = c;
  return CHFSI_OK;
}

void comm_destroy(chfsi_ctx ctx) {
  delete ctx->comm;  // the library handle stays loaded; the communicator belongs to the caller
  ctx->comm = nullptr;
}

static chfsi_status nccl_check(chfsi_ctx ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return CHFSI_OK;
  set_err(ctx, std::string(what) + ": " + ctx->comm->errstr(r));
  return CHFSI_ERR_NCCL;
}

chfsi_status comm_allgather_inplace(chfsi_ctx ctx, double* buf, size_t count) {
  if (ctx->nranks == 1 || count == 0) return CHFSI_OK;
  return nccl_check(ctx,
                    ctx->comm->allgather(buf + count * ctx->rank, buf, count, ncclDouble, ctx->comm->comm, ctx->stream),
                    "ncclAllGather");
}

chfsi_status comm_allreduce_sum(chfsi_ctx ctx, double* buf, size_t count) {
  if (ctx->nranks == 1 || count == 0) return CHFSI_OK;
  return nccl_check(ctx, ctx->comm->allreduce(buf, buf, count, ncclDouble, ncclSum, ctx->comm->comm, ctx->stream),
                    "ncclAllReduce");
}

chfsi_status comm_bcast(chfsi_ctx ctx, double* buf, size_t count, int root) {
  if (ctx->nranks == 1 || count == 0) return CHFSI_OK;
  return nccl_check(ctx, ctx->comm->bcast(buf, buf, count, ncclDouble, root, ctx->comm->comm, ctx->stream),
                    "ncclBroadcast");
}

}  // namespace chfsi
