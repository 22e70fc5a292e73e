// §8b multi-GPU boundary: NCCL collectives on the context stream for the
// row-sharded configurations (config 4's one all-reduce of
// the sketched rows, config 3's per-half-sweep strip exchange, the residual
// partials). NCCL (over NVLink / NVSwitch on a B200 box) is loaded at the
// first call with dlopen("libnccl.so.2"), so the library itself has no
// link-time NCCL dependency; without it the entry points return
// SLRA_ERR_UNSUPPORTED. Every collective is enqueued on the context's stream:
// it orders after the kernels that produced its input and before those that
// consume its output, with no host synchronisation.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"

struct slra_comm_s {
  ncclComm_t nc = nullptr;
  slra_dev::Context* cx = nullptr;
  int nranks = 1, rank = 0;
};

namespace slra_dev {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(dlsym(h, "ncclBroadcast"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.all_gather &&
             api.broadcast && api.error_string;
  });
  return api;
}

int nccl_status(ncclResult_t r, const char* where) {
  if (r == ncclSuccess) return SLRA_OK;
  set_last_error(std::string(where) + ": " + nccl().error_string(r));
  return r == ncclInvalidArgument || r == ncclInvalidUsage ? SLRA_ERR_INVALID_ARGUMENT : SLRA_ERR_CUDA;
}

}  // namespace
}  // namespace slra_dev

using namespace slra_dev;

extern "C" {

int slra_comm_available(void) { return nccl().ok ? 1 : 0; }

int slra_comm_unique_id(void* h_id) {
  if (!h_id) return SLRA_ERR_INVALID_ARGUMENT;
  if (!nccl().ok) {
    set_last_error("libnccl.so.2 not found");
    return SLRA_ERR_UNSUPPORTED;
  }
  ncclUniqueId id;
  const int st = nccl_status(nccl().get_unique_id(&id), "ncclGetUniqueId");
  if (st == SLRA_OK) memcpy(h_id, &id, sizeof(id));
  return st;
}

int slra_comm_init(slra_ctx ctx, int nranks, int rank, const void* h_id, slra_comm* out) {
  if (!ctx || !h_id || !out || nranks < 1 || rank < 0 || rank >= nranks) return SLRA_ERR_INVALID_ARGUMENT;
  if (!nccl().ok) {
    set_last_error("libnccl.so.2 not found");
    return SLRA_ERR_UNSUPPORTED;
  }
  Context* cx = C(ctx);
  SLRA_CUDA(cudaSetDevice(cx->device));
  ncclUniqueId id;
  memcpy(&id, h_id, sizeof(id));
  auto* c = new slra_comm_s;
  c->cx = cx;
  c->nranks = nranks;
  c->rank = rank;
  const int st = nccl_status(nccl().comm_init_rank(&c->nc, nranks, id, rank), "ncclCommInitRank");
  if (st != SLRA_OK) {
    delete c;
    return st;
  }
  *out = c;
  return SLRA_OK;
}

int slra_comm_destroy(slra_comm comm) {
  if (!comm) return SLRA_OK;
  cudaStreamSynchronize(comm->cx->stream);
  const int st = comm->nc ? nccl_status(nccl().comm_destroy(comm->nc), "ncclCommDestroy") : SLRA_OK;
  delete comm;
  return st;
}

int slra_comm_allreduce_sum(slra_comm comm, const double* d_send, double* d_recv, int64_t count) {
  if (!comm || count < 0 || (count > 0 && (!d_send || !d_recv))) return SLRA_ERR_INVALID_ARGUMENT;
  if (count == 0) return SLRA_OK;
  SLRA_TIMED(comm->cx, "comm_allreduce",
             const int st = nccl_status(nccl().all_reduce(d_send, d_recv, (size_t)count, ncclFloat64, ncclSum,
                                                          comm->nc, comm->cx->stream),
                                        "ncclAllReduce");
             if (st != SLRA_OK) return st;)
  return SLRA_OK;
}

int slra_comm_allreduce_max(slra_comm comm, const double* d_send, double* d_recv, int64_t count) {
  if (!comm || count < 0 || (count > 0 && (!d_send || !d_recv))) return SLRA_ERR_INVALID_ARGUMENT;
  if (count == 0) return SLRA_OK;
  return nccl_status(nccl().all_reduce(d_send, d_recv, (size_t)count, ncclFloat64, ncclMax, comm->nc,
                                       comm->cx->stream),
                     "ncclAllReduce");
}

int slra_comm_allgather(slra_comm comm, const double* d_send, double* d_recv, int64_t count_per_rank) {
  if (!comm || count_per_rank < 0 || (count_per_rank > 0 && (!d_send || !d_recv))) return SLRA_ERR_INVALID_ARGUMENT;
  if (count_per_rank == 0) return SLRA_OK;
  SLRA_TIMED(comm->cx, "comm_allgather",
             const int st = nccl_status(nccl().all_gather(d_send, d_recv, (size_t)count_per_rank, ncclFloat64,
                                                          comm->nc, comm->cx->stream),
                                        "ncclAllGather");
             if (st != SLRA_OK) return st;)
  return SLRA_OK;
}

int slra_comm_broadcast(slra_comm comm, double* d_buf, int64_t count, int root) {
  if (!comm || count < 0 || root < 0 || root >= comm->nranks) return SLRA_ERR_INVALID_ARGUMENT;
  if (count == 0) return SLRA_OK;
  return nccl_status(nccl().broadcast(d_buf, d_buf, (size_t)count, ncclFloat64, root, comm->nc, comm->cx->stream),
                     "ncclBroadcast");
}

int slra_comm_size(slra_comm comm) { return comm ? comm->nranks : 0; }
int slra_comm_rank(slra_comm comm) { return comm ? comm->rank : -1; }

}  // extern "C"
