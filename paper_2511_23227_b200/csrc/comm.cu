// comm.cu -- the weight-gradient all-reduce of SURVEY.md §8(e): one
// ncclAllReduce(sum) of dW per layer and backward over NVLink / NVSwitch,
// on the context stream.  Whole point clouds are sharded per GPU (pairs never
// cross batches, spatial.cpp:68-77), so this is the only exchange the path
// has; dW = sum over ranks of each rank's sum over its triplets
// (vvor.hpp:79-84).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2; inside a PyTorch
// process that is the library torch already loaded), so libnpcg.so loads on
// hosts without NCCL and single-GPU users never touch it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "npcg_internal.cuh"

struct npcg_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
};

namespace npcg {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL not available: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!api.get_unique_id || !api.comm_init_rank || !api.comm_destroy || !api.all_reduce)
      err = "NCCL library lacks the required entry points";
  });
  if (!err.empty()) fail(NPCG_ERR_UNSUPPORTED, err);
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const char* m = nccl().error_string ? nccl().error_string(r) : "?";
  fail(NPCG_ERR_CUDA, std::string(what) + ": " + m);
}

}  // namespace
}  // namespace npcg

using namespace npcg;

static_assert(NCCL_UNIQUE_ID_BYTES == NPCG_COMM_ID_BYTES, "unique id size");

npcg_status npcg_comm_unique_id(uint8_t* id) {
  if (!id) return NPCG_ERR_INVALID;
  return guard(nullptr, [&] {
    ncclUniqueId u;
    check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  });
}

npcg_status npcg_comm_create(npcg_context* ctx, int nranks, int rank, const uint8_t* id,
                             npcg_comm** out) {
  if (!ctx || !id || !out) return NPCG_ERR_INVALID;
  *out = nullptr;
  return guard(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(NPCG_ERR_INVALID, "comm: bad rank / size");
    NPCG_CUDA(cudaSetDevice(ctx->device));
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    auto c = std::make_unique<npcg_comm>();
    check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
  });
}

npcg_status npcg_comm_destroy(npcg_comm* comm) {
  if (!comm) return NPCG_ERR_INVALID;
  if (comm->comm) nccl().comm_destroy(comm->comm);
  delete comm;
  return NPCG_OK;
}

// dW (K, G, C_out, C_in) summed over ranks in place, stream-ordered on the
// context stream (asynchronous; overlap it with the next layer's dgrad by
// giving that layer another context / stream).
npcg_status npcg_allreduce_dw(npcg_context* ctx, npcg_comm* comm, npcg_dtype dtype, void* dw,
                              int64_t count) {
  if (!ctx || !comm) return NPCG_ERR_INVALID;
  return guard(ctx, [&] {
    if (dtype != NPCG_F32 && dtype != NPCG_F64) fail(NPCG_ERR_INVALID, "bad dtype");
    if (count < 0) fail(NPCG_ERR_SHAPE, "allreduce: negative count");
    if (count == 0) return;
    if (!dw) fail(NPCG_ERR_INVALID, "allreduce: null buffer");
    check(nccl().all_reduce(dw, dw, static_cast<size_t>(count),
                            dtype == NPCG_F32 ? ncclFloat32 : ncclFloat64, ncclSum, comm->comm,
                            ctx->stream),
          "ncclAllReduce");
  });
}
