// NCCL binding for the one exchange step of the sharded sweep:
// an fp64-sum allreduce of the partial sketched core Y_n (and of the last core)
// over NVLink/NVSwitch.  libnccl is resolved at run time with dlopen so the
// process uses the NCCL that torch.distributed already loaded (no second copy).
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "common.cuh"

namespace ttr {

struct NcclApi {
  bool loaded = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;
static std::mutex g_nccl_mu;

static int nccl_load() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.loaded) return TT_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error("NCCL not found (dlopen libnccl.so.2): %s", dlerror());
    return TT_ERR_NCCL;
  }
#define LOAD(field, name)                                                   \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name));  \
  if (!g_nccl.field) {                                                      \
    set_error("NCCL symbol %s missing", name);                              \
    return TT_ERR_NCCL;                                                     \
  }
  LOAD(getUniqueId, "ncclGetUniqueId");
  LOAD(commInitRank, "ncclCommInitRank");
  LOAD(allReduce, "ncclAllReduce");
  LOAD(commDestroy, "ncclCommDestroy");
  LOAD(getErrorString, "ncclGetErrorString");
#undef LOAD
  g_nccl.loaded = true;
  return TT_OK;
}

#define TTR_NCCL(expr)                                                               \
  do {                                                                               \
    ncclResult_t r__ = (expr);                                                       \
    if (r__ != ncclSuccess) {                                                        \
      set_error("%s failed: %s", #expr, g_nccl.getErrorString(r__));                 \
      return TT_ERR_NCCL;                                                            \
    }                                                                                \
  } while (0)

int nccl_unique_id(uint8_t id[128]) {
  TTR_TRY(nccl_load());
  ncclUniqueId u;
  TTR_NCCL(g_nccl.getUniqueId(&u));
  static_assert(sizeof(u.internal) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, u.internal, 128);
  return TT_OK;
}

int nccl_comm_create(Ctx& c, const uint8_t* id, int rank, int world) {
  TTR_TRY(nccl_load());
  ncclUniqueId u;
  memcpy(u.internal, id, 128);
  ncclComm_t comm = nullptr;
  TTR_NCCL(g_nccl.commInitRank(&comm, world, u, rank));
  c.comm = comm;
  return TT_OK;
}

int nccl_comm_destroy(Ctx& c) {
  if (c.comm && g_nccl.loaded) g_nccl.commDestroy(static_cast<ncclComm_t>(c.comm));
  c.comm = nullptr;
  return TT_OK;
}

int allreduce_sum(Ctx& c, double* buf, size_t n) {
  if (c.world <= 1 || n == 0) return TT_OK;
  TTR_NCCL(g_nccl.allReduce(buf, buf, n, ncclFloat64, ncclSum,
                            static_cast<ncclComm_t>(c.comm), c.stream));
  return TT_OK;
}

int allreduce_sum_i64(Ctx& c, int64_t* hostbuf, size_t n) {
  if (c.world <= 1 || n == 0) return TT_OK;
  int64_t* d = nullptr;
  TTR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), n * sizeof(int64_t), c.stream));
  TTR_CUDA(cudaMemcpyAsync(d, hostbuf, n * sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
  TTR_NCCL(g_nccl.allReduce(d, d, n, ncclInt64, ncclSum, static_cast<ncclComm_t>(c.comm),
                            c.stream));
  TTR_CUDA(cudaMemcpyAsync(hostbuf, d, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  TTR_CUDA(cudaFreeAsync(d, c.stream));
  TTR_CUDA(cudaStreamSynchronize(c.stream));
  return TT_OK;
}

}  // namespace ttr
