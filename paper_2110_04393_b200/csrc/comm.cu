// Communicators of the sharded path: the one exchange step of the
// sweep is an fp64-sum allreduce of the partial sketched core Y_n (and of the
// last core).
//  * NCCL over NVLink/NVSwitch, one process per GPU.  libnccl is resolved at run
//    time with dlopen so the process uses the NCCL torch.distributed loaded.
//  * Loopback (tt_loopback_create): `world` contexts in ONE process, driven from
//    host threads, on one device.  A rank's allreduce copies its buffer into its
//    own device slot, synchronises its stream and meets the other ranks at a host
//    barrier; each rank then sums the slots in rank order 0..world-1 (identical
//    bits on every rank) and meets them at a second barrier before the slots are
//    reused.  No kernel ever waits on another rank's kernel (the barriers are on
//    the host, after stream synchronisation), so the ranks may run in any order
//    on the GPU.  It exists so the sharded code path of the library can run and
//    be tested where there is one GPU; it is not a performance path.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
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

// One-rank NCCL communicator built and used the way the sharded path uses it
// (dlopen'd libnccl, ncclCommInitRank, fp64-sum and int64 allreduce on the
// context's stream).  With one rank a sum allreduce must return its input: the
// largest deviation is reported.  Runs on a box with one GPU, where world > 1
// cannot be formed.
int nccl_selftest(Ctx& c, size_t n, double* max_abs_diff) {
  TTR_TRY(nccl_load());
  ncclUniqueId u;
  TTR_NCCL(g_nccl.getUniqueId(&u));
  ncclComm_t comm = nullptr;
  TTR_NCCL(g_nccl.commInitRank(&comm, 1, u, 0));
  std::vector<double> h(n), back(n);
  for (size_t i = 0; i < n; ++i) h[i] = 1.0 / double(i + 1) - 0.5 * double(i % 7);
  double* d = nullptr;
  int rc = TT_OK;
  do {
    if (cudaMalloc(reinterpret_cast<void**>(&d), std::max<size_t>(n, 1) * sizeof(double)) !=
        cudaSuccess) {
      set_error("nccl_selftest: cudaMalloc failed");
      rc = TT_ERR_CUDA;
      break;
    }
    cudaMemcpyAsync(d, h.data(), n * sizeof(double), cudaMemcpyHostToDevice, c.stream);
    ncclResult_t r = g_nccl.allReduce(d, d, n, ncclFloat64, ncclSum, comm, c.stream);
    if (r != ncclSuccess) {
      set_error("ncclAllReduce (fp64 sum) failed: %s", g_nccl.getErrorString(r));
      rc = TT_ERR_NCCL;
      break;
    }
    cudaMemcpyAsync(back.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, c.stream);
    int64_t w[2] = {int64_t(n), -3};
    int64_t* dw = reinterpret_cast<int64_t*>(d);
    if (n >= 2) {
      cudaMemcpyAsync(dw, w, sizeof(w), cudaMemcpyHostToDevice, c.stream);
      r = g_nccl.allReduce(dw, dw, 2, ncclInt64, ncclMax, comm, c.stream);
      if (r != ncclSuccess) {
        set_error("ncclAllReduce (int64 max) failed: %s", g_nccl.getErrorString(r));
        rc = TT_ERR_NCCL;
        break;
      }
      cudaMemcpyAsync(w, dw, sizeof(w), cudaMemcpyDeviceToHost, c.stream);
    }
    if (cudaStreamSynchronize(c.stream) != cudaSuccess) {
      set_error("nccl_selftest: stream failed: %s", cudaGetErrorString(cudaGetLastError()));
      rc = TT_ERR_CUDA;
      break;
    }
    double m = 0.0;
    for (size_t i = 0; i < n; ++i) m = std::max(m, std::fabs(back[i] - h[i]));
    if (w[0] != int64_t(n) || w[1] != -3) m = std::max(m, 1.0);
    *max_abs_diff = m;
  } while (0);
  if (d) cudaFree(d);
  g_nccl.commDestroy(comm);
  return rc;
}

// ------------------------------------------------------------------ loopback
struct LoopGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<double*> slot;          // device slot per rank
  std::vector<size_t> cap;            // doubles
  std::vector<std::vector<int64_t>> hb;   // host words per rank
  // host barrier with a timeout (a rank that failed outside a collective must
  // not hang the others forever)
  int barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return TT_OK;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; })) {
      set_error("loopback communicator: barrier timed out (another rank did not arrive)");
      return TT_ERR_NCCL;
    }
    return TT_OK;
  }
  ~LoopGroup() {
    for (double* p : slot)
      if (p) cudaFree(p);
  }
};

LoopGroup* loop_create(int world) {
  LoopGroup* g = new LoopGroup;
  g->world = world;
  g->slot.assign(world, nullptr);
  g->cap.assign(world, 0);
  g->hb.assign(world, {});
  return g;
}
void loop_destroy(LoopGroup* g) { delete g; }

namespace {
constexpr int kMaxLoop = 16;
struct SlotPtrs {
  const double* p[kMaxLoop];
};
__global__ void sum_slots_kernel(SlotPtrs s, int world, size_t n, double* __restrict__ out) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    double v = s.p[0][i];
    for (int r = 1; r < world; ++r) v += s.p[r][i];
    out[i] = v;
  }
}
}  // namespace

static int loop_allreduce(Ctx& c, double* buf, size_t n) {
  LoopGroup& g = *c.loop;
  if (g.world > kMaxLoop) {
    set_error("loopback communicator supports at most %d ranks", kMaxLoop);
    return TT_ERR_ARG;
  }
  if (g.cap[c.rank] < n) {   // only this rank touches its own slot here
    TTR_CUDA(cudaStreamSynchronize(c.stream));
    if (g.slot[c.rank]) cudaFree(g.slot[c.rank]);
    g.slot[c.rank] = nullptr;
    g.cap[c.rank] = 0;
    TTR_CUDA(cudaMalloc(&g.slot[c.rank], n * sizeof(double)));
    g.cap[c.rank] = n;
  }
  TTR_CUDA(cudaMemcpyAsync(g.slot[c.rank], buf, n * sizeof(double), cudaMemcpyDeviceToDevice,
                           c.stream));
  TTR_CUDA(cudaStreamSynchronize(c.stream));
  TTR_TRY(g.barrier());            // every slot holds its rank's partial
  SlotPtrs sp{};
  for (int r = 0; r < g.world; ++r) sp.p[r] = g.slot[r];
  const int blocks = int(std::min<size_t>((n + 255) / 256, size_t(c.sm_count) * 8));
  sum_slots_kernel<<<std::max(1, blocks), 256, 0, c.stream>>>(sp, g.world, n, buf);
  TTR_TRY(launched());
  TTR_CUDA(cudaStreamSynchronize(c.stream));
  return g.barrier();              // nobody rewrites a slot before all have read it
}

static int loop_allreduce_i64(Ctx& c, int64_t* h, size_t n, int op) {
  LoopGroup& g = *c.loop;
  g.hb[c.rank].assign(h, h + n);
  TTR_TRY(g.barrier());
  for (size_t i = 0; i < n; ++i) {
    int64_t v = g.hb[0][i];
    for (int r = 1; r < g.world; ++r) {
      const int64_t x = g.hb[r][i];
      v = op == kOpSum ? v + x : (op == kOpMax ? std::max(v, x) : std::min(v, x));
    }
    h[i] = v;
  }
  return g.barrier();
}

// ------------------------------------------------------------------ dispatch
int allreduce_sum(Ctx& c, double* buf, size_t n) {
  if (!c.multi() || n == 0) return TT_OK;
  if (c.loop) return loop_allreduce(c, buf, n);
  TTR_NCCL(g_nccl.allReduce(buf, buf, n, ncclFloat64, ncclSum,
                            static_cast<ncclComm_t>(c.comm), c.stream));
  return TT_OK;
}

int allreduce_i64(Ctx& c, int64_t* hostbuf, size_t n, int op) {
  if (!c.multi() || n == 0) return TT_OK;
  if (c.loop) return loop_allreduce_i64(c, hostbuf, n, op);
  int64_t* d = nullptr;
  TTR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), n * sizeof(int64_t), c.stream));
  TTR_CUDA(cudaMemcpyAsync(d, hostbuf, n * sizeof(int64_t), cudaMemcpyHostToDevice, c.stream));
  const ncclRedOp_t nop = op == kOpSum ? ncclSum : (op == kOpMax ? ncclMax : ncclMin);
  TTR_NCCL(g_nccl.allReduce(d, d, n, ncclInt64, nop, static_cast<ncclComm_t>(c.comm),
                            c.stream));
  TTR_CUDA(cudaMemcpyAsync(hostbuf, d, n * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  TTR_CUDA(cudaFreeAsync(d, c.stream));
  TTR_CUDA(cudaStreamSynchronize(c.stream));
  return TT_OK;
}

int allreduce_sum_i64(Ctx& c, int64_t* hostbuf, size_t n) {
  return allreduce_i64(c, hostbuf, n, kOpSum);
}

}  // namespace ttr
