// Internal shared definitions of libttround (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ttround.h"

namespace ttr {

// guards the one-time kernel attribute setup (calls may come from several host
// threads, one context each)
std::mutex& init_mutex();

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
const char* last_error();

struct Status {
  int code = TT_OK;
  bool ok() const { return code == TT_OK; }
};

#define TTR_CUDA(expr)                                                          \
  do {                                                                          \
    cudaError_t e__ = (expr);                                                   \
    if (e__ != cudaSuccess) {                                                   \
      ::ttr::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,               \
                       cudaGetErrorString(e__));                                \
      return e__ == cudaErrorMemoryAllocation ? TT_ERR_OOM : TT_ERR_CUDA;       \
    }                                                                           \
  } while (0)

#define TTR_TRY(expr)                                                           \
  do {                                                                          \
    int r__ = (expr);                                                           \
    if (r__ != TT_OK) return r__;                                               \
  } while (0)

// Launch tracing (diagnostics, TTR_TRACE=<file>): while a Tracer is installed on
// the calling thread, every launch records an event on the traced stream, so the
// time between consecutive events is the in-pipeline duration (gaps included) of
// the launch site -- aggregated per source line at the end of the call.
struct TraceRec {
  cudaEvent_t e;
  const char* file;
  int line;
};
struct Tracer {
  cudaStream_t s = nullptr;
  std::vector<TraceRec> recs;
  std::vector<cudaEvent_t> pool;   // created up front: the host stays ahead of the GPU
};
extern thread_local Tracer* t_tracer;
extern thread_local const char* t_site_file;   // set around GEMM calls (SiteGuard)
extern thread_local int t_site_line;
inline void trace_mark(const char* file, int line) {
  if (t_site_file) { file = t_site_file; line = t_site_line; }
  cudaEvent_t e;
  if (t_tracer->recs.size() < t_tracer->pool.size()) {
    e = t_tracer->pool[t_tracer->recs.size()];
  } else if (cudaEventCreate(&e) == cudaSuccess) {
    t_tracer->pool.push_back(e);
  } else {
    return;
  }
  cudaEventRecord(e, t_tracer->s);
  t_tracer->recs.push_back({e, file, line});
}

// every kernel launch of the library goes through this counter (tt_launch_count)
extern std::atomic<uint64_t> g_launches;
inline int launched_at(const char* file, int line) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (t_tracer) trace_mark(file, line);
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    set_error("kernel launch failed at %s:%d: %s", file, line, cudaGetErrorString(e));
    return TT_ERR_CUDA;
  }
  return TT_OK;
}
#define launched() ::ttr::launched_at(__FILE__, __LINE__)

// ---------------------------------------------------------------- device buffers
// Stream-ordered allocations from the device's default memory pool (kept
// cached across calls: release threshold = max).
struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { *this = std::move(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
};
int dalloc(DBuf& b, size_t ndoubles, cudaStream_t s);

struct IBuf {  // small int32 device buffer (flags, ranks)
  int* p = nullptr;
  cudaStream_t s = nullptr;
  IBuf() = default;
  IBuf(const IBuf&) = delete;
  IBuf& operator=(const IBuf&) = delete;
  ~IBuf() { if (p) cudaFreeAsync(p, s); }
};
int ialloc(IBuf& b, size_t n, cudaStream_t s);

// ---------------------------------------------------------------- context
struct NcclApi;
struct LoopGroup;   // in-process loopback communicator (comm.cu)

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t copy_stream = nullptr;   // H2D staging of host inputs
  bool own_stream = false;
  int rank = 0, world = 1;
  void* comm = nullptr;                 // ncclComm_t
  // the sharded code path (agreed validation, exchange steps) runs when there is
  // more than one rank, or when a ONE-rank NCCL communicator was asked for
  // (tt_ctx_create with world == 1 and an id: the NCCL path on a one-GPU box)
  bool multi() const { return world > 1 || comm != nullptr; }
  LoopGroup* loop = nullptr;            // loopback communicator (borrowed), else NCCL
  bool timing = false;
  double last_ms[8] = {0};
  int sm_count = 148;
  // reusable scratch for small per-call host->device uploads
  DBuf scratch;
  // split-K partials of the GEMMs
  DBuf gemm_ws;
  // per-CTA partial Grams of the fused CholeskyQR passes (cqr.cu)
  DBuf cqr_ws;
  // device status words, see linalg.cu (route flags 0/4/5, sticky 1-3, counters 8-13)
  IBuf flags;
  int nflags = 0;
  // false once the context (and its stream) is destroyed: results and sketches
  // created on it then free their memory after a device-wide synchronisation
  std::shared_ptr<std::atomic<bool>> alive = std::make_shared<std::atomic<bool>>(true);
  // lazily created second stream with its own GEMM workspace (side_ctx()),
  // for work off a sweep's critical path; shares `flags`
  std::unique_ptr<Ctx> side;
  // true while a CUDA graph is being captured on `stream` (tt_plan_create): no
  // host synchronisation, no host reads of device flags, no workspace growth
  bool capturing = false;
  // concurrent roundings on one GPU (tt_ctx_set_concurrency): persistent and
  // cooperative grids are sized to grid_sms SMs (0: all), leaving the rest to the
  // latency-bound chain of another context; chain: a highest-priority stream the
  // QR and truncation chain runs on (ordered with `stream` by events), so its
  // one-CTA / one-cluster kernels are dispatched ahead of another context's GEMM tiles
  int grid_sms = 0;
  cudaStream_t chain = nullptr;
  cudaEvent_t chain_ev[2] = {nullptr, nullptr};
};
// SMs a persistent / cooperative grid of c is sized to
inline int grid_sms(const Ctx& c) {
  return c.grid_sms > 0 && c.grid_sms < c.sm_count ? c.grid_sms : c.sm_count;
}
// The side context of c (created on first use); destroyed with c (destroy_side).
int side_ctx(Ctx& c, Ctx** out);
void destroy_side(Ctx& c);

int allreduce_sum(Ctx& c, double* buf, size_t n);   // in place, fp64 sum on c.stream
constexpr int kOpSum = 0, kOpMax = 1, kOpMin = 2;
int allreduce_i64(Ctx& c, int64_t* hostbuf, size_t n, int op);   // host words, blocking
int allreduce_sum_i64(Ctx& c, int64_t* hostbuf, size_t n);
LoopGroup* loop_create(int world);
void loop_destroy(LoopGroup* g);

// ---------------------------------------------------------------- GEMM
// C = alpha * op(A) * op(B) + beta * C, column-major, per batch entry.
struct GemmDesc {
  const double* A;
  const double* B;
  double* C;
  int M, N, K;
  int lda, ldb, ldc;
};
constexpr int kMaxGemmBatch = 64;

// Batched FP64 DMMA GEMM (all entries share ta/tb/alpha/beta).  `gate`: optional
// device flag; the launch is a no-op unless *gate == gate_val (device-side
// branching of the QR without a host round trip).
// flags: kGemmTriB -- op(B) is upper triangular (zero below the diagonal), the
// K range of a column tile stops at its last column; kGemmLower -- only the
// tiles meeting the lower triangle of C are computed (Grams feeding a Cholesky).
constexpr unsigned kGemmTriB = 1u, kGemmLower = 2u;
int gemm_impl(Ctx& c, bool ta, bool tb, const GemmDesc* d, int nbatch, double alpha,
              double beta, cudaStream_t s, const int* gate = nullptr, int gate_val = 0,
              unsigned flags = 0);
inline int gemm1_impl(Ctx& c, bool ta, bool tb, int M, int N, int K, double alpha,
                      const double* A, int lda, const double* B, int ldb, double beta,
                      double* C, int ldc, cudaStream_t s, const int* gate = nullptr,
                      int gate_val = 0, unsigned flags = 0) {
  GemmDesc d{A, B, C, M, N, K, lda, ldb, ldc};
  return gemm_impl(c, ta, tb, &d, 1, alpha, beta, s, gate, gate_val, flags);
}
// the call site of a GEMM, for launch tracing (the launches happen in gemm.cu)
struct SiteGuard {
  const char* f0;
  int l0;
  SiteGuard(const char* f, int l) : f0(t_site_file), l0(t_site_line) {
    if (!t_site_file) { t_site_file = f; t_site_line = l; }
  }
  ~SiteGuard() { t_site_file = f0; t_site_line = l0; }
};
#define gemm(...) ([&]() { ::ttr::SiteGuard g__(__FILE__, __LINE__); return ::ttr::gemm_impl(__VA_ARGS__); }())
#define gemm1(...) ([&]() { ::ttr::SiteGuard g__(__FILE__, __LINE__); return ::ttr::gemm1_impl(__VA_ARGS__); }())

// Persistent warp-specialised batched GEMM for short K (pgemm.cu): C_j = A_j B_j,
// column-major, beta = 0.  Returns 1 (nothing launched) when it does not apply.
int pgemm(Ctx& c, const GemmDesc* d, int nb, cudaStream_t s);

// ---------------------------------------------------------------- fused sweep step
// Alg. 7 lines 11 + 13 for one step in one cooperative launch (fused.cu):
// M = Q^T X (l x sumR, ld l), then X1 + xoff[j] = M(:, moff[j] ..) Y1[j] (R_j x N_j,
// ld R_j) for every summand.  Returns 1 (nothing launched) when it does not apply.
int proj_carry(Ctx& c, int64_t m, int l, int sumR, const double* Q, const double* Xn, double* M,
               int S, const double* const* Y1, const int64_t* Rj, const int64_t* Nj,
               const int64_t* moff, double* X1, const int64_t* xoff, cudaStream_t s);

// ---------------------------------------------------------------- CholeskyQR pass
// One persistent launch (cqr.cu): Q = op(A) Rinv (Rinv n x n upper, ld n; nullptr:
// Q = op(A)), written to Q (m x n, ld ldq) unless Q == nullptr, and G = Q^T Q
// (n x n, both triangles, ld n) unless G == nullptr.  op(A) = A (m x n, ld lda) or,
// trans, A^T (A n x m, ld lda).  n <= 160 (cqr_fits).  Gated like gemm().
bool cqr_fits(int64_t n);
int cqr_pass(Ctx& c, int64_t m, int n, const double* A, int64_t lda, bool trans,
             const double* Rinv, double* Q, int64_t ldq, double* G, cudaStream_t s,
             const int* gate = nullptr, int gate_val = 0);

// ---------------------------------------------------------------- sketch
int philox_fill(Ctx& c, double* out, int64_t count, uint64_t seed, uint32_t n,
                uint32_t tag, double scale, cudaStream_t s);
// the mode slab [i_lo, i_lo + I_loc) of the r0 x I_g x r1 core philox_fill would write
int philox_fill_slab(Ctx& c, double* out, int64_t r0, int64_t I_loc, int64_t r1, int64_t i_lo,
                     int64_t I_g, uint64_t seed, uint32_t n, uint32_t tag, double scale,
                     cudaStream_t s);

// ---------------------------------------------------------------- dense linalg
// Thin QR of the m x n matrix op(A) (m >= n): trans=false: A is m x n (ld lda);
// trans=true: A is n x m (ld lda) and the QR is of its transpose.
// Q: m x n (ld m).  R (optional): n x n upper (ld n).  Flags written to
// c.flags (fallback/breakdown).  Uses shifted CholeskyQR3 with a Householder
// fallback.
// dist: the m rows are this rank's share of mglob rows (mode-slab sharding): every
// Gram is all-reduced over the ranks before its Cholesky (no Householder fallback).
// robust_q (the deterministic baseline's Alg. 1 / Alg. 2 QRs of the assembled,
// typically exactly rank-deficient sum): the R-only path's four clamped passes
// and Q = op(A) R^{-1} from the last one -- A = QR to working precision, Q
// orthonormal except along numerically null directions (R's rows there are at
// the clamp level), no Householder fallback.
int qr(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, bool trans, double* Q,
       double* R, cudaStream_t s, bool dist = false, int64_t mglob = 0, bool robust_q = false);
// One-sided Jacobi SVD of the m x n (m >= n) matrix A (ld lda): AV = U Sigma
// (m x n, ld m), V (n x n, ld n), sigma (n) sorted descending.
int svd_jacobi(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
               double* V, double* sigma, cudaStream_t s);
// One-sided Jacobi of the m x n (m >= n, m <= 256, m n <= 26624) matrix A without
// forming V: AV = U Sigma (m x n, ld m, sorted) and sigma.  svd_nov_fits() tells
// whether the shape is supported.
int svd_nov(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
            double* sigma, cudaStream_t s);
bool svd_nov_fits(int64_t m, int64_t n);
// The same one-sided Jacobi as svd_jacobi on a cooperative grid (one warp per
// pair of a round, negligible columns not rotated), for m n > 26624; V ==
// nullptr: V is not formed.
int svd_jacobi_grid(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
                    double* V, double* sigma, cudaStream_t s);
// B(:, c) = AV(:, c) / sigma_c^(halfpow/2), c < k; 0 where sigma_c <= rel_thr sigma_0
// (negligible / pseudo-inverse cutoff)
int scale_by_inv_sigma(Ctx& c, const double* AV, int64_t m, int64_t k, const double* sigma,
                       double* B, int halfpow, double rel_thr, cudaStream_t s);
// Q of an m x n matrix whose columns are already close to orthonormal: one
// CholeskyQR pass (n <= 160; else qr())
int cholesky(Ctx& c, int64_t n, const double* G, int64_t m, int shifted, double* Rinv, double* L,
             cudaStream_t s);
int qr_near_orthonormal(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* Q,
                        cudaStream_t s);
// columns c of the m x n matrix A with sigma_c <= rel_thr sigma_0 set to e_c
int unit_cut_columns(Ctx& c, double* A, int64_t m, int64_t n, const double* sigma,
                     double rel_thr, cudaStream_t s);
// Q(:, c) negated where Q(:, c) . ref(:, c) < 0 (m x n, ld m)
int align_column_signs(Ctx& c, double* Q, const double* ref, int64_t m, int64_t n,
                       cudaStream_t s);
// k = eps-rank of sigma (n values, descending) given absolute eps and cap rmax
// (0 = none), written to dst (device int).
int eps_rank_dev(Ctx& c, const double* sigma, int n, const double* eps_dev, double eps_host,
                 int rmax, int* dst, cudaStream_t s);
// *out = sum x_i^2 in a fixed order (partial: 256 doubles of scratch)
int sumsq_det(Ctx& c, const double* x, int64_t n, double* out, double* partial,
              cudaStream_t s);
// x <- 2^shift x (exact)
int scale_pow2(Ctx& c, double* x, int64_t n, int shift, cudaStream_t s);
// x <- 2^{-e} x, e = floor(log2 ||x||_F) computed and stored (*e_out) on the device
int normalize_pow2(Ctx& c, double* x, int64_t n, double* ssq, double* partial, int* e_out,
                   cudaStream_t s);
// x <- 2^{sign * *e} x (device exponent)
int scale_pow2_dev(Ctx& c, double* x, int64_t n, const int* e, int sign, cudaStream_t s);
// out = ||x||_F (device scalar)
int fro_norm(Ctx& c, const double* x, int64_t n, double* out, cudaStream_t s);
// dst (cols x rows, ld ldd) = src^T (src rows x cols, ld lds)
int transpose(Ctx& c, const double* src, int64_t rows, int64_t cols, int64_t lds,
              double* dst, int64_t ldd, cudaStream_t s);
int fill_zero(Ctx& c, double* p, int64_t n, cudaStream_t s);
// TT-GMRES helpers (NEXT-4): y(a,i,b) = dg[i] x(a,i,b) for an r0 x I x r1 core;
// y = a x; M += identity / diag / dense factor; Minv = M^{-1} (M SPD, n x n)
int scale_mode2(Ctx& c, const double* x, int64_t r0, int64_t I, int64_t r1, const double* dg,
                double* y, cudaStream_t s);
int scale_copy(Ctx& c, const double* x, int64_t n, double a, double* y, cudaStream_t s);
int add_factor(Ctx& c, double* M, int n, int kind, const double* F, cudaStream_t s);
int spd_inverse(Ctx& c, const double* M, int n, double* Minv, cudaStream_t s);
// diagonal of the n x n matrix p (ld n) set to 1 (other entries untouched)
int set_identity(Ctx& c, double* p, int64_t n, cudaStream_t s);

}  // namespace ttr
