// One-sided (Hestenes) Jacobi SVD of the small square factor of the truncation
// (P:667-670 via Alg. 2 lines 3-10 mirrored, R3): [U, Sigma, V] =
// svd(R^T) with R the ell x ell triangular factor of qr(H(X_n)^T).  V is never
// formed: the truncation needs only U Sigma.
//
// Layout (one CTA): the m x n matrix W lives in shared memory, column-major with
// ld = 8*RPT (rows m..ld-1 are zero).  A round of the round-robin ("circle")
// ordering pairs all columns disjointly; every pair is handled by a group of
// 8 threads at the same time (4n threads for n columns).  Thread t of a group
// owns the row pairs {16 s + 2 t, 16 s + 2 t + 1}, so a group reads one column
// as 128-byte double2 segments: conflict-free whatever the pair.
//
// Convergence (LAPACK dgesvj-style): a pair is rotated iff its cosine exceeds
// 2 m u AND both columns are above the negligible level 16 m u ||A||_F.  Columns
// at rounding level relative to ||A|| cannot be orthogonalised (every rotation
// against a large column re-randomises them) and contribute < 16 m u ||A|| to
// the tensor; without this test the sweep never stops on the numerically
// rank-deficient bond matrices of config 5.
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace ttr {

namespace {

constexpr int kGroup = 8;   // threads per column pair

// Register cap: a CTA of W warps puts ceil(W/4) warps on one SM sub-partition,
// whose register file holds 16K registers -> <= 96 registers at 18-20 warps.
template <int RPT>   // rows per thread (even); m <= 8 * RPT
__global__ void __launch_bounds__(32 * RPT) __maxnreg__(RPT >= 18 ? 96 : 128)
    jacobi_rr_kernel(const double* __restrict__ A, int64_t lda, int m, int n,
                     double* __restrict__ AV, double* __restrict__ sigma, int max_sweeps,
                     int* __restrict__ flags) {
  constexpr int LDW = 8 * RPT;
  constexpr int S2 = RPT / 2;   // double2 segments per thread and column
  extern __shared__ __align__(16) double W[];   // n x LDW
  __shared__ double red[32];
  __shared__ double nrm[256];
  __shared__ double cn[256];   // squared column norms
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int grp = tid / kGroup, t8 = tid % kGroup;

  double part = 0.0;
  for (int e = tid; e < n * LDW; e += nt) {
    const int i = e % LDW, j = e / LDW;
    const double v = (i < m) ? A[i + int64_t(j) * lda] : 0.0;
    W[e] = v;
    part = fma(v, v, part);
  }
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) red[warp] = part;
  __syncthreads();
  double fro2 = 0.0;
  for (int w = 0; w < (nt + 31) / 32; ++w) fro2 += red[w];

  const double u = 0x1p-53;
  const double tol = 2.0 * m * u;                       // cosine threshold
  const double neg = 16.0 * m * u;
  const double small = neg * neg * fro2;                // negligible squared norm
  const int np = (n + 1) & ~1;
  const int half = np / 2;
  const int nw = nt / 32;

  int sweep = 0;
  bool conv = false;
  for (; sweep < max_sweeps; ++sweep) {
    // squared column norms, recomputed every sweep and updated analytically
    // after each rotation (alpha' = alpha - t gamma, beta' = beta + t gamma), so
    // a round only forms the cross products gamma; a sweep without rotations
    // (the convergence test) sees exact norms
    for (int j = warp; j < n; j += nw) {
      double s2 = 0.0;
      for (int i = lane; i < m; i += 32) s2 = fma(W[i + j * LDW], W[i + j * LDW], s2);
      for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      if (lane == 0) cn[j] = s2;
    }
    int rot = 0;
    // circle ordering: group grp pairs (p, q) = (0 or 1 + (grp-1+r) mod (np-1),
    // 1 + (np-2-grp+r) mod (np-1)), advanced incrementally
    int pp = grp - 1, qq = np - 2 - grp;
    for (int r = 0; r < np - 1; ++r) {
      __syncthreads();
      const int p0 = (grp == 0) ? 0 : pp + 1, q0 = qq + 1;
      pp = (pp + 1 == np - 1) ? 0 : pp + 1;
      qq = (qq + 1 == np - 1) ? 0 : qq + 1;
      // every thread takes part in the shuffles (full mask: no divergence
      // checks); groups without a pair work on column 0 and write nothing
      const bool act = grp < half && max(p0, q0) < n;
      const int p = act ? min(p0, q0) : 0, q = act ? max(p0, q0) : 0;
      double2* wp = reinterpret_cast<double2*>(W + p * LDW) + t8;
      double2* wq = reinterpret_cast<double2*>(W + q * LDW) + t8;
      double2 x[S2], y[S2];
      double ga = 0.0;
#pragma unroll
      for (int s = 0; s < S2; ++s) {
        x[s] = wp[s * kGroup];
        y[s] = wq[s * kGroup];
        ga = fma(x[s].x, y[s].x, fma(x[s].y, y[s].y, ga));
      }
#pragma unroll
      for (int o = 4; o; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
      const double al = cn[p], be = cn[q];
      if (!act || !(fmin(al, be) > small) || !(ga * ga > tol * tol * (al * be))) continue;
      // angle as in the cluster kernel: MUFU-approximate t, Newton-exact cosine
      const double d = be - al, e = 2.0 * ga;
      const double r2 = fma(d, d, e * e);
      double rs, rc, cs;
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(r2));
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(fabs(d) + r2 * rs));
      const double tt = copysign(1.0, d) * e * rc;
      const double qq1 = fma(tt, tt, 1.0);
      asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(cs) : "d"(qq1));
      cs = cs * fma(-0.5 * qq1 * cs, cs, 1.5);
      cs = cs * fma(-0.5 * qq1 * cs, cs, 1.5);
      const double sn = cs * tt;
#pragma unroll
      for (int s = 0; s < S2; ++s) {
        wp[s * kGroup] = make_double2(fma(cs, x[s].x, -sn * y[s].x), fma(cs, x[s].y, -sn * y[s].y));
        wq[s * kGroup] = make_double2(fma(sn, x[s].x, cs * y[s].x), fma(sn, x[s].y, cs * y[s].y));
      }
      if (t8 == 0) {
        cn[p] = al - tt * ga;
        cn[q] = be + tt * ga;
      }
      rot = 1;
    }
    if (!__syncthreads_or(rot)) {
      conv = true;
      break;
    }
  }
  if (tid == 0) {
    if (!conv) atomicOr(&flags[3], 2);
    flags[12] += conv ? sweep + 1 : sweep;   // Jacobi sweeps (counter)
    flags[13] += 1;                          // Jacobi calls (counter)
  }
  __syncthreads();
  // sigma_j = ||w_j||, then columns sorted by descending norm (ties by index)
  for (int j = warp; j < n; j += nw) {
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) s2 = fma(W[i + j * LDW], W[i + j * LDW], s2);
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) nrm[j] = sqrt(s2);
  }
  __syncthreads();
  for (int j = warp; j < n; j += nw) {
    const double sj = nrm[j];
    int rank = 0;
    for (int k = lane; k < n; k += 32) {
      const double sk = nrm[k];
      rank += (sk > sj) || (sk == sj && k < j);
    }
    for (int o = 16; o; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    for (int i = lane; i < m; i += 32) AV[i + int64_t(rank) * m] = W[i + j * LDW];
    if (lane == 0) sigma[rank] = sj;
  }
}

template <int RPT>
int launch_rr(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
              double* sigma, cudaStream_t s) {
  static std::atomic<bool> attr[64];
  const size_t shm = size_t(n) * 8 * RPT * sizeof(double);
  std::unique_lock<std::mutex> init_lock(init_mutex(), std::defer_lock);
  if (!attr[c.device & 63]) init_lock.lock();
  if (!attr[c.device & 63]) {
    TTR_CUDA(cudaFuncSetAttribute(jacobi_rr_kernel<RPT>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, 222 * 1024));
    attr[c.device & 63] = true;
  }
  const int half = int((n + 1) / 2);
  const int threads = std::max(32, ((half * kGroup + 31) / 32) * 32);
  jacobi_rr_kernel<RPT><<<1, threads, shm, s>>>(A, lda, int(m), int(n), AV, sigma, 40,
                                                 c.flags.p);
  const int rc = launched();
  if (rc != TT_OK) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, jacobi_rr_kernel<RPT>);
    set_error("jacobi_rr_kernel<%d> launch failed (%d threads, %zu B smem; kernel: %d regs, "
              "max %d threads, %zu B static smem, max dyn %d B): %s", RPT, threads, shm,
              fa.numRegs, fa.maxThreadsPerBlock, fa.sharedSizeBytes,
              fa.maxDynamicSharedSizeBytes, last_error());
  }
  return rc;
}

}  // namespace

// m <= 160: W (n x 8 RPT doubles) fits in shared memory and 8 ceil(n/2) <= 32 RPT
// threads (the launch bound) for every n <= m
bool svd_nov_fits(int64_t m, int64_t n) { return n >= 1 && m >= n && m <= 160; }
bool svd_cluster_fits(int64_t m, int64_t n);
int svd_nov_cluster(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
                    double* sigma, cudaStream_t s);

int svd_nov(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
            double* sigma, cudaStream_t s) {
  if (!svd_nov_fits(m, n)) {
    set_error("svd_nov: unsupported shape m=%lld n=%lld", (long long)m, (long long)n);
    return TT_ERR_ARG;
  }
  static const char* force = getenv("TTR_JACOBI");   // diagnostics: "cta" = single-CTA kernel
  const bool cta = force && strcmp(force, "cta") == 0;
  if (!cta && svd_cluster_fits(m, n)) return svd_nov_cluster(c, m, n, A, lda, AV, sigma, s);
  if (m <= 16) return launch_rr<2>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 32) return launch_rr<4>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 64) return launch_rr<8>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 96) return launch_rr<12>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 128) return launch_rr<16>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 144) return launch_rr<18>(c, m, n, A, lda, AV, sigma, s);
  return launch_rr<20>(c, m, n, A, lda, AV, sigma, s);
}

}  // namespace ttr

// ============================================================================
// Cluster version for 64 <= n <= 160: the same one-sided Jacobi (same rotation
// formulas, thresholds and convergence test) on a cluster of 8 CTAs, over
// UNITS of four columns (block-cyclic ordering).
//
// Units u = (4u .. 4u+3) take part in a circle ordering; a "group" (one warp)
// holds a top and a bottom unit (8 columns in shared memory).  Round 0 of a
// sweep first rotates the 12 intra-unit pairs (3 sub-rounds of 4 disjoint
// pairs); every round then rotates the 16 cross pairs in 4 sub-rounds
// (t_i, b_{(i+s) mod 4}), one pair per 8-lane subgroup (rows t + 8 s), with only
// __syncwarp between sub-rounds.  The last sub-round writes its rotated columns
// straight into the slots of the groups that own the units next round (top row
// shifts right, bottom row left, unit 0 fixed): the move is the write-back, and
// only the units crossing a CTA boundary go through distributed shared memory.
// One cluster barrier per round: 35 per sweep for n = 144 instead of 143.
// ============================================================================
namespace ttr {
namespace {

constexpr int kCl = 8;          // CTAs per cluster
constexpr int kUw = 4;          // columns per unit
constexpr int kGpc = 3;         // groups (warps) per CTA: n <= 160 -> <= 20 groups
constexpr int kG8 = 8;          // threads per pair
constexpr int kRps = 20;        // rows per thread (m <= 160)
constexpr int kRows = kG8 * kRps;

struct JcShared {
  alignas(16) double slot[3][kGpc][2 * kUw][kRows];   // [buffer][group][t0..t3, b0..b3][rows]
  double alpha[3][kGpc][2 * kUw];         // squared norms travelling with the columns
  int col[3][kGpc][2 * kUw];              // column ids travelling with the columns
  double norms[kCl * kGpc * 2 * kUw];     // final column norms (all columns, by id)
  double red[8];
  int rot;
  // point-to-point round hand-off (P2P variant): ready[b][g] completes when both
  // units of group g's next round have landed in buffer b (2 arrivals, one per
  // source group); freeb[b][g] completes when both groups that group g writes
  // into have finished reading their buffer b
  alignas(8) unsigned long long ready[3][kGpc];
  alignas(8) unsigned long long freeb[3][kGpc];
};

constexpr int kJcThreads = kGpc * 32;

__device__ __forceinline__ uint32_t jc_saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// arrive (release, cluster scope) on the mbarrier at local address `la` of CTA `rank`
__device__ __forceinline__ void jc_remote_arrive(uint32_t la, uint32_t rank) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(ra)
               : "memory");
}
__device__ __forceinline__ void jc_wait(uint32_t la, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "JCW_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra JCW_%=;\n"
      "}\n" ::"r"(la),
      "r"(parity)
      : "memory");
}

// rotate the pair (X, Y) held by this 8-lane subgroup (ids cx, cy, squared
// norms ax, ay); p = min(id) is rotated as column p of the single-CTA kernel.
// Rows are held as double2 (rows 2 t + 16 s, +1).  The angle
//   t = sign(d) e / (|d| + sqrt(d^2 + e^2)),  d = a_q - a_p, e = 2 gamma
// (= sign(zeta)/(|zeta| + sqrt(1 + zeta^2)), zeta = d/e) is computed in fp32 after
// an exact power-of-two scaling: its error only changes how much of gamma one
// rotation removes; the rotation stays orthogonal to working precision because
// cs = rsqrt(1 + t^2) and sn = cs t are formed in fp64.
constexpr int kR2 = kRps / 2;
__device__ __forceinline__ bool jc_rotate(double2 (&x)[kR2], double2 (&y)[kR2], int cx, int cy,
                                          double& ax, double& ay, int n, double small, double tol) {
  double ga0 = 0.0, ga1 = 0.0, ga2 = 0.0, ga3 = 0.0;   // 4 short FMA chains
#pragma unroll
  for (int s = 0; s < kR2; s += 2) {
    ga0 = fma(x[s].x, y[s].x, ga0);
    ga1 = fma(x[s].y, y[s].y, ga1);
    ga2 = fma(x[s + 1].x, y[s + 1].x, ga2);
    ga3 = fma(x[s + 1].y, y[s + 1].y, ga3);
  }
  double ga = (ga0 + ga1) + (ga2 + ga3);
#pragma unroll
  for (int o = 4; o; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
  const bool swp = cx > cy;
  const double ap = swp ? ay : ax, aq = swp ? ax : ay;
  // |cos| > tol  <=>  gamma^2 > tol^2 a_p a_q (no sqrt on the critical path)
  if (!(cx < n && cy < n && fmin(ap, aq) > small && ga * ga > tol * tol * (ap * aq))) return false;
  const double d = aq - ap, e = 2.0 * ga;
  // t from MUFU approximations (rel. error ~1e-5 at most changes how much of gamma
  // this rotation removes); cs = 1/sqrt(1 + t^2) is then made exact by two Newton steps
  const double r2 = fma(d, d, e * e);
  double rs, rc;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rs) : "d"(r2));
  const double den = fabs(d) + r2 * rs;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(den));
  double tt = copysign(1.0, d) * e * rc;
  const double q = fma(tt, tt, 1.0);
  double cs;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(cs) : "d"(q));
  cs = cs * fma(-0.5 * q * cs, cs, 1.5);
  cs = cs * fma(-0.5 * q * cs, cs, 1.5);
  double sn = cs * tt;
  if (swp) { sn = -sn; tt = -tt; }
#pragma unroll
  for (int s = 0; s < kR2; ++s) {
    const double2 xs = x[s], ys = y[s];
    x[s] = make_double2(fma(cs, xs.x, -sn * ys.x), fma(cs, xs.y, -sn * ys.y));
    y[s] = make_double2(fma(sn, xs.x, cs * ys.x), fma(sn, xs.y, cs * ys.y));
  }
  ax -= tt * ga;
  ay += tt * ga;
  return true;
}

// P2P = true: instead of one cluster barrier per round, a group waits only for
// the two groups whose units it receives (ready) and, before writing into its two
// destination groups' next buffer, for those groups to have released it (freeb);
// one cluster barrier per sweep remains (the convergence vote).
template <bool P2P>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kJcThreads)
    jacobi_cluster_kernel(const double* __restrict__ A, int64_t lda, int m, int n, int gpc,
                          double* __restrict__ AV, double* __restrict__ sigma, int max_sweeps,
                          int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char jc_raw[];
  JcShared& sh = *reinterpret_cast<JcShared*>(jc_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int crank = int(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lg = warp, rho = lane >> 3, t8 = lane & 7;    // group, pair slot, thread in pair
  const int U = (n + kUw - 1) / kUw, UP = U + (U & 1), halfU = UP / 2;
  const int g = crank * gpc + lg;
  const bool live = lg < gpc && g < halfU;
  const int lgc = live ? lg : 0;

  // round 0: group g holds top unit (g == 0 ? 0 : g) and bottom unit UP - 1 - g
  {
    const int ut = live ? g : -1, ub = live ? UP - 1 - g : -1;
    for (int c8 = 0; c8 < 2 * kUw; ++c8) {
      const int unit = c8 < kUw ? ut : ub;
      const int c0 = unit < 0 ? n : kUw * unit + (c8 % kUw);
      const int cid = c0 < n ? c0 : n;
      double* sl = sh.slot[0][lg][c8];
      for (int i = lane; i < kRows; i += 32)
        sl[i] = (cid < n && i < m) ? A[i + int64_t(cid) * lda] : 0.0;
      if (lane == 0) {
        sh.col[0][lg][c8] = cid;
        sh.alpha[0][lg][c8] = 0.0;
      }
    }
  }
  __syncthreads();
  double part = 0.0;
  for (int c8 = 0; c8 < 2 * kUw; ++c8)
    for (int i = lane; i < kRows; i += 32) {
      const double v = sh.slot[0][lg][c8][i];
      part = fma(v, v, part);
    }
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) sh.red[warp] = part;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kGpc; ++w) s += sh.red[w];
    for (int r = 0; r < kCl; ++r) cl.map_shared_rank(&sh, r)->norms[crank] = s;   // scratch
    if (P2P) {
      for (int b = 0; b < 3; ++b)
        for (int q = 0; q < kGpc; ++q) {
          asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(jc_saddr(&sh.ready[b][q])),
                       "r"(2));
          asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(jc_saddr(&sh.freeb[b][q])),
                       "r"(2));
        }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
  }
  cl.sync();
  double fro2 = 0.0;
  for (int r = 0; r < kCl; ++r) fro2 += sh.norms[r];
  cl.sync();

  const double u = 0x1p-53;
  const double tol = 2.0 * m * u;
  const double negl = 16.0 * m * u;
  const double small = negl * negl * fro2;

  // destinations of this group's units after a round (fixed for the run):
  // top:    g == 0 -> (0, top); g < halfU-1 -> (g+1, top); g == halfU-1 -> (g, bottom)
  // bottom: g == 0 -> (1, top); g >= 1 -> (g-1, bottom)
  const int gt = (g == 0) ? 0 : (g < halfU - 1 ? g + 1 : g);
  const int wt = (g == 0 || g < halfU - 1) ? 0 : kUw;
  const int gb = (g == 0) ? 1 : g - 1, wb = (g == 0) ? 0 : kUw;
  JcShared* sht = (gt / gpc == crank) ? &sh : cl.map_shared_rank(&sh, gt / gpc);
  JcShared* shb = (gb / gpc == crank) ? &sh : cl.map_shared_rank(&sh, gb / gpc);
  const int lt = gt % gpc, lb = gb % gpc;
  // groups whose units group g receives: its top slot from max(g-1, 0), its
  // bottom slot from g+1 (or itself, the last group)
  const int st = g > 0 ? g - 1 : 0, sb = (g == halfU - 1) ? g : g + 1;
  uint32_t round_g = 0;   // rounds done so far (all sweeps): ring position / phase

  // rotate slots (cx, cy) of the current buffer in place
  auto in_place = [&](double (*sl)[kRows], double* al, const int* cid, int cx, int cy,
                      int& rot) {
    double2 x[kR2], y[kR2];
    const double2* px = reinterpret_cast<const double2*>(sl[cx]) + t8;
    const double2* py = reinterpret_cast<const double2*>(sl[cy]) + t8;
#pragma unroll
    for (int s = 0; s < kR2; ++s) {
      x[s] = px[kG8 * s];
      y[s] = py[kG8 * s];
    }
    double ax = al[cx], ay = al[cy];
    if (live && jc_rotate(x, y, cid[cx], cid[cy], ax, ay, n, small, tol)) {
      rot = 1;
      double2* wx = reinterpret_cast<double2*>(sl[cx]) + t8;
      double2* wy = reinterpret_cast<double2*>(sl[cy]) + t8;
#pragma unroll
      for (int s = 0; s < kR2; ++s) {
        wx[kG8 * s] = x[s];
        wy[kG8 * s] = y[s];
      }
      if (t8 == 0) { al[cx] = ax; al[cy] = ay; }
    }
    __syncwarp();
  };

  int buf = 0, sweep = 0;
  bool conv = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) sh.rot = 0;
    int rot = 0;
    for (int r = 0; r < UP - 1; ++r) {
      if (P2P && live && round_g > 0)   // this round's units have landed in buffer buf
        jc_wait(jc_saddr(&sh.ready[buf][lg]), ((round_g - 1) / 3) & 1);
      double (*sl)[kRows] = sh.slot[buf][lgc];
      double* al = sh.alpha[buf][lgc];
      const int* cid = sh.col[buf][lgc];
      if (r == 0) {
        // exact squared norms (subgroup rho: columns rho and 4 + rho) ...
        for (int c = rho; c < 2 * kUw; c += kUw) {
          double a2 = 0.0;
#pragma unroll
          for (int s = 0; s < kRps; ++s) a2 = fma(sl[c][t8 + kG8 * s], sl[c][t8 + kG8 * s], a2);
#pragma unroll
          for (int o = 4; o; o >>= 1) a2 += __shfl_xor_sync(0xffffffffu, a2, o);
          if (live && t8 == 0) al[c] = a2;
        }
        __syncwarp();
        // ... then the intra-unit pairs: {(0,1),(2,3)}, {(0,2),(1,3)}, {(0,3),(1,2)}
        // in both units (subgroup rho: unit rho >> 1, pair rho & 1)
#pragma unroll 1
        for (int k = 0; k < 3; ++k) {
          const int base = kUw * (rho >> 1), pr = rho & 1;
          const int a0 = (k == 0) ? 2 * pr : (k == 1 ? pr : (pr ? 1 : 0));
          const int b0 = (k == 0) ? 2 * pr + 1 : (k == 1 ? pr + 2 : (pr ? 2 : 3));
          in_place(sl, al, cid, base + a0, base + b0, rot);
        }
      }
      // cross pairs (t_i, b_{(i+s) mod 4}), s = 0..3: the top column t_rho stays
      // in this subgroup's registers for the whole round and the bottom columns
      // rotate through the subgroups (subgroup rho holds b_{(rho+s) mod 4} at
      // sub-round s) by 8-lane shuffles -- no shared-memory round trip per
      // sub-round (a sub-round of the smem version moved 640 B per lane)
      const int cx = rho, cy = kUw + ((rho + kUw - 1) & 3);   // slots of the last pair
      double2 x[kR2], y[kR2];
      {
        const double2* px = reinterpret_cast<const double2*>(sl[rho]) + t8;
        const double2* py = reinterpret_cast<const double2*>(sl[kUw + rho]) + t8;
#pragma unroll
        for (int s = 0; s < kR2; ++s) {
          x[s] = px[kG8 * s];
          y[s] = py[kG8 * s];
        }
      }
      double ax = al[rho], ay = al[kUw + rho];
      const int idx = cid[rho];
      int idy = cid[kUw + rho];
      {
        const int src = (lane + kG8) & 31;
#pragma unroll 1
        for (int sr = 0; sr < kUw; ++sr) {
          if (live && jc_rotate(x, y, idx, idy, ax, ay, n, small, tol)) rot = 1;
          if (sr == kUw - 1) break;
#pragma unroll
          for (int s = 0; s < kR2; ++s) {
            y[s].x = __shfl_sync(0xffffffffu, y[s].x, src);
            y[s].y = __shfl_sync(0xffffffffu, y[s].y, src);
          }
          ay = __shfl_sync(0xffffffffu, ay, src);
          idy = __shfl_sync(0xffffffffu, idy, src);
        }
      }
      // the rotated columns go to the next owners
      {
        const int nb = P2P ? (buf == 2 ? 0 : buf + 1) : (buf ^ 1);
        // three buffers: the destinations' buffer nb was last read two rounds ago
        if (P2P && live && round_g >= 2)
          jc_wait(jc_saddr(&sh.freeb[nb][lg]), ((round_g - 2) / 3) & 1);
        if (live) {
          double2* dx = reinterpret_cast<double2*>(sht->slot[nb][lt][wt + cx]) + t8;
          double2* dy = reinterpret_cast<double2*>(shb->slot[nb][lb][wb + (cy - kUw)]) + t8;
#pragma unroll
          for (int s = 0; s < kR2; ++s) {
            dx[kG8 * s] = x[s];
            dy[kG8 * s] = y[s];
          }
          if (t8 == 0) {
            sht->alpha[nb][lt][wt + cx] = ax;
            shb->alpha[nb][lb][wb + cy - kUw] = ay;
            sht->col[nb][lt][wt + cx] = idx;
            shb->col[nb][lb][wb + cy - kUw] = idy;
          }
          if (P2P) {
            // the warp's writes into the destinations' buffer nb are done and it is
            // done reading its buffer buf: after the warp barrier (memory ordering
            // among the lanes) one lane releases at cluster scope (cumulative)
            __syncwarp();
            if (lane == 0) {
              jc_remote_arrive(jc_saddr(&sh.ready[nb][lt]), uint32_t(gt / gpc));
              jc_remote_arrive(jc_saddr(&sh.ready[nb][lb]), uint32_t(gb / gpc));
              jc_remote_arrive(jc_saddr(&sh.freeb[buf][st % gpc]), uint32_t(st / gpc));
              jc_remote_arrive(jc_saddr(&sh.freeb[buf][sb % gpc]), uint32_t(sb / gpc));
            }
          }
        }
      }
      buf = P2P ? (buf == 2 ? 0 : buf + 1) : (buf ^ 1);
      ++round_g;
      if (!P2P) cl.sync();
    }
    if (rot) atomicOr(&cl.map_shared_rank(&sh, 0)->rot, 1);
#ifdef TTR_JAC_PROF
    if (live && rot && (tid & 31) == 0) atomicAdd(&flags[40 + min(sweep, 23)], 1);
#endif
    cl.sync();
    const int any = cl.map_shared_rank(&sh, 0)->rot;
    cl.sync();
    if (!any) {
      conv = true;
      break;
    }
  }
  if (crank == 0 && tid == 0) {
    if (!conv) atomicOr(&flags[3], 2);
    flags[12] += conv ? sweep + 1 : sweep;
    flags[13] += 1;
  }
  // norms of every column into every CTA (by column id), then sort by rank
  for (int c8 = 0; c8 < 2 * kUw; ++c8) {
    const double* sl = sh.slot[buf][lgc][c8];
    double s2 = 0.0;
    for (int i = lane; i < kRows; i += 32) s2 = fma(sl[i], sl[i], s2);
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const int col = sh.col[buf][lgc][c8];
    if (live && lane == 0 && col < n)
      for (int rr = 0; rr < kCl; ++rr) cl.map_shared_rank(&sh, rr)->norms[col] = sqrt(s2);
  }
  cl.sync();
  if (live) {
    for (int c8 = 0; c8 < 2 * kUw; ++c8) {
      const double* sl = sh.slot[buf][lg][c8];
      const int col = sh.col[buf][lg][c8];
      if (col >= n) continue;
      const double sj = sh.norms[col];
      int rank = 0;
      for (int k = lane; k < n; k += 32) {
        const double sk = sh.norms[k];
        rank += (sk > sj) || (sk == sj && k < col);
      }
      for (int o = 16; o; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
      for (int i = lane; i < m; i += 32) AV[i + int64_t(rank) * m] = sl[i];
      if (lane == 0) sigma[rank] = sj;
    }
  }
}

// ------------------------------------------------------------------------
// Large-n one-sided Jacobi (n > 160: the deterministic baseline's bond factors,
// NEXT-1, ranks of the assembled sum up to ~1000): the round-robin ordering of
// the single-CTA jacobi_kernel (linalg.cu) -- same pairs per round, same
// per-pair arithmetic -- plus the cluster kernel's negligible-column test, every
// pair of a round on its own warp across a cooperative grid, W (and V) in global
// memory (L2-resident: 2.9 MB each for n = 600), one grid barrier per round.
// The single-CTA kernel processes the ~n/2 pairs of a round with 32 warps out of
// global memory (about 2.7 s per 600 x 600 SVD with V).
constexpr int kJgThreads = 256;
__global__ void __launch_bounds__(kJgThreads)
    jacobi_grid_kernel(double* __restrict__ W, int m, int n, double* __restrict__ Vw,
                       double* __restrict__ AV, double* __restrict__ Vout,
                       double* __restrict__ sigma, double* __restrict__ nrm,
                       int* __restrict__ rot, int max_sweeps, int* __restrict__ flags) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int gw = int((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = int((gridDim.x * blockDim.x) >> 5);
  const int np = (n + 1) & ~1;
  const double tol = double(m) * 0x1p-52;
  // ||A||_F^2 (column sums in a fixed order by warp, then by column: nrm[] as
  // scratch) for the dgesvj-style negligible-column test of the cluster kernel:
  // columns below 16 m u ||A||_F are not rotated (a rank-deficient bond matrix
  // -- hundreds of null columns of the assembled sum -- otherwise keeps
  // re-rotating rounding noise: 25 sweeps instead of ~10)
  for (int j = gw; j < n; j += nwarps) {
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) s2 += W[i + int64_t(j) * m] * W[i + int64_t(j) * m];
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) nrm[j] = s2;
  }
  grid.sync();
  double fro2 = 0.0;
  for (int j = lane; j < n; j += 32) fro2 += nrm[j];
  for (int o = 16; o; o >>= 1) fro2 += __shfl_xor_sync(0xffffffffu, fro2, o);
  fro2 = __shfl_sync(0xffffffffu, fro2, 0);
  const double negl = 16.0 * m * 0x1p-53;
  const double small = negl * negl * fro2;
  grid.sync();   // nrm[] is reused below
  int sweep = 0;
  bool conv = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (blockIdx.x == 0 && threadIdx.x == 0) rot[(sweep + 1) % 3] = 0;
    int rotated = 0;
    for (int round = 0; round < np - 1; ++round) {
      for (int pi = gw; pi < np / 2; pi += nwarps) {
        int p = (pi == 0) ? 0 : ((pi - 1 + round) % (np - 1)) + 1;
        int q = ((np - 2 - pi + round) % (np - 1)) + 1;
        if (p >= n || q >= n) continue;
        if (p > q) { const int t = p; p = q; q = t; }
        double* ap = W + int64_t(p) * m;
        double* aq = W + int64_t(q) * m;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < m; i += 32) {
          const double x = ap[i], y = aq[i];
          al += x * x; be += y * y; ga += x * y;
        }
        for (int o = 16; o; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (!(fmin(al, be) > small) || !(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int i = lane; i < m; i += 32) {
          const double x = ap[i], y = aq[i];
          ap[i] = cs * x - sn * y;
          aq[i] = sn * x + cs * y;
        }
        if (Vw) {
          double* vp = Vw + int64_t(p) * n;
          double* vq = Vw + int64_t(q) * n;
          for (int i = lane; i < n; i += 32) {
            const double x = vp[i], y = vq[i];
            vp[i] = cs * x - sn * y;
            vq[i] = sn * x + cs * y;
          }
        }
        rotated = 1;
      }
      grid.sync();
    }
    if (rotated && lane == 0) atomicOr(&rot[sweep % 3], 1);
    grid.sync();
    if (rot[sweep % 3] == 0) {
      conv = true;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!conv) atomicOr(&flags[3], 2);
    flags[12] += conv ? sweep + 1 : sweep;
    flags[13] += 1;
  }
  // sigma_j = ||w_j||, sorted descending (stable by index): AV, Vout, sigma
  for (int j = gw; j < n; j += nwarps) {
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) s2 += W[i + int64_t(j) * m] * W[i + int64_t(j) * m];
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) nrm[j] = sqrt(s2);
  }
  grid.sync();
  for (int j = gw; j < n; j += nwarps) {
    const double sj = nrm[j];
    int rank = 0;
    for (int k = lane; k < n; k += 32) {
      const double sk = nrm[k];
      rank += (sk > sj) || (sk == sj && k < j);
    }
    for (int o = 16; o; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    for (int i = lane; i < m; i += 32) AV[i + int64_t(rank) * m] = W[i + int64_t(j) * m];
    if (Vout)
      for (int i = lane; i < n; i += 32) Vout[i + int64_t(rank) * n] = Vw[i + int64_t(j) * n];
    if (lane == 0) sigma[rank] = sj;
  }
}

__global__ void jg_init_kernel(const double* __restrict__ A, int64_t lda, int m, int n,
                               double* __restrict__ W, double* __restrict__ Vw) {
  const int64_t mn = int64_t(m) * n, nn = int64_t(n) * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < mn + (Vw ? nn : 0);
       e += int64_t(gridDim.x) * blockDim.x) {
    if (e < mn) {
      const int64_t i = e % m, j = e / m;
      W[e] = A[i + j * lda];
    } else {
      const int64_t f = e - mn;
      Vw[f] = (f % n == f / n) ? 1.0 : 0.0;
    }
  }
}

}  // namespace

bool svd_cluster_fits(int64_t m, int64_t n) {
  const int64_t U = (n + kUw - 1) / kUw, UP = U + (U & 1);
  return n >= 64 && m >= n && m <= kRows && UP / 2 <= kCl * kGpc;
}

int svd_nov_cluster(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
                    double* sigma, cudaStream_t s) {
  static std::atomic<bool> attr[64];
  const size_t shm = sizeof(JcShared);
  std::unique_lock<std::mutex> init_lock(init_mutex(), std::defer_lock);
  if (!attr[c.device & 63]) init_lock.lock();
  if (!attr[c.device & 63]) {
    TTR_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel<true>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
    TTR_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel<false>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
    attr[c.device & 63] = true;
  }
  const int64_t U = (n + kUw - 1) / kUw, UP = U + (U & 1);
  const int gpc = int((UP / 2 + kCl - 1) / kCl);
  // default: one cluster barrier per round (0.99 ms per 144^2 SVD); the
  // point-to-point variant (TTR_JACOBI=p2p) measured 1.24 ms
  static const bool p2p = [] {
    const char* v = getenv("TTR_JACOBI");
    return v && strcmp(v, "p2p") == 0;
  }();
  if (!p2p)
    jacobi_cluster_kernel<false><<<kCl, kJcThreads, shm, s>>>(A, lda, int(m), int(n), gpc, AV,
                                                                sigma, 40, c.flags.p);
  else
    jacobi_cluster_kernel<true><<<kCl, kJcThreads, shm, s>>>(A, lda, int(m), int(n), gpc, AV,
                                                               sigma, 40, c.flags.p);
  return launched();
}

// Grid-cooperative one-sided Jacobi (large n): AV = U Sigma (m x n, ld m, sorted),
// sigma, and, if V != nullptr, V (n x n, ld n).
int svd_jacobi_grid(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
                    double* V, double* sigma, cudaStream_t s) {
  if (m < n || n < 1) {
    set_error("svd_jacobi_grid: need m >= n >= 1");
    return TT_ERR_ARG;
  }
  DBuf W, Vw, nrm;
  IBuf rot;
  TTR_TRY(dalloc(W, size_t(m) * n, s));
  if (V) TTR_TRY(dalloc(Vw, size_t(n) * n, s));
  TTR_TRY(dalloc(nrm, size_t(n), s));
  TTR_TRY(ialloc(rot, 3, s));
  TTR_CUDA(cudaMemsetAsync(rot.p, 0, 3 * sizeof(int), s));
  jg_init_kernel<<<c.sm_count * 4, 256, 0, s>>>(A, lda, int(m), int(n), W.p, V ? Vw.p : nullptr);
  TTR_TRY(launched());
  // one warp per pair of a round (n/2 pairs), at most one CTA per SM
  const int warps = kJgThreads / 32;
  int per_sm = 0;
  TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_grid_kernel, kJgThreads, 0));
  if (per_sm < 1) {
    set_error("svd_jacobi_grid: kernel cannot be resident");
    return TT_ERR_CUDA;
  }
  const int want = int(((n + 1) / 2 + warps - 1) / warps);
  const int blocks = std::max(1, std::min(want, c.sm_count));   // per_sm >= 1 checked above
  double* Wp = W.p;
  double* Vwp = V ? Vw.p : nullptr;
  int mi = int(m), ni = int(n), maxs = 40;
  double* np_ = nrm.p;
  int* rp = rot.p;
  int* fl = c.flags.p;
  void* args[] = {&Wp, &mi, &ni, &Vwp, &AV, &V, &sigma, &np_, &rp, &maxs, &fl};
  TTR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(jacobi_grid_kernel),
                                       dim3(blocks), dim3(kJgThreads), args, 0, s));
  return launched();
}

}  // namespace ttr
