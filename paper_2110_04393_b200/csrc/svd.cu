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
  const unsigned gmask = 0xFFu << (lane & 24);
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
      if (grp >= half) continue;
      const int p = min(p0, q0), q = max(p0, q0);
      if (q >= n) continue;                             // dummy column (odd n)
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
      for (int o = 4; o; o >>= 1) ga += __shfl_xor_sync(gmask, ga, o, kGroup);
      const double al = cn[p], be = cn[q];
      if (!(fmin(al, be) > small) || !(fabs(ga) > tol * sqrt(al * be))) continue;
      const double zeta = (be - al) / (2.0 * ga);
      const double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
      const double cs = rsqrt(fma(tt, tt, 1.0)), sn = cs * tt;
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
  static bool attr[64] = {false};
  const size_t shm = size_t(n) * 8 * RPT * sizeof(double);
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
  if (svd_cluster_fits(m, n)) return svd_nov_cluster(c, m, n, A, lda, AV, sigma, s);
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
// formulas, thresholds and convergence test) spread over a cluster of 8 CTAs.
//
// Column pairs are "groups" of 16 threads (row t + 16 s of a column per
// thread); group g of the circle ordering lives in CTA g / GPC_G.  A group
// keeps its two columns in registers for the round, rotates them and writes
// them straight into the slots of the groups that own them next round
// (top row shifts right, bottom row shifts left, position 0 fixed), so the
// move IS the write-back; only the two columns crossing a CTA boundary go
// through distributed shared memory.  One cluster barrier per round.
// ============================================================================
namespace ttr {
namespace {

constexpr int kCl = 8;          // CTAs per cluster
constexpr int kGpc = 9;         // groups per CTA (n <= 144 -> 72 groups)
constexpr int kG16 = 16;        // threads per group
constexpr int kRps = 10;        // rows per thread (m <= 160)
constexpr int kRows = kG16 * kRps;       // 160 rows per column slot

struct JcShared {
  double slot[2][kGpc][2][kRows];   // [buffer][local group][top/bottom][rows]
  double alpha[2][kGpc][2];         // squared norms travelling with the columns
  int col[2][kGpc][2];              // column ids travelling with the columns
  double norms[kCl * kGpc * 2];     // final column norms (all columns, by id)
  double red[8];
  int rot;
};

constexpr int kJcThreads = ((kGpc * kG16 + 31) / 32) * 32;   // 160: whole warps

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kJcThreads)
    jacobi_cluster_kernel(const double* __restrict__ A, int64_t lda, int m, int n, int gpc,
                          double* __restrict__ AV, double* __restrict__ sigma, int max_sweeps,
                          int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char jc_raw[];
  JcShared& sh = *reinterpret_cast<JcShared*>(jc_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int crank = int(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lg = tid / kG16, t16 = tid % kG16;
  const int np = (n + 1) & ~1, half = np / 2;
  const int g = crank * gpc + lg;                 // global group index
  const bool live = lg < gpc && lg < kGpc && g < half;

  // round 0 of the circle ordering: group g holds top = column g (0 for g = 0)
  // and bottom = column np - 1 - g (index n is the dummy column of an odd n)
  if (lg < kGpc) {
    for (int which = 0; which < 2; ++which) {
      const int c0 = live ? (which ? np - 1 - g : g) : n;
      double* sl = sh.slot[0][lg][which];
      for (int i = t16; i < kRows; i += kG16)
        sl[i] = (c0 < n && i < m) ? A[i + int64_t(c0) * lda] : 0.0;
      if (t16 == 0) {
        sh.col[0][lg][which] = c0;
        sh.alpha[0][lg][which] = 0.0;
      }
    }
  }
  // ||A||_F^2 over the cluster
  double part = 0.0;
  if (lg < kGpc)
    for (int which = 0; which < 2; ++which)
      for (int i = t16; i < kRows; i += kG16) {
        const double v = sh.slot[0][lg][which][i];
        part = fma(v, v, part);
      }
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) sh.red[warp] = part;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < (blockDim.x + 31) / 32; ++w) s += sh.red[w];
    for (int r = 0; r < kCl; ++r) cl.map_shared_rank(&sh, r)->norms[crank] = s;   // scratch
  }
  cl.sync();
  double fro2 = 0.0;
  for (int r = 0; r < kCl; ++r) fro2 += sh.norms[r];
  cl.sync();

  const double u = 0x1p-53;
  const double tol = 2.0 * m * u;
  const double negl = 16.0 * m * u;
  const double small = negl * negl * fro2;

  // where this group's columns go after a round (fixed for the whole run):
  // top:    g == 0 -> (0, top); g < half-1 -> (g+1, top); g == half-1 -> (g, bottom)
  // bottom: g == 0 -> (1, top); g >= 1 -> (g-1, bottom)
  const int gt = (g == 0) ? 0 : (g < half - 1 ? g + 1 : g), wt = (g == 0 || g < half - 1) ? 0 : 1;
  const int gb = (g == 0) ? 1 : g - 1, wb = (g == 0) ? 0 : 1;
  JcShared* sht = (gt / gpc == crank) ? &sh : cl.map_shared_rank(&sh, gt / gpc);
  JcShared* shb = (gb / gpc == crank) ? &sh : cl.map_shared_rank(&sh, gb / gpc);
  const int lt = gt % gpc, lb = gb % gpc;
  const int lgc = live ? lg : 0;   // non-live groups compute on slot 0 and write nothing

  int buf = 0, sweep = 0;
  bool conv = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) sh.rot = 0;
    int rot = 0;
    for (int r = 0; r < np - 1; ++r) {
      {   // every thread of the CTA (5 full warps) runs this: full-warp shuffles
        const double* st = sh.slot[buf][lgc][0];
        const double* sb = sh.slot[buf][lgc][1];
        double x[kRps], y[kRps];
        double ga = 0.0, al = 0.0, be = 0.0;
#pragma unroll
        for (int s = 0; s < kRps; ++s) {
          x[s] = st[t16 + kG16 * s];
          y[s] = sb[t16 + kG16 * s];
          ga = fma(x[s], y[s], ga);
        }
        const int colt = sh.col[buf][lgc][0], colb = sh.col[buf][lgc][1];
        if (r == 0) {   // exact squared norms at the start of every sweep
#pragma unroll
          for (int s = 0; s < kRps; ++s) {
            al = fma(x[s], x[s], al);
            be = fma(y[s], y[s], be);
          }
#pragma unroll
          for (int o = 8; o; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
          }
        } else {
          al = sh.alpha[buf][lgc][0];
          be = sh.alpha[buf][lgc][1];
        }
#pragma unroll
        for (int o = 8; o; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
        // rotation of (p, q) = (min, max) column ids, applied as T' = c T - s' B,
        // B' = s' T + c B with s' = -s when the top column is q
        const bool swp = colt > colb;
        const double ap = swp ? be : al, aq = swp ? al : be;
        double cs = 1.0, sn = 0.0, tt = 0.0;
        if (live && colt < n && colb < n && fmin(ap, aq) > small &&
            fabs(ga) > tol * sqrt(ap * aq)) {
          const double zeta = (aq - ap) / (2.0 * ga);
          tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
          cs = rsqrt(fma(tt, tt, 1.0));
          sn = cs * tt;
          rot = 1;
        }
        if (swp) { sn = -sn; tt = -tt; }
        if (live) {
          const int nb = buf ^ 1;
          double* dt = sht->slot[nb][lt][wt];
          double* db = shb->slot[nb][lb][wb];
#pragma unroll
          for (int s = 0; s < kRps; ++s) {
            dt[t16 + kG16 * s] = fma(cs, x[s], -sn * y[s]);
            db[t16 + kG16 * s] = fma(sn, x[s], cs * y[s]);
          }
          if (t16 == 0) {
            sht->alpha[nb][lt][wt] = al - tt * ga;
            shb->alpha[nb][lb][wb] = be + tt * ga;
            sht->col[nb][lt][wt] = colt;
            shb->col[nb][lb][wb] = colb;
          }
        }
      }
      buf ^= 1;
      cl.sync();
    }
    // cluster-wide OR of "rotated in this sweep"
    if (rot) atomicOr(&cl.map_shared_rank(&sh, 0)->rot, 1);
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
  {
    for (int which = 0; which < 2; ++which) {
      const double* sl = sh.slot[buf][lgc][which];
      double s2 = 0.0;
#pragma unroll
      for (int s = 0; s < kRps; ++s) s2 = fma(sl[t16 + kG16 * s], sl[t16 + kG16 * s], s2);
#pragma unroll
      for (int o = 8; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
      const int col = sh.col[buf][lgc][which];
      if (live && t16 == 0 && col < n)
        for (int rr = 0; rr < kCl; ++rr) cl.map_shared_rank(&sh, rr)->norms[col] = sqrt(s2);
    }
  }
  cl.sync();
  if (live) {
    for (int which = 0; which < 2; ++which) {
      const double* sl = sh.slot[buf][lg][which];
      const int col = sh.col[buf][lg][which];
      if (col >= n) continue;
      const double sj = sh.norms[col];
      int rank = 0;
      for (int k = t16; k < n; k += kG16) {
        const double sk = sh.norms[k];
        rank += (sk > sj) || (sk == sj && k < col);
      }
#pragma unroll
      for (int o = 8; o; o >>= 1) rank += __shfl_xor_sync(0xffffu << (lane & 16), rank, o);
      for (int i = t16; i < m; i += kG16) AV[i + int64_t(rank) * m] = sl[i];
      if (t16 == 0) sigma[rank] = sj;
    }
  }
}

}  // namespace

bool svd_cluster_fits(int64_t m, int64_t n) {
  return n >= 64 && m >= n && m <= kG16 * kRps && (n + 1) / 2 <= kCl * kGpc;
}

int svd_nov_cluster(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
                    double* sigma, cudaStream_t s) {
  static bool attr[64] = {false};
  const size_t shm = sizeof(JcShared);
  if (!attr[c.device & 63]) {
    TTR_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(shm)));
    attr[c.device & 63] = true;
  }
  const int half = int((n + 1) / 2);
  const int gpc = (half + kCl - 1) / kCl;
  jacobi_cluster_kernel<<<kCl, kJcThreads, shm, s>>>(A, lda, int(m), int(n), gpc, AV, sigma,
                                                       40, c.flags.p);
  return launched();
}

}  // namespace ttr
