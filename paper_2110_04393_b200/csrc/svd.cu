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
// formulas, thresholds and convergence test) on a cluster of 8 CTAs, over
// UNITS of two columns (block-cyclic ordering).
//
// Units u = (2u, 2u+1) take part in a circle ordering; a "group" (one warp)
// holds a top and a bottom unit.  Round 0 of a sweep first rotates the two
// intra-unit pairs; every round then rotates the four cross pairs in two
// sub-rounds ((t0,b0),(t1,b1)) and ((t0,b1),(t1,b0)), one pair per half-warp
// (16 threads, rows t + 16 s).  The second sub-round writes its rotated columns
// straight into the slots of the groups that own the units next round (top row
// shifts right, bottom row left, unit 0 fixed), so the move is the write-back;
// only the units crossing a CTA boundary go through distributed shared memory.
// One cluster barrier per round, half as many rounds as column pairs.
// ============================================================================
namespace ttr {
namespace {

constexpr int kCl = 8;          // CTAs per cluster
constexpr int kGpc = 5;         // groups (warps) per CTA: n <= 160 -> <= 40 groups
constexpr int kG16 = 16;        // threads per pair
constexpr int kRps = 10;        // rows per thread (m <= 160)
constexpr int kRows = kG16 * kRps;

struct JcShared {
  double slot[2][kGpc][4][kRows];   // [buffer][group][t0, t1, b0, b1][rows]
  double alpha[2][kGpc][4];         // squared norms travelling with the columns
  int col[2][kGpc][4];              // column ids travelling with the columns
  double norms[kCl * kGpc * 4];     // final column norms (all columns, by id)
  double red[8];
  int rot;
};

constexpr int kJcThreads = kGpc * 32;

// rotate the pair (X, Y) held by this half-warp (ids cx, cy, squared norms ax,
// ay); p = min(id) is rotated as column p of the single-CTA kernel
__device__ __forceinline__ bool jc_rotate(double (&x)[kRps], double (&y)[kRps], int cx, int cy,
                                          double& ax, double& ay, int n, double small, double tol) {
  double ga = 0.0;
#pragma unroll
  for (int s = 0; s < kRps; ++s) ga = fma(x[s], y[s], ga);
#pragma unroll
  for (int o = 8; o; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
  const bool swp = cx > cy;
  const double ap = swp ? ay : ax, aq = swp ? ax : ay;
  if (!(cx < n && cy < n && fmin(ap, aq) > small && fabs(ga) > tol * sqrt(ap * aq))) return false;
  const double zeta = (aq - ap) / (2.0 * ga);
  double tt = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
  const double cs = rsqrt(fma(tt, tt, 1.0));
  double sn = cs * tt;
  if (swp) { sn = -sn; tt = -tt; }
#pragma unroll
  for (int s = 0; s < kRps; ++s) {
    const double xs = x[s], ys = y[s];
    x[s] = fma(cs, xs, -sn * ys);
    y[s] = fma(sn, xs, cs * ys);
  }
  ax -= tt * ga;
  ay += tt * ga;
  return true;
}

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kJcThreads)
    jacobi_cluster_kernel(const double* __restrict__ A, int64_t lda, int m, int n, int gpc,
                          double* __restrict__ AV, double* __restrict__ sigma, int max_sweeps,
                          int* __restrict__ flags) {
  extern __shared__ __align__(16) unsigned char jc_raw[];
  JcShared& sh = *reinterpret_cast<JcShared*>(jc_raw);
  cg::cluster_group cl = cg::this_cluster();
  const int crank = int(cl.block_rank());
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int lg = warp, h = lane >> 4, t16 = lane & 15;    // group, half, thread in half
  const int U = (n + 1) / 2, UP = U + (U & 1), halfU = UP / 2;
  const int g = crank * gpc + lg;
  const bool live = lg < gpc && g < halfU;
  const int lgc = live ? lg : 0;

  // round 0: group g holds top unit (g == 0 ? 0 : g) and bottom unit UP - 1 - g
  {
    const int ut = live ? g : -1, ub = live ? UP - 1 - g : -1;
    for (int c4 = 0; c4 < 4; ++c4) {
      const int unit = c4 < 2 ? ut : ub;
      const int c0 = unit < 0 ? n : 2 * unit + (c4 & 1);
      const int cid = c0 < n ? c0 : n;
      double* sl = sh.slot[0][lg][c4];
      for (int i = lane; i < kRows; i += 32)
        sl[i] = (cid < n && i < m) ? A[i + int64_t(cid) * lda] : 0.0;
      if (lane == 0) {
        sh.col[0][lg][c4] = cid;
        sh.alpha[0][lg][c4] = 0.0;
      }
    }
  }
  __syncthreads();
  double part = 0.0;
  for (int c4 = 0; c4 < 4; ++c4)
    for (int i = lane; i < kRows; i += 32) {
      const double v = sh.slot[0][lg][c4][i];
      part = fma(v, v, part);
    }
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if (lane == 0) sh.red[warp] = part;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kGpc; ++w) s += sh.red[w];
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

  // destinations of this group's units after a round (fixed for the run):
  // top:    g == 0 -> (0, top); g < halfU-1 -> (g+1, top); g == halfU-1 -> (g, bottom)
  // bottom: g == 0 -> (1, top); g >= 1 -> (g-1, bottom)
  const int gt = (g == 0) ? 0 : (g < halfU - 1 ? g + 1 : g);
  const int wt = (g == 0 || g < halfU - 1) ? 0 : 2;
  const int gb = (g == 0) ? 1 : g - 1, wb = (g == 0) ? 0 : 2;
  JcShared* sht = (gt / gpc == crank) ? &sh : cl.map_shared_rank(&sh, gt / gpc);
  JcShared* shb = (gb / gpc == crank) ? &sh : cl.map_shared_rank(&sh, gb / gpc);
  const int lt = gt % gpc, lb = gb % gpc;

  int buf = 0, sweep = 0;
  bool conv = false;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) sh.rot = 0;
    int rot = 0;
    for (int r = 0; r < UP - 1; ++r) {
      double (*sl)[kRows] = sh.slot[buf][lgc];
      double* al = sh.alpha[buf][lgc];
      const int* cid = sh.col[buf][lgc];
      double x[kRps], y[kRps];
      if (r == 0) {
        // exact squared norms, then the intra-unit pairs (t0,t1) | (b0,b1)
        const int cx = 2 * h, cy = 2 * h + 1;
#pragma unroll
        for (int s = 0; s < kRps; ++s) {
          x[s] = sl[cx][t16 + kG16 * s];
          y[s] = sl[cy][t16 + kG16 * s];
        }
        double ax = 0.0, ay = 0.0;
#pragma unroll
        for (int s = 0; s < kRps; ++s) {
          ax = fma(x[s], x[s], ax);
          ay = fma(y[s], y[s], ay);
        }
#pragma unroll
        for (int o = 8; o; o >>= 1) {
          ax += __shfl_xor_sync(0xffffffffu, ax, o);
          ay += __shfl_xor_sync(0xffffffffu, ay, o);
        }
        if (live && jc_rotate(x, y, cid[cx], cid[cy], ax, ay, n, small, tol)) rot = 1;
        if (live) {   // (non-live warps alias group 0's slots: read only)
#pragma unroll
          for (int s = 0; s < kRps; ++s) {
            sl[cx][t16 + kG16 * s] = x[s];
            sl[cy][t16 + kG16 * s] = y[s];
          }
        }
        __syncwarp();
        if (live && t16 == 0) { al[cx] = ax; al[cy] = ay; }
        __syncwarp();
      }
      // sub-round 1: (t0, b0) | (t1, b1), in place
      {
        const int cx = h, cy = 2 + h;
#pragma unroll
        for (int s = 0; s < kRps; ++s) {
          x[s] = sl[cx][t16 + kG16 * s];
          y[s] = sl[cy][t16 + kG16 * s];
        }
        double ax = al[cx], ay = al[cy];
        if (live && jc_rotate(x, y, cid[cx], cid[cy], ax, ay, n, small, tol)) rot = 1;
        if (live) {   // (non-live warps alias group 0's slots: read only)
#pragma unroll
          for (int s = 0; s < kRps; ++s) {
            sl[cx][t16 + kG16 * s] = x[s];
            sl[cy][t16 + kG16 * s] = y[s];
          }
        }
        __syncwarp();
        if (live && t16 == 0) { al[cx] = ax; al[cy] = ay; }
        __syncwarp();
      }
      // sub-round 2: (t0, b1) | (t1, b0), written to the next owners
      {
        const int cx = h, cy = 3 - h;
#pragma unroll
        for (int s = 0; s < kRps; ++s) {
          x[s] = sl[cx][t16 + kG16 * s];
          y[s] = sl[cy][t16 + kG16 * s];
        }
        double ax = al[cx], ay = al[cy];
        const int idx = cid[cx], idy = cid[cy];
        if (live && jc_rotate(x, y, idx, idy, ax, ay, n, small, tol)) rot = 1;
        if (live) {
          const int nb = buf ^ 1;
          double* dx = sht->slot[nb][lt][wt + h];          // top unit column h
          double* dy = shb->slot[nb][lb][wb + (1 - h)];    // bottom unit column 1-h
#pragma unroll
          for (int s = 0; s < kRps; ++s) {
            dx[t16 + kG16 * s] = x[s];
            dy[t16 + kG16 * s] = y[s];
          }
          if (t16 == 0) {
            sht->alpha[nb][lt][wt + h] = ax;
            shb->alpha[nb][lb][wb + 1 - h] = ay;
            sht->col[nb][lt][wt + h] = idx;
            shb->col[nb][lb][wb + 1 - h] = idy;
          }
        }
      }
      buf ^= 1;
      cl.sync();
    }
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
  for (int c4 = 0; c4 < 4; ++c4) {
    const double* sl = sh.slot[buf][lgc][c4];
    double s2 = 0.0;
    for (int i = lane; i < kRows; i += 32) s2 = fma(sl[i], sl[i], s2);
    for (int o = 16; o; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    const int col = sh.col[buf][lgc][c4];
    if (live && lane == 0 && col < n)
      for (int rr = 0; rr < kCl; ++rr) cl.map_shared_rank(&sh, rr)->norms[col] = sqrt(s2);
  }
  cl.sync();
  if (live) {
    for (int c4 = 0; c4 < 4; ++c4) {
      const double* sl = sh.slot[buf][lg][c4];
      const int col = sh.col[buf][lg][c4];
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

}  // namespace

bool svd_cluster_fits(int64_t m, int64_t n) {
  const int64_t U = (n + 1) / 2, UP = U + (U & 1);
  return n >= 64 && m >= n && m <= kRows && UP / 2 <= kCl * kGpc;
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
  const int64_t U = (n + 1) / 2, UP = U + (U & 1);
  const int gpc = int((UP / 2 + kCl - 1) / kCl);
  jacobi_cluster_kernel<<<kCl, kJcThreads, shm, s>>>(A, lda, int(m), int(n), gpc, AV, sigma,
                                                       40, c.flags.p);
  return launched();
}

}  // namespace ttr
