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
#include <math.h>

#include "common.cuh"

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

int svd_nov(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
            double* sigma, cudaStream_t s) {
  if (!svd_nov_fits(m, n)) {
    set_error("svd_nov: unsupported shape m=%lld n=%lld", (long long)m, (long long)n);
    return TT_ERR_ARG;
  }
  if (m <= 16) return launch_rr<2>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 32) return launch_rr<4>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 64) return launch_rr<8>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 96) return launch_rr<12>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 128) return launch_rr<16>(c, m, n, A, lda, AV, sigma, s);
  if (m <= 144) return launch_rr<18>(c, m, n, A, lda, AV, sigma, s);
  return launch_rr<20>(c, m, n, A, lda, AV, sigma, s);
}

}  // namespace ttr
