// Dense building blocks of the sweep besides the GEMM:
//  * Philox4x32-10 Gaussian fill of the sketch cores (Def. 3.1; R9)
//  * shifted CholeskyQR3 pieces: Cholesky + triangular inverse of the Gram (one CTA)
//  * Householder QR fallback (one CTA, only when CholeskyQR breaks down)
//  * one-sided Jacobi SVD (one CTA) for the truncation step (R3)
//  * eps-rank, Frobenius norm, transpose, fill
#include <math.h>

#include "common.cuh"

namespace ttr {

// ============================================================== Philox
namespace {

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2,
                                             uint32_t& c3, uint32_t k0, uint32_t k1) {
  const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
  const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
  const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
  c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
}

__device__ __forceinline__ double unit53(uint32_t lo, uint32_t hi) {
  const uint64_t v = (uint64_t(hi) << 32) | uint64_t(lo);
  return (double(v >> 11) + 0.5) * 0x1p-53;
}

__global__ void philox_fill_kernel(double* __restrict__ out, int64_t count, uint32_t key0,
                                   uint32_t key1, uint32_t n, uint32_t tag, double scale) {
  const int64_t npair = (count + 1) / 2;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < npair;
       k += int64_t(gridDim.x) * blockDim.x) {
    uint32_t c0 = uint32_t(k), c1 = uint32_t(uint64_t(k) >> 32), c2 = n, c3 = tag;
    uint32_t k0 = key0, k1 = key1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      philox_round(c0, c1, c2, c3, k0, k1);
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const double u1 = unit53(c0, c1), u2 = unit53(c2, c3);
    const double r = sqrt(-2.0 * log(u1));
    const double th = 2.0 * 3.141592653589793 * u2;
    double sn, cs;
    sincos(th, &sn, &cs);
    const double z0 = (r * cs) * scale, z1 = (r * sn) * scale;
    const int64_t e = 2 * k;
    if (e + 1 < count) {
      reinterpret_cast<double2*>(out)[k] = make_double2(z0, z1);
    } else {
      out[e] = z0;
    }
  }
}

}  // namespace

int philox_fill(Ctx& c, double* out, int64_t count, uint64_t seed, uint32_t n, uint32_t tag,
                double scale, cudaStream_t s) {
  if (count <= 0) return TT_OK;
  const int64_t npair = (count + 1) / 2;
  const int threads = 256;
  const int64_t want = (npair + threads - 1) / threads;
  const int blocks = int(std::min<int64_t>(want, int64_t(c.sm_count) * 16));
  philox_fill_kernel<<<blocks, threads, 0, s>>>(out, count, uint32_t(seed & 0xffffffffu),
                                                uint32_t(seed >> 32), n, tag, scale);
  return launched();
}

// ============================================================== Cholesky + inverse
namespace {

constexpr int kCholThreads = 1024;
constexpr int kSmemLimitDoubles = 26 * 1024;   // 208 KB of dynamic shared memory

// flags layout (Ctx.flags): 0 = breakdown in current QR, 1 = fallback used (sticky),
// 2 = zero sketch seen (sticky), 3 = numeric failure (sticky)

// G (n x n, ld n, symmetric) -> Rinv (upper, ld n) with G + shift*I = R^T R,
// optionally R.  mode: 0 = unshifted, 1 = shifted (sCholQR3 first pass, shift
// 11(mn + n(n+1))u * trace(G)), 2 = unshifted + final-pass check ||diag R - 1||.
template <int QN>
__global__ void __launch_bounds__(kCholThreads)
    chol_inv_kernel(const double* __restrict__ G, int n, int64_t m, int mode,
                    double* __restrict__ Rinv, double* __restrict__ Rout,
                    double* __restrict__ gwork, int* __restrict__ flags) {
  extern __shared__ double sh[];
  const bool in_smem = (n * n <= kSmemLimitDoubles);
  double* L = in_smem ? sh : gwork;
  __shared__ double s_shift;
  __shared__ int s_bad;
  const int tid = threadIdx.x;
  if (tid == 0) { s_bad = 0; }
  // trace for the shift and the zero test
  if (tid < 32) {
    double tr = 0.0;
    for (int i = tid; i < n; i += 32) tr += G[i + int64_t(i) * n];
    for (int o = 16; o; o >>= 1) tr += __shfl_xor_sync(0xffffffffu, tr, o);
    if (tid == 0) {
      if (!(tr > 0.0)) {
        if (tr == 0.0) atomicOr(&flags[2], 1);   // Y_n == 0: zero sum (R16)
        s_bad = 1;
      }
      const double u = 0x1p-53;
      s_shift = (mode == 1) ? 11.0 * (double(m) * n + double(n) * (n + 1)) * u * tr : 0.0;
    }
  }
  __syncthreads();
  const double shift = s_shift;
  for (int e = tid; e < n * n; e += kCholThreads) {
    const int i = e % n, j = e / n;
    L[e] = (i >= j) ? G[e] + ((i == j) ? shift : 0.0) : 0.0;
  }
  __syncthreads();
  // right-looking Cholesky, lower L in column-major L[i + j n]
  for (int j = 0; j < n; ++j) {
    const double djj = L[j + j * n];
    const bool okp = djj > 0.0 && isfinite(djj);
    const double d = okp ? sqrt(djj) : 1.0;
    if (!okp && tid == 0) s_bad = 1;
    const double inv = 1.0 / d;
    for (int i = j + 1 + tid; i < n; i += kCholThreads) L[i + j * n] *= inv;
    __syncthreads();
    if (tid == 0) L[j + j * n] = d;
    const int rem = n - j - 1;
    for (int e = tid; e < rem * rem; e += kCholThreads) {
      const int r = e % rem, cc = e / rem;
      if (cc <= r) {
        const int i = j + 1 + r, k = j + 1 + cc;
        L[i + k * n] -= L[i + j * n] * L[k + j * n];
      }
    }
    __syncthreads();
  }
  // X = L^{-1} (lower), one warp per column, column-oriented forward substitution;
  // Rinv = X^T (upper).  x lives in registers: lane owns rows lane + 32 q.
  const int warp = tid >> 5, lane = tid & 31;
  constexpr int kMaxQ = QN;  // n <= 32 * QN
  for (int col = warp; col < n; col += kCholThreads / 32) {
    double x[kMaxQ];
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) {
      const int i = lane + 32 * q;
      x[q] = (i == col) ? 1.0 : 0.0;
    }
    for (int k = col; k < n; ++k) {
      // x_k /= L_kk, then x_i -= L_ik x_k for i > k
      const int qk = k >> 5, lk = k & 31;
      double xk = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxQ; ++q)
        if (q == qk) xk = x[q];
      xk = __shfl_sync(0xffffffffu, xk, lk) / L[k + k * n];
#pragma unroll
      for (int q = 0; q < kMaxQ; ++q) {
        const int i = lane + 32 * q;
        if (i == k) x[q] = xk;
        else if (i > k && i < n) x[q] -= L[i + k * n] * xk;
      }
    }
#pragma unroll
    for (int q = 0; q < kMaxQ; ++q) {
      const int i = lane + 32 * q;
      if (i < n) Rinv[col + int64_t(i) * n] = (i >= col) ? x[q] : 0.0;  // Rinv(col, i) = X(i, col)
    }
  }
  if (Rout) {
    for (int e = tid; e < n * n; e += kCholThreads) {
      const int i = e % n, j = e / n;     // R(i, j) = L(j, i) for j >= i
      Rout[e] = (j >= i) ? L[j + i * n] : 0.0;
    }
  }
  __syncthreads();
  if (tid == 0) {
    int bad = s_bad;
    if (mode == 2 && !bad) {
      double dev = 0.0;
      for (int i = 0; i < n; ++i) dev = fmax(dev, fabs(L[i + i * n] - 1.0));
      if (!(dev < 1e-6)) bad = 1;
    }
    if (bad && !(flags[2] & 1)) atomicOr(&flags[0], 1);
  }
}

// ---------------------------------------------------------- Householder fallback
// Single CTA; runs only if flags[0] is set (breakdown).  A (m x n) is copied to
// the workspace, factored in place (LAPACK-style reflectors with v0 = 1), then
// Q = H_0 ... H_{n-1} [I; 0] is formed by backward accumulation into Q.
constexpr int kHhThreads = 1024;

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (warp == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? red[lane] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

__global__ void __launch_bounds__(kHhThreads)
    householder_kernel(const double* __restrict__ A, int64_t lda, bool trans, int64_t m, int n,
                       double* __restrict__ W, double* __restrict__ tau,
                       double* __restrict__ Q, double* __restrict__ R, int* flags) {
  if (!(flags[0] & 1)) return;
  __shared__ double red[32];
  __shared__ double s_beta, s_tau;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = kHhThreads / 32;
  // W = op(A)
  for (int64_t e = tid; e < m * n; e += kHhThreads) {
    const int64_t i = e % m, j = e / m;
    W[e] = trans ? A[j + i * lda] : A[i + j * lda];
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    double* a = W + int64_t(j) * m;
    double ss = 0.0;
    for (int64_t i = j + 1 + tid; i < m; i += kHhThreads) ss += a[i] * a[i];
    ss = block_sum(ss, red);
    if (tid == 0) {
      const double alpha = a[j];
      if (ss == 0.0) {
        s_tau = 0.0;
        s_beta = alpha;
      } else {
        const double nrm = sqrt(alpha * alpha + ss);
        const double beta = (alpha >= 0.0) ? -nrm : nrm;
        s_tau = (beta - alpha) / beta;
        s_beta = beta;
        a[j] = alpha - beta;  // v0 before scaling
      }
    }
    __syncthreads();
    const double tj = s_tau;
    if (tj != 0.0) {
      const double v0 = a[j];
      const double sc = 1.0 / v0;
      for (int64_t i = j + 1 + tid; i < m; i += kHhThreads) a[i] *= sc;
    }
    __syncthreads();
    if (tid == 0) { a[j] = s_beta; tau[j] = tj; }
    __syncthreads();
    // apply H_j = I - tau v v^T (v = [1; a[j+1:]]) to trailing columns, warp per column
    if (tj != 0.0) {
      for (int cc = j + 1 + warp; cc < n; cc += nw) {
        double* b = W + int64_t(cc) * m;
        double w = (lane == 0) ? b[j] : 0.0;
        for (int64_t i = j + 1 + lane; i < m; i += 32) w += a[i] * b[i];
        for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w *= tj;
        if (lane == 0) b[j] -= w;
        for (int64_t i = j + 1 + lane; i < m; i += 32) b[i] -= w * a[i];
      }
    }
    __syncthreads();
  }
  if (R) {
    for (int e = tid; e < n * n; e += kHhThreads) {
      const int i = e % n, jj = e / n;
      R[e] = (i <= jj) ? W[i + int64_t(jj) * m] : 0.0;
    }
  }
  // Q = [I; 0], then for j = n-1..0: Q[j:, j:] = H_j Q[j:, j:]
  for (int64_t e = tid; e < m * n; e += kHhThreads) {
    const int64_t i = e % m, jj = e / m;
    Q[e] = (i == jj) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int j = n - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj != 0.0) {
      const double* a = W + int64_t(j) * m;
      for (int cc = j + warp; cc < n; cc += nw) {
        double* q = Q + int64_t(cc) * m;
        double w = (lane == 0) ? q[j] : 0.0;
        for (int64_t i = j + 1 + lane; i < m; i += 32) w += a[i] * q[i];
        for (int o = 16; o; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
        w *= tj;
        if (lane == 0) q[j] -= w;
        for (int64_t i = j + 1 + lane; i < m; i += 32) q[i] -= w * a[i];
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    atomicOr(&flags[1], 1);
    flags[0] = 0;
  }
}

}  // namespace

int qr(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, bool trans, double* Q,
       double* R, cudaStream_t s) {
  if (m < n || n < 1) {
    set_error("qr: need m >= n >= 1 (m=%lld n=%lld)", (long long)m, (long long)n);
    return TT_ERR_ARG;
  }
  if (n > 1024) {
    set_error("qr: n = %lld > 1024 unsupported", (long long)n);
    return TT_ERR_ARG;
  }
  const int ni = int(n);
  DBuf T1, T2, Gm, Rinv, Rk, Racc, Rtmp, gw;
  TTR_TRY(dalloc(T1, size_t(m) * n, s));
  TTR_TRY(dalloc(T2, size_t(m) * n, s));
  TTR_TRY(dalloc(Gm, size_t(n) * n, s));
  TTR_TRY(dalloc(Rinv, size_t(n) * n, s));
  const bool big = ni * ni > kSmemLimitDoubles;
  if (big) TTR_TRY(dalloc(gw, size_t(n) * n, s));
  if (R) {
    TTR_TRY(dalloc(Rk, size_t(n) * n, s));
    TTR_TRY(dalloc(Racc, size_t(n) * n, s));
    TTR_TRY(dalloc(Rtmp, size_t(n) * n, s));
  }
  TTR_CUDA(cudaMemsetAsync(c.flags.p, 0, sizeof(int), s));  // flags[0]: this QR's breakdown
  const size_t shm = big ? 0 : size_t(ni) * ni * sizeof(double);
  static bool attr = false;
  if (!attr) {
    TTR_CUDA(cudaFuncSetAttribute(chol_inv_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimitDoubles * 8));
    TTR_CUDA(cudaFuncSetAttribute(chol_inv_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimitDoubles * 8));
    attr = true;
  }
  auto chol = ni <= 160 ? chol_inv_kernel<5> : chol_inv_kernel<32>;
  const int mi = int(m);
  const double* src = A;
  double* bufs[3] = {T1.p, T2.p, Q};
  for (int pass = 0; pass < 3; ++pass) {
    // Gram G = op(src)^T op(src)
    if (pass == 0 && trans) {
      TTR_TRY(gemm1(c, false, true, ni, ni, mi, 1.0, src, int(lda), src, int(lda), 0.0, Gm.p,
                    ni, s));
    } else {
      const int ld = pass == 0 ? int(lda) : mi;
      TTR_TRY(gemm1(c, true, false, ni, ni, mi, 1.0, src, ld, src, ld, 0.0, Gm.p, ni, s));
    }
    chol<<<1, kCholThreads, shm, s>>>(Gm.p, ni, m, pass == 0 ? 1 : (pass == 2 ? 2 : 0),
                                                 Rinv.p, R ? Rk.p : nullptr, gw.p, c.flags.p);
    TTR_TRY(launched());
    // Q_{pass} = op(src) * Rinv
    if (pass == 0 && trans) {
      TTR_TRY(gemm1(c, true, false, mi, ni, ni, 1.0, src, int(lda), Rinv.p, ni, 0.0, bufs[pass],
                    mi, s));
    } else {
      const int ld = pass == 0 ? int(lda) : mi;
      TTR_TRY(gemm1(c, false, false, mi, ni, ni, 1.0, src, ld, Rinv.p, ni, 0.0, bufs[pass], mi,
                    s));
    }
    if (R) {
      if (pass == 0) {
        TTR_CUDA(cudaMemcpyAsync(Racc.p, Rk.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice,
                                 s));
      } else {
        // Racc = Rk * Racc
        TTR_TRY(gemm1(c, false, false, ni, ni, ni, 1.0, Rk.p, ni, Racc.p, ni, 0.0, Rtmp.p, ni, s));
        std::swap(Racc, Rtmp);
      }
    }
    src = bufs[pass];
  }
  if (R) {
    TTR_CUDA(cudaMemcpyAsync(R, Racc.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  }
  // fallback (no-op unless flags[0] is set)
  DBuf hw, htau;
  TTR_TRY(dalloc(hw, size_t(m) * n, s));
  TTR_TRY(dalloc(htau, size_t(n), s));
  householder_kernel<<<1, kHhThreads, 0, s>>>(A, lda, trans, m, ni, hw.p, htau.p, Q, R, c.flags.p);
  TTR_TRY(launched());
  return TT_OK;
}

// ============================================================== Jacobi SVD
namespace {

constexpr int kJacThreads = 1024;

// One-sided (Hestenes) Jacobi on the columns of W (m x n, ld m), V (n x n) accumulates
// the rotations.  Cyclic round-robin ordering; a warp owns a pair per turn.
__global__ void __launch_bounds__(kJacThreads)
    jacobi_kernel(const double* __restrict__ A, int64_t lda, int m, int n,
                  double* __restrict__ Wg, double* __restrict__ Vg,
                  double* __restrict__ AV, double* __restrict__ Vout,
                  double* __restrict__ sigma, int max_sweeps, int* flags) {
  extern __shared__ double sh[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = kJacThreads / 32;
  const bool w_in_smem = (m * n + n * n) <= kSmemLimitDoubles;
  const bool wonly_smem = !w_in_smem && (m * n) <= kSmemLimitDoubles;
  double* W = (w_in_smem || wonly_smem) ? sh : Wg;
  double* V = w_in_smem ? sh + m * n : Vg;
  const int np = (n + 1) & ~1;          // even count (a dummy column when n is odd)
  __shared__ int perm[1026];
  __shared__ int s_rot;
  for (int e = tid; e < m * n; e += kJacThreads) {
    const int i = e % m, j = e / m;
    W[e] = A[i + int64_t(j) * lda];
  }
  for (int e = tid; e < n * n; e += kJacThreads) V[e] = ((e % n) == (e / n)) ? 1.0 : 0.0;
  for (int e = tid; e < np; e += kJacThreads) perm[e] = e;
  __syncthreads();
  const double tol = 1e-15;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    int rotated = 0;
    for (int round = 0; round < np - 1; ++round) {
      for (int pi = warp; pi < np / 2; pi += nw) {
        int p = perm[pi], q = perm[np - 1 - pi];
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
        if (al == 0.0 || be == 0.0 || !(fabs(ga) > tol * sqrt(al) * sqrt(be))) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int i = lane; i < m; i += 32) {
          const double x = ap[i], y = aq[i];
          ap[i] = cs * x - sn * y;
          aq[i] = sn * x + cs * y;
        }
        double* vp = V + int64_t(p) * n;
        double* vq = V + int64_t(q) * n;
        for (int i = lane; i < n; i += 32) {
          const double x = vp[i], y = vq[i];
          vp[i] = cs * x - sn * y;
          vq[i] = sn * x + cs * y;
        }
        rotated = 1;
      }
      __syncthreads();
      // rotate the tournament: keep perm[0], shift the rest
      if (tid == 0) {
        const int last = perm[np - 1];
        for (int k = np - 1; k > 1; --k) perm[k] = perm[k - 1];
        perm[1] = last;
      }
      __syncthreads();
    }
    if (rotated) atomicOr(&s_rot, 1);
    __syncthreads();
    if (!s_rot) break;
    if (sweep == max_sweeps - 1 && tid == 0) atomicOr(&flags[3], 2);
    __syncthreads();
  }
  // sigma_j = ||w_j||, sort descending (stable by index), write AV, V, sigma
  __shared__ double nrm[1024];
  for (int j = warp; j < n; j += nw) {
    double s2 = 0.0;
    for (int i = lane; i < m; i += 32) s2 += W[i + int64_t(j) * m] * W[i + int64_t(j) * m];
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
    for (int i = lane; i < m; i += 32) AV[i + int64_t(rank) * m] = W[i + int64_t(j) * m];
    for (int i = lane; i < n; i += 32) Vout[i + int64_t(rank) * n] = V[i + int64_t(j) * n];
    if (lane == 0) sigma[rank] = sj;
  }
}

__global__ void eps_rank_kernel(const double* __restrict__ sigma, int n, const double* eps_dev,
                                double eps_host, int rmax, int* dst) {
  if (threadIdx.x != 0) return;
  const double eps = eps_dev ? *eps_dev : eps_host;
  int k = n;
  if (eps > 0.0) {
    double tail = 0.0;
    for (int i = n - 1; i > 0; --i) {
      const double t2 = tail + sigma[i] * sigma[i];
      if (sqrt(t2) <= eps) { tail = t2; k = i; } else break;
    }
  }
  if (rmax > 0 && k > rmax) k = rmax;
  if (k < 1) k = 1;
  if (k > n) k = n;
  *dst = k;
}

__global__ void fro_norm_kernel(const double* __restrict__ x, int64_t n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * x[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = sqrt(s);
}

__global__ void transpose_kernel(const double* __restrict__ src, int64_t rows, int64_t cols,
                                 int64_t lds, double* __restrict__ dst, int64_t ldd) {
  __shared__ double tile[32][33];
  const int64_t r0 = int64_t(blockIdx.x) * 32, c0 = int64_t(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < rows && c < cols) tile[k][threadIdx.x] = src[r + c * lds];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int64_t c = c0 + threadIdx.x, r = r0 + k;   // dst(c, r) = src(r, c)
    if (r < rows && c < cols) dst[c + r * ldd] = tile[threadIdx.x][k];
  }
}

__global__ void fill_zero_kernel(double* p, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i] = 0.0;
}

}  // namespace

int svd_jacobi(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* AV,
               double* V, double* sigma, cudaStream_t s) {
  if (m < n || n < 1 || n > 1024) {
    set_error("svd_jacobi: need 1 <= n <= min(m, 1024) (m=%lld n=%lld)", (long long)m,
              (long long)n);
    return TT_ERR_ARG;
  }
  static bool attr = false;
  if (!attr) {
    TTR_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimitDoubles * 8));
    attr = true;
  }
  const int64_t wn = m * n, vn = n * n;
  size_t shm = 0;
  DBuf Wg, Vg;
  if (wn + vn <= kSmemLimitDoubles) {
    shm = size_t(wn + vn) * 8;
  } else if (wn <= kSmemLimitDoubles) {
    shm = size_t(wn) * 8;
    TTR_TRY(dalloc(Vg, size_t(vn), s));
  } else {
    TTR_TRY(dalloc(Wg, size_t(wn), s));
    TTR_TRY(dalloc(Vg, size_t(vn), s));
  }
  jacobi_kernel<<<1, kJacThreads, shm, s>>>(A, lda, int(m), int(n), Wg.p, Vg.p, AV, V, sigma, 40,
                                           c.flags.p);
  return launched();
}

int eps_rank_dev(Ctx& c, const double* sigma, int n, const double* eps_dev, double eps_host,
                 int rmax, int* dst, cudaStream_t s) {
  eps_rank_kernel<<<1, 32, 0, s>>>(sigma, n, eps_dev, eps_host, rmax, dst);
  return launched();
}

int fro_norm(Ctx& c, const double* x, int64_t n, double* out, cudaStream_t s) {
  fro_norm_kernel<<<1, 1024, 0, s>>>(x, n, out);
  return launched();
}

int transpose(Ctx& c, const double* src, int64_t rows, int64_t cols, int64_t lds, double* dst,
              int64_t ldd, cudaStream_t s) {
  dim3 grid(unsigned((rows + 31) / 32), unsigned((cols + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(src, rows, cols, lds, dst, ldd);
  return launched();
}

int fill_zero(Ctx& c, double* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return TT_OK;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8));
  fill_zero_kernel<<<blocks, 256, 0, s>>>(p, n);
  return launched();
}

}  // namespace ttr
