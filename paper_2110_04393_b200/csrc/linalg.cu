// Dense building blocks of the sweep besides the GEMM:
//  * Philox4x32-10 Gaussian fill of the sketch cores (Def. 3.1; R9)
//  * shifted CholeskyQR3 pieces: Cholesky + triangular inverse of the Gram (one CTA)
//  * Householder QR fallback (one CTA, only when CholeskyQR breaks down)
//  * one-sided Jacobi SVD (one CTA) for the truncation step (R3)
//  * eps-rank, Frobenius norm, transpose, fill
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

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

// The slab [i_lo, i_lo + I_loc) of mode index i of an r0 x I_g x r1 Gaussian core:
// element (a, il, b) is element e = a + r0 (i_lo + il + I_g b) of the full core,
// i.e. number e & 1 of Philox pair e >> 1 -- the same bits as philox_fill_kernel.
__global__ void philox_fill_slab_kernel(double* __restrict__ out, int64_t r0, int64_t I_loc,
                                        int64_t r1, int64_t i_lo, int64_t I_g, uint32_t key0,
                                        uint32_t key1, uint32_t n, uint32_t tag, double scale) {
  const int64_t cnt = r0 * I_loc * r1;
  for (int64_t x = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; x < cnt;
       x += int64_t(gridDim.x) * blockDim.x) {
    const int64_t a = x % r0, il = (x / r0) % I_loc, b = x / (r0 * I_loc);
    const int64_t e = a + r0 * (i_lo + il + I_g * b);
    const int64_t k = e >> 1;
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
    out[x] = (e & 1) ? (r * sn) * scale : (r * cs) * scale;
  }
}

}  // namespace

int philox_fill_slab(Ctx& c, double* out, int64_t r0, int64_t I_loc, int64_t r1, int64_t i_lo,
                     int64_t I_g, uint64_t seed, uint32_t n, uint32_t tag, double scale,
                     cudaStream_t s) {
  const int64_t cnt = r0 * I_loc * r1;
  if (cnt <= 0) return TT_OK;
  const int blocks = int(std::min<int64_t>((cnt + 255) / 256, int64_t(c.sm_count) * 16));
  philox_fill_slab_kernel<<<blocks, 256, 0, s>>>(out, r0, I_loc, r1, i_lo, I_g,
                                                 uint32_t(seed & 0xffffffffu), uint32_t(seed >> 32),
                                                 n, tag, scale);
  return launched();
}

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

constexpr int kCholThreads = 512;   // generic (n > 160) Cholesky: 128 registers for the inverse's column
constexpr int kSmemLimitDoubles = 26 * 1024;   // 208 KB of dynamic shared memory
constexpr int kCholTsmDoubles = 225 * 1024 / 8;   // generic Cholesky's T_J staging (+ static smem <= 227 KB)

// flags layout (Ctx.flags; see common.cuh):
//  0 = route state of the current QR: 0 plain CholeskyQR2, 1 shifted CholeskyQR3,
//      2 doubly shifted CholeskyQR4, 3 all failed (-> Householder / TSQR)
//  1 = Householder fallback used (sticky)      2 = zero sketch seen (sticky)
//  3 = numeric failure bits (sticky)
//  8.. = counters: 8 CholQR2, 10 sCholQR3, 11 Householder, 12 Jacobi sweeps,
//        13 Jacobi calls, 14 TSQR, 15 sCholQR4
enum CholMode : int {
  CH_FIRST = 0,    // route 0, pass 1 (input):  failure -> route 1
  CH_SECOND = 1,   // route 0, pass 2:          failure or |diag R - 1| > kDevTol -> route 1
  CH_THIRD = 2,    // (unused)
  CH_SHIFT = 3,    // route 1, pass 1 (shifted): failure -> route 3
  CH_SPLAIN = 4,   // route 1, pass 2:          failure -> route 2
  CH_SLAST = 5,    // route 1, pass 3:          failure or deviation -> route 2
  CH_SHIFT2 = 6,   // route 2, pass 2 (shifted again): failure -> route 3
  CH_S2PLAIN = 7,  // route 2, pass 3:          failure -> route 3
  CH_S2LAST = 8,   // route 2, pass 4:          failure or deviation -> route 3
  CH_SHIFT1B = 9,  // route 2, pass 1 (shifted, on the input again): failure -> route 3
  // robust R-only QR (truncation): no routes, never fails on a finite input
  CH_RSHIFT = 10,  // passes 1, 2: shifted (compress kappa)
  CH_RCLAMP = 11,  // passes 3, 4: plain, pivots below tau = 64 n u max(diag G)
                   // (numerically null directions only) clamped to tau
};
constexpr double kDevTol = 0.05;
constexpr int kNearIdFlag = 20;   // flags[20]: 1 = run the full Cholesky for pass 4 (R only)
// mode bit of the R-only QR: a plain pass whose pivots spread by more than
// 2^20 (kappa(Q1)^2 u no longer small) cannot give an accurate R -> next route
constexpr int kStrict = 0x100;
constexpr double kStrictRatio = 0x1p-20;

// passes whose input should already be close to orthonormal (|diag R - 1| test);
// the plain pass right after a shifted one legitimately is not
__device__ __forceinline__ bool needs_dev(int mode) {
  return mode == CH_SECOND || mode == CH_SLAST || mode == CH_S2LAST;
}

// route state machine of the CholeskyQR family (flags[0], see above)
__device__ __forceinline__ void route_update(int* flags, int mode, bool bad, double dev) {
  const bool fail = bad || (needs_dev(mode) && !(dev <= kDevTol));
  switch (mode) {
    case CH_FIRST:
      if (bad) flags[0] = 1;
      break;
    case CH_SECOND:
      if (fail) flags[0] = 1;
      else flags[8] += 1;
      break;
    case CH_SHIFT:
      if (bad) flags[0] = 3;
      break;
    case CH_SPLAIN:
      if (fail) flags[0] = 2;
      break;
    case CH_SLAST:
      if (fail) flags[0] = 2;
      else flags[10] += 1;
      break;
    case CH_SHIFT1B:
    case CH_SHIFT2:
    case CH_S2PLAIN:
      if (fail) flags[0] = 3;
      break;
    case CH_S2LAST:
      if (fail) flags[0] = 3;
      else flags[15] += 1;
      break;
    case CH_RSHIFT:
    case CH_RCLAMP:
      if (bad) atomicOr(&flags[3], 1);   // non-finite input even with the shift
      break;
  }
}

// generic (n > 163) Cholesky's shared memory: the blocked inverse's T_J staging
// (32 x 34 per block column) or the factorisation's X_kk (32 x 33) + k-major panel
__host__ __device__ __forceinline__ int chol_panel_ld(int n) {
  const int n8 = (n + 7) & ~7;
  return n8 + ((20 - n8 % 16) % 16);
}
__host__ __device__ __forceinline__ int chol_tsm_doubles(int n) {
  const int a = ((n + 31) / 32) * 32 * 34, b = 32 * 33 + 32 * chol_panel_ld(n);
  return a > b ? a : b;
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// G (n x n, ld n, symmetric) -> Rinv (upper, ld n) with G + shift*I = R^T R, and
// optionally L = R^T (lower, ld n).  Shift (CH_SHIFT only) = 11(mn + n(n+1))u * trace(G) (shifted
// CholeskyQR3, Fukaya et al.).  Runs iff *gate == gate_val.
template <int QN>
__global__ void __launch_bounds__(kCholThreads)
    chol_inv_kernel(const double* __restrict__ G, int n, int64_t m, int mode,
                    double* __restrict__ Rinv, double* __restrict__ Rout,
                    double* __restrict__ gwork, int* __restrict__ flags, const int* gate,
                    int gate_val) {
  if (gate && *gate != gate_val) return;
  extern __shared__ double sh[];
  const bool in_smem = (n * n <= kSmemLimitDoubles);
  double* L = in_smem ? sh : gwork;
  // L in global memory: the dynamic shared memory (if any) stages the blocked
  // inverse's T_J blocks (32 x 34 doubles per block column, n <= 832)
  double* Tsm = in_smem ? nullptr : sh;
  const bool tsm_ok = !in_smem && chol_tsm_doubles(n) <= kCholTsmDoubles;
  if (!tsm_ok) Tsm = nullptr;
  __shared__ double s_shift, s_tau;
  __shared__ int s_bad, s_zero;
  const int tid = threadIdx.x;
  if (tid == 0) { s_bad = 0; s_zero = 0; }
  // trace for the shift and the zero test; max diagonal for the clamp level
  if (tid < 32) {
    double tr = 0.0, dmx = 0.0;
    for (int i = tid; i < n; i += 32) {
      tr += G[i + int64_t(i) * n];
      dmx = fmax(dmx, G[i + int64_t(i) * n]);
    }
    for (int o = 16; o; o >>= 1) {
      tr += __shfl_xor_sync(0xffffffffu, tr, o);
      dmx = fmax(dmx, __shfl_xor_sync(0xffffffffu, dmx, o));
    }
    if (tid == 0) {
      // CH_RCLAMP: a pivot below tau = 64 n u max diag G (a numerically null
      // direction) is clamped to tau, as in the blocked kernels
      s_tau = ((mode & 0xff) == CH_RCLAMP) ? 64.0 * n * 0x1p-53 * dmx : 0.0;
      if (!isfinite(tr)) atomicOr(&flags[3], 4);   // NaN/Inf in the input (TT_ERR_NONFINITE)
      if (!(tr > 0.0)) {
        if (tr == 0.0) { atomicOr(&flags[2], 1); s_zero = 1; }   // Y_n == 0: zero sum (R16)
        s_bad = 1;
      }
      const double u = 0x1p-53;
      s_shift = ((mode & 0xff) == CH_SHIFT || (mode & 0xff) == CH_SHIFT2 ||
                     (mode & 0xff) == CH_SHIFT1B || (mode & 0xff) == CH_RSHIFT)
                    ? 11.0 * (double(m) * n + double(n) * (n + 1)) * u * tr : 0.0;
    }
  }
  __syncthreads();
  const double shift = s_shift;
  for (int e = tid; e < n * n; e += kCholThreads) {
    const int i = e % n, j = e / n;
    L[e] = (i >= j) ? G[e] + ((i == j) ? shift : 0.0) : 0.0;
  }
  __syncthreads();
  const int warp0 = tid >> 5, lane0 = tid & 31;
  constexpr int kNW = kCholThreads / 32;
  if (!in_smem && Tsm) {
    // ---- L in global memory (n > 163): right-looking, 32-column blocks on DMMA.
    //  (a) warp 0 factors the diagonal block in registers (lane = row; clamped
    //      pivots decoupled as below) and forms its inverse X_kk (lane = column),
    //  (b) the panel L_ik = A_ik X_kk^T on DMMA (rows in 8-row tiles over the
    //      warps), copied k-major into shared memory,
    //  (c) the trailing lower 8 x 8 tiles A_ij -= L_ik L_jk^T on DMMA from the
    //      shared panel (each tile read and written once per block column).
    // The 8-column panel loop below took 5.9 ms at n = 600 (L2 latency per
    // rank-1 update pass).
    double* Xk = Tsm;                          // 32 x 33: X_kk (row j zeroed if clamped)
    double* Pn = Tsm + 32 * 33;                // panel, k-major: Pn[k * pld + r]
    const int pld = chol_panel_ld(n);
    const int g = lane0 >> 2, t4 = lane0 & 3;
    for (int k0 = 0; k0 < n; k0 += 32) {
      const int kb = min(32, n - k0);
      if (warp0 == 0) {
        const int i = lane0;
        double a[32];
#pragma unroll
        for (int q = 0; q < 32; ++q)
          a[q] = (i < kb && q <= i && q < kb) ? L[(k0 + i) + int64_t(k0 + q) * n] : 0.0;
        int bad = 0;
        unsigned clmask = 0u;
        double dinv = 1.0;   // 1 / L_ii of this lane's row (for X_kk)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < kb) {
            double piv = __shfl_sync(0xffffffffu, a[j], j);
            const bool cl = s_tau > 0.0 && isfinite(piv) && !(piv > s_tau);
            if (cl) piv = s_tau;
            const bool okp = piv > 0.0 && isfinite(piv);
            bad |= !okp;
            const double d = okp ? sqrt(piv) : 1.0;
            if (cl) clmask |= 1u << j;
            const double l = (i > j) ? (cl ? 0.0 : a[j] / d) : (i == j ? d : 0.0);
            a[j] = l;
            if (i == j) dinv = 1.0 / d;
#pragma unroll
            for (int q = j + 1; q < 32; ++q) {
              const double lq = __shfl_sync(0xffffffffu, l, q);
              if (q <= i) a[q] -= l * lq;
            }
          }
        }
        // L_kk back to global (lower), diagonal included
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (i < kb && q <= i && q < kb) L[(k0 + i) + int64_t(k0 + q) * n] = a[q];
        if (bad && i == 0) s_bad = 1;
        // X_kk = L_kk^{-1}: lane c solves column c (x_j for j >= c)
        double x[32];
#pragma unroll
        for (int q = 0; q < 32; ++q) x[q] = (q == i) ? 1.0 : 0.0;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const double djinv = __shfl_sync(0xffffffffu, dinv, j);
          if (j < kb) {
            const double xj = x[j] * djinv;
            x[j] = xj;
#pragma unroll
            for (int q = j + 1; q < 32; ++q) {
              const double lqj = __shfl_sync(0xffffffffu, a[j], q);   // L(q, j) from lane q
              x[q] -= lqj * xj;
            }
          }
        }
        // Xk[r * 33 + c] = X(r, c); rows of clamped directions zeroed (their
        // panel column stays 0)
#pragma unroll
        for (int q = 0; q < 32; ++q) Xk[q * 33 + i] = ((clmask >> q) & 1u) ? 0.0 : x[q];
      }
      __syncthreads();
      const int r0 = k0 + kb, nr = n - r0;
      if (nr > 0) {
        // (b) panel: rows r0 .. n-1 in 8-row tiles, one warp per tile (all four
        // column tiles: the tile's A_ik is read before any of it is overwritten)
        const int rt8 = (nr + 7) / 8;
        for (int rt = warp0; rt < rt8; rt += kNW) {
          const int row = r0 + 8 * rt + g;
          double a[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int kc = 4 * kk + t4;
            a[kk] = (row < n && kc < kb) ? L[row + int64_t(k0 + kc) * n] : 0.0;
          }
          double c[4][2];
#pragma unroll
          for (int ct = 0; ct < 4; ++ct) {
            c[ct][0] = c[ct][1] = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              dmma884(c[ct][0], c[ct][1], a[kk], Xk[(8 * ct + g) * 33 + 4 * kk + t4]);   // X(c, kc)
          }
          __syncwarp();
          if (row < n) {
#pragma unroll
            for (int ct = 0; ct < 4; ++ct)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int col = 8 * ct + 2 * t4 + e;
                if (col < kb) {
                  L[row + int64_t(k0 + col) * n] = c[ct][e];
                  Pn[col * pld + (row - r0)] = c[ct][e];
                }
              }
          }
        }
        // zero panel columns past kb (k-range of the trailing DMMAs is 32)
        for (int e = tid; e < (32 - kb) * nr; e += kCholThreads)
          Pn[(kb + e / nr) * pld + (e % nr)] = 0.0;
        __syncthreads();
        // (c) trailing lower tiles (ti >= tj) of rows/cols r0 .. n-1
        const int nt = (nr + 7) / 8, ntiles = nt * (nt + 1) / 2;
        for (int u = warp0; u < ntiles; u += kNW) {
          int ti = int((sqrtf(8.0f * u + 1.0f) - 1.0f) * 0.5f);
          while ((ti + 1) * (ti + 2) / 2 <= u) ++ti;
          while (ti * (ti + 1) / 2 > u) --ti;
          const int tj = u - ti * (ti + 1) / 2;
          const int row = r0 + 8 * ti + g, colb = r0 + 8 * tj;
          const int c2 = colb + 2 * t4;
          double o0 = 0.0, o1 = 0.0;
          if (row < n && c2 < n) o0 = L[row + int64_t(c2) * n];
          if (row < n && c2 + 1 < n) o1 = L[row + int64_t(c2 + 1) * n];
          double a[8], b[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int kc = 4 * kk + t4;
            a[kk] = Pn[kc * pld + (8 * ti + g)];   // L(row, k0 + kc)
            b[kk] = Pn[kc * pld + (8 * tj + g)];   // L(colb + g, k0 + kc)
          }
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) dmma884(c0, c1, a[kk], b[kk]);
          if (row < n) {
            if (c2 < n && c2 <= row) L[row + int64_t(c2) * n] = o0 - c0;
            if (c2 + 1 < n && c2 + 1 <= row) L[row + int64_t(c2 + 1) * n] = o1 - c1;
          }
        }
      }
      __syncthreads();
    }
  } else {
  // right-looking Cholesky, lower L in column-major L[i + j n], in panels of 8
  // columns: the panel is factored column by column, then the trailing lower
  // part takes the panel's 8 rank-1 updates in one pass (each L(i, k) read and
  // written once per panel instead of once per column; one warp per column,
  // lanes over rows: coalesced).  The subtractions happen in the same order as
  // column by column, so the bits are those of the unblocked algorithm.
  for (int j0 = 0; j0 < n; j0 += 8) {
    const int jw = min(8, n - j0);
    for (int jj = 0; jj < jw; ++jj) {
      const int j = j0 + jj;
      double djj = L[j + j * n];
      // a clamped (numerically null) direction is also decoupled: its column
      // below the pivot is zeroed, so rounding-level couplings divided by
      // sqrt(tau) cannot grow through the later pivots (with hundreds of null
      // directions -- a rank-deficient assembled sum -- they overflowed)
      const bool clj = s_tau > 0.0 && isfinite(djj) && !(djj > s_tau);
      if (clj) djj = s_tau;
      const bool okp = djj > 0.0 && isfinite(djj);
      const double d = okp ? sqrt(djj) : 1.0;
      if (!okp && tid == 0) s_bad = 1;
      const double inv = clj ? 0.0 : 1.0 / d;
      for (int i = j + 1 + tid; i < n; i += kCholThreads) L[i + j * n] *= inv;
      __syncthreads();
      if (tid == 0) L[j + j * n] = d;
      for (int k = j + 1 + warp0; k < j0 + jw; k += kNW) {   // the rest of the panel
        const double lkj = L[k + j * n];
        for (int i = k + lane0; i < n; i += 32) L[i + k * n] -= L[i + j * n] * lkj;
      }
      __syncthreads();
    }
    for (int k = j0 + jw + warp0; k < n; k += kNW) {         // trailing part
      double lk[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) lk[jj] = (jj < jw) ? L[k + (j0 + jj) * n] : 0.0;
      for (int i = k + lane0; i < n; i += 32) {
        double acc = L[i + k * n];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (jj < jw) acc -= L[i + (j0 + jj) * n] * lk[jj];
        L[i + k * n] = acc;
      }
    }
    __syncthreads();
  }
  }
  const int warp = tid >> 5, lane = tid & 31;
  if (!in_smem && Tsm) {
    // X = L^{-1} by 32 x 32 blocks on DMMA (L in global memory / L2): the
    // diagonal blocks' inverses X_II first (one warp each, forward substitution,
    // lane = column), then block row by block row
    //   X_IJ = -X_II sum_{K=J}^{I-1} L_IK X_KJ   (J < I),
    // the sums for all J of a row at once (8 x 8 tiles over the warps, the
    // fragments of a 32-wide k-block loaded before its 8 DMMAs), staged in shared
    // memory, then multiplied by X_II.  X is kept transposed in Rinv (Rinv(c, i)
    // = X(i, c)).  The column-oriented substitution below read all of L once per
    // column of X (33 ms of a 39 ms call at n = 600).
    const int nb = (n + 31) / 32;
    for (int e = tid; e < n * n; e += kCholThreads) {   // Rinv's strictly lower part
      const int r = e % n, c2 = e / n;
      if (r > c2) Rinv[e] = 0.0;
    }
    for (int I = warp; I < nb; I += kNW) {
      const int r0 = 32 * I, bs = min(32, n - r0);
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) x[i] = (i == lane) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        if (k < bs) {
          const double xk = x[k] / L[(r0 + k) + int64_t(r0 + k) * n];
          x[k] = xk;
#pragma unroll
          for (int i = k + 1; i < 32; ++i)
            if (i < bs) x[i] -= L[(r0 + i) + int64_t(r0 + k) * n] * xk;
        }
      }
      if (lane < bs)
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i >= lane && i < bs) Rinv[(r0 + lane) + int64_t(r0 + i) * n] = x[i];
    }
    __syncthreads();
    const int g = lane >> 2, t4 = lane & 3;
    constexpr int kLdT = 34;
    for (int I = 1; I < nb; ++I) {
      const int rI = 32 * I;
      // T_J = sum_{K=J}^{I-1} L_IK X_KJ, J < I: unit = (J, 8 x 8 tile)
      for (int u = warp; u < I * 16; u += kNW) {
        const int J = u >> 4, tr = (u >> 2) & 3, tc = u & 3;
        const int row = rI + 8 * tr + g, col = 32 * J + 8 * tc + g;
        double c0 = 0.0, c1 = 0.0;
        for (int K = J; K < I; ++K) {
          double a[8], b[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int k = 32 * K + 4 * kk + t4;
            a[kk] = (row < n && k < n) ? L[row + int64_t(k) * n] : 0.0;
            b[kk] = (col < n && k < n) ? Rinv[col + int64_t(k) * n] : 0.0;   // X(k, col)
          }
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) dmma884(c0, c1, a[kk], b[kk]);
        }
        double* T = Tsm + J * (32 * kLdT);
        const int rr = 8 * tr + g, cc = 8 * tc + 2 * t4;
        T[rr + cc * kLdT] = c0;
        T[rr + (cc + 1) * kLdT] = c1;
      }
      __syncthreads();
      // X_IJ = -X_II T_J
      for (int u = warp; u < I * 16; u += kNW) {
        const int J = u >> 4, tr = (u >> 2) & 3, tc = u & 3;
        const int row = rI + 8 * tr + g;
        const double* T = Tsm + J * (32 * kLdT);
        double a[8], b[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int k = 4 * kk + t4;
          a[kk] = (row < n && rI + k < n) ? Rinv[(rI + k) + int64_t(row) * n] : 0.0;   // X(row, rI + k)
          b[kk] = T[k + (8 * tc + g) * kLdT];
        }
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) dmma884(c0, c1, a[kk], b[kk]);
        const int col = 32 * J + 8 * tc + 2 * t4;
        if (row < n) {
          if (col < n) Rinv[col + int64_t(row) * n] = -c0;
          if (col + 1 < n) Rinv[(col + 1) + int64_t(row) * n] = -c1;
        }
      }
      __syncthreads();
    }
  } else {
  // X = L^{-1} (lower), one warp per column, column-oriented forward substitution;
  // Rinv = X^T (upper).  x lives in registers: lane owns rows lane + 32 q.
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
  }
  __syncthreads();
  if (Rout) {
    for (int e = tid; e < n * n; e += kCholThreads) {
      const int i = e % n, j = e / n;     // Lout = R^T (lower)
      Rout[e] = (i >= j) ? L[i + j * n] : 0.0;
    }
  }
  __syncthreads();
  if (tid == 0 && !s_zero && !(flags[2] & 1)) {
    int bad = s_bad;
    double dev = 0.0, dmin = INFINITY, dmax = 0.0;
    for (int i = 0; i < n; ++i) {
      const double d = fabs(L[i + i * n]);
      dmin = fmin(dmin, d);
      dmax = fmax(dmax, d);
      if (needs_dev(mode & 0xff)) dev = fmax(dev, fabs(L[i + i * n] - 1.0));
    }
    if ((mode & kStrict) && !(dmin >= dmax * kStrictRatio)) bad = 1;
    route_update(flags, mode & 0xff, bad, dev);
  }
}

constexpr int kBlkThreads = 512;

// optional phase timing of chol_blk_kernel (build with -DTTR_CHOL_PROF): thread 0
// adds clock64 deltas / 64 of C1, C2, C3, I0, I-phase to flags[32..36]
#ifdef TTR_CHOL_PROF
#define CHOL_PROF(slot)                                              \
  do {                                                               \
    if (threadIdx.x == 0) {                                          \
      const long long t__ = clock64();                               \
      atomicAdd(&flags[32 + (slot)], int((t__ - prof_t) >> 6));     \
      prof_t = t__;                                                  \
    }                                                                \
  } while (0)
#else
#define CHOL_PROF(slot) do { } while (0)
#endif


// leading dimension of the Cholesky working matrix: >= round8(n) + 4 and
// == 4 (mod 16) doubles, so DMMA fragment loads (8 rows x 4 columns) are
// conflict-free
__host__ __device__ __forceinline__ int chol_ld(int n) {
  const int n8 = (n + 7) & ~7;
  return n8 + ((20 - n8 % 16) % 16);
}

// Blocked Cholesky + in-place triangular inverse for n <= 32*NB (one CTA of
// 512 threads, 16 warps).  Same contract and flags as chol_inv_kernel.  The
// working matrix S (ld = chol_ld(n), columns padded to a multiple of 8) holds L
// in its lower triangle.  Per 32-column block k:
//  C1  warp 0 factors the diagonal block: lane i keeps the not yet eliminated
//      part of row i in registers, shifted left after every pivot (static
//      register indices in a rolled loop: fully unrolled elimination code runs
//      once per block and thrashes the instruction cache);
//  C2  panel L_ik = A_ik L_kk^{-T} by forward substitution, 4 threads per row
//      (8 columns each, quad shuffles between the quarters);
//  C3  trailing update A_ij -= L_ik L_jk^T on 8x8 DMMA tiles (m8n8k4).
// Then X = L^{-1} in place: I0 every diagonal block X_kk at once (one warp per
// block, column-wise forward substitution, parked in the unused upper
// triangle), then block columns right to left (LAPACK dtrtri order), both on
// DMMA tiles: I1 A21 <- X22 A21, I2 A21 <- -A21 X11; I3 X11 into the lower
// triangle.
template <int NB>
__global__ void __launch_bounds__(kBlkThreads, 1)
    chol_blk_kernel(const double* __restrict__ G, int n, int64_t m, int mode,
                    double* __restrict__ Rinv, double* __restrict__ Rout,
                    int* __restrict__ flags, const int* gate, int gate_val) {
  if (gate && *gate != gate_val) return;
  extern __shared__ double S[];
  __shared__ double rdiag[32 * NB];   // 1 / L(i, i)
  __shared__ double colb[128];        // pivot column broadcast (C1), doubled, x2 buffers
  __shared__ double ttmp[256];        // 16 x 16 product L21 X11 of the diagonal-block inverse
  __shared__ double s_tr, s_dmax;
  __shared__ int s_bad, s_zero, s_clamped;
  constexpr int NW = kBlkThreads / 32;
  const int ld = chol_ld(n);
  const int n8 = (n + 7) & ~7, nt8 = n8 / 8;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;   // DMMA fragment coordinates
  const int nb = (n + 31) / 32;
  const int md = mode & 0xff;
  if (tid == 0) { s_bad = 0; s_zero = 0; s_clamped = 0; }
  if (tid < 32) {
    double tr = 0.0, dmax = 0.0;
    for (int i = tid; i < n; i += 32) {
      const double gi = G[i + int64_t(i) * n];
      tr += gi;
      dmax = fmax(dmax, gi);
    }
    for (int o = 16; o; o >>= 1) {
      tr += __shfl_xor_sync(0xffffffffu, tr, o);
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if (tid == 0) {
      if (!isfinite(tr)) atomicOr(&flags[3], 4);   // NaN/Inf in the input (TT_ERR_NONFINITE)
      if (!(tr > 0.0)) {
        if (tr == 0.0) { atomicOr(&flags[2], 1); s_zero = 1; }   // Y_n == 0: zero sum (R16)
        s_bad = 1;
      }
      s_tr = tr;
      s_dmax = dmax;
    }
  }
  __syncthreads();
  const bool shifted = md == CH_SHIFT || md == CH_SHIFT2 || md == CH_SHIFT1B || md == CH_RSHIFT;
  const double shift = shifted ? 11.0 * (double(m) * n + double(n) * (n + 1)) * 0x1p-53 * s_tr : 0.0;
  const bool clamp = md == CH_RCLAMP;
  const double tau = 64.0 * n * 0x1p-53 * s_dmax;
#ifdef TTR_CHOL_PROF
  long long prof_t = clock64();
#endif
  // lower triangle of G (+ shift) into S, pads 0; loads batched 8 deep (the
  // loop is latency bound: one L2 round trip per batch, not per element)
  // (2-D loops: no integer division by the runtime n / ld per element)
  for (int j = w; j < n8; j += NW) {
#pragma unroll 4
    for (int i = lane; i < ld; i += 32)
      S[i + j * ld] = (i < n && j < n && i >= j) ? G[i + int64_t(j) * n] + ((i == j) ? shift : 0.0)
                                                 : 0.0;
  }
  __syncthreads();
  CHOL_PROF(5);
#pragma unroll 1
  for (int k = 0; k < nb; ++k) {
    const int k0 = 32 * k, kb = min(32, n - k0);
    // ---- C1 (warp 0): lane i keeps the not yet eliminated part of row i in
    // registers, a[q] = A(i, j0 + q); pivots in groups of 4 with static
    // register offsets, then a shift by 4 (a fully unrolled elimination is ~15k
    // instructions run once per block: instruction-cache bound).  The pivot
    // column is broadcast through shared memory (colb).  The pivot step is
    // branch-free: clamping and the finiteness test are selects, and
    // 1/L_jj = rsqrt(pivot) is MUFU.RSQ64H + two Newton steps (no slow path:
    // pivots are normal numbers here).  Updates of the upper slots (column >
    // row) are harmless garbage.
    if (w == 0) {
      const int i = lane;
      double a[32];
#pragma unroll
      for (int q = 0; q < 32; ++q)
        a[q] = (i < kb && q <= i) ? S[(k0 + i) + (k0 + q) * ld] : 0.0;
      int bad = 0, nclamp = 0;
      const int kb4 = (kb + 3) & ~3;
#pragma unroll 1
      for (int j0 = 0; j0 < kb4; j0 += 4) {
#pragma unroll
        for (int sft = 0; sft < 4; ++sft) {
          const int j = j0 + sft;
          double piv = __shfl_sync(0xffffffffu, a[sft], j);
          piv = (j < kb) ? piv : 1.0;                       // padding pivot
          const bool fin = fabs(piv) <= 1.79e308;           // false for inf / nan
          const bool cl = clamp && fin && !(piv > tau);     // numerically null direction
          piv = cl ? tau : piv;
          nclamp += cl;
          const bool ok = fin && piv > 0.0;
          bad |= !ok;
          const double pv = ok ? piv : 1.0;
          double rd;
          asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(pv));
          rd = rd * fma(-0.5 * pv * rd, rd, 1.5);           // Newton steps for 1/sqrt
          rd = rd * fma(-0.5 * pv * rd, rd, 1.5);
          const double lij = (i > j) ? a[sft] * rd : (i == j ? pv * rd : 0.0);
          if (j < kb && i >= j && i < kb) S[(k0 + i) + (k0 + j) * ld] = lij;
          if (i == j && j < kb) rdiag[k0 + j] = rd;
          colb[i] = lij;          // doubled buffer: colb[j + qq] needs no wrap,
          colb[i + 32] = lij;     // so every load is [base + constant]
          __syncwarp();
          const double* cb = colb + j;
#pragma unroll
          for (int qq = 1; qq < 32 - sft; ++qq) a[sft + qq] = fma(-lij, cb[qq], a[sft + qq]);
          __syncwarp();
        }
#pragma unroll
        for (int q = 0; q < 28; ++q) a[q] = a[q + 4];
        a[28] = a[29] = a[30] = a[31] = 0.0;
      }
      if (lane == 0) {
        if (bad) s_bad = 1;
        if (nclamp) s_clamped += nclamp;
      }
      CHOL_PROF(6);
      // X_kk = L_kk^{-1} (lower), 2 x 2 blocked: lanes 0-15 invert the 16 x 16
      // L11, lanes 16-31 L22 (column-wise forward substitution, lane = column,
      // the column in registers, L rows broadcast from shared memory); then
      // X21 = -X22 (L21 X11) on DMMA tiles.  X(r, c), r > c, is parked at (c, r)
      // in the unused upper triangle of the block, the diagonal is rdiag (the
      // panel below and the inverse phase read it there)
      __syncwarp();
      {
        const int h = lane >> 4, c = lane & 15, o = 16 * h;
        double x[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          double s0 = 0.0, s1 = 0.0;
#pragma unroll
          for (int t = 0; t < r; ++t) {
            const double l = (o + r < kb) ? S[(k0 + o + r) + (k0 + o + t) * ld] : 0.0;
            if (t & 1) s1 = fma(l, x[t], s1);
            else s0 = fma(l, x[t], s0);
          }
          const double rdr = (o + r < kb) ? rdiag[k0 + o + r] : 0.0;
          x[r] = (r < c || o + r >= kb) ? 0.0 : (r == c ? rdr : -rdr * (s0 + s1));
        }
#pragma unroll
        for (int r = 1; r < 16; ++r)
          if (r > c && o + r < kb) S[(k0 + o + c) + (k0 + o + r) * ld] = x[r];
      }
      __syncwarp();
      if (kb > 16) {
        // X11(row, col) / X22(row, col), block-local 0..15, row >= col
        auto x11 = [&](int row, int col) -> double {
          return row < col ? 0.0
                           : (row == col ? rdiag[k0 + row] : S[(k0 + col) + (k0 + row) * ld]);
        };
        auto x22 = [&](int row, int col) -> double {
          if (row < col || 16 + row >= kb) return 0.0;
          return row == col ? rdiag[k0 + 16 + row] : S[(k0 + 16 + col) + (k0 + 16 + row) * ld];
        };
        double tacc[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // T = L21 X11, tile (8 (q >> 1), 8 (q & 1))
          const int R = 8 * (q >> 1), C = 8 * (q & 1);
          tacc[q][0] = tacc[q][1] = 0.0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int kc = 4 * kk + t4;
            const double av = (16 + R + g < kb) ? S[(k0 + 16 + R + g) + (k0 + kc) * ld] : 0.0;
            dmma884(tacc[q][0], tacc[q][1], av, x11(kc, C + g));
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int R = 8 * (q >> 1), C = 8 * (q & 1);
          ttmp[(R + g) + 16 * (C + 2 * t4)] = tacc[q][0];
          ttmp[(R + g) + 16 * (C + 2 * t4 + 1)] = tacc[q][1];
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // X21 = -X22 T
          const int R = 8 * (q >> 1), C = 8 * (q & 1);
          double c0 = 0.0, c1 = 0.0;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const int kc = 4 * kk + t4;
            dmma884(c0, c1, x22(R + g, kc), ttmp[kc + 16 * (C + g)]);
          }
          const int r = R + g, cA = C + 2 * t4;   // X(16 + r, cA) parked at (cA, 16 + r)
          if (16 + r < kb) {
            S[(k0 + cA) + (k0 + 16 + r) * ld] = -c0;
            S[(k0 + cA + 1) + (k0 + 16 + r) * ld] = -c1;
          }
        }
      }
    }
    __syncthreads();
    CHOL_PROF(0);
    if (s_bad) break;
    const int r0 = k0 + kb;   // first row below the block (kb == 32 if r0 < n)
    if (r0 >= n) break;
    // ---- C2: panel L_ik = A_ik X_kk^T on 8x8 DMMA tiles (K = 32); all tiles
    // to registers first (a tile reads the whole 32-column row block it overwrites)
    {
      const int tb = r0 / 8, nrt = nt8 - tb, ntiles = nrt * 4;
      double acc[4][2];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[q][0] = acc[q][1] = 0.0;
        const int tt = w + NW * q;
        if (tt < ntiles) {
          const int R = 8 * (tb + tt / 4), cb = 8 * (tt % 4);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int tl = 4 * kk + t4, cl = cb + g;   // B(tl, cl) = X_kk(cl, tl)
            const double av = S[(R + g) + (k0 + tl) * ld];
            const double bv = (cl < tl) ? 0.0
                              : (cl == tl ? rdiag[k0 + cl] : S[(k0 + tl) + (k0 + cl) * ld]);
            dmma884(acc[q][0], acc[q][1], av, bv);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tt = w + NW * q;
        if (tt < ntiles) {
          const int R = 8 * (tb + tt / 4), C = k0 + 8 * (tt % 4);
          const int r = R + g, cA = C + 2 * t4;
          S[r + cA * ld] = acc[q][0];
          S[r + (cA + 1) * ld] = acc[q][1];
        }
      }
    }
    __syncthreads();
    CHOL_PROF(1);
    // ---- C3: trailing A(r, c) -= sum_t L(r, t) L(c, t) on the lower 8x8 tiles
    {
      const int tb = r0 / 8, nrt = nt8 - tb;
      const int ntiles = nrt * (nrt + 1) / 2;
#pragma unroll 1
      for (int tt = w; tt < ntiles; tt += NW) {
        int tr = int((sqrtf(8.0f * tt + 1.0f) - 1.0f) * 0.5f);   // tt = tr(tr+1)/2 + tc
        while ((tr + 1) * (tr + 2) / 2 <= tt) ++tr;
        while (tr * (tr + 1) / 2 > tt) --tr;
        const int tc = tt - tr * (tr + 1) / 2;
        const int R = 8 * (tb + tr), C = 8 * (tb + tc);
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int tcol = k0 + 4 * kk + t4;
          dmma884(c0, c1, S[(R + g) + tcol * ld], S[(C + g) + tcol * ld]);
        }
        const int r = R + g, cA = C + 2 * t4;
        if (r < n) {
          if (cA < n) S[r + cA * ld] -= c0;
          if (cA + 1 < n) S[r + (cA + 1) * ld] -= c1;
        }
      }
    }
    __syncthreads();
    CHOL_PROF(2);
  }
  __syncthreads();
  const bool bad_final = s_bad;
  // route checks on diag(L); R = L^T before L is overwritten by its inverse
  if (w == 0 && !s_zero) {   // route checks on diag(L), warp-parallel
    double dev = 0.0, dmin = INFINITY, dmax = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double d = fabs(S[i + i * ld]);
      dmin = fmin(dmin, d);
      dmax = fmax(dmax, d);
      dev = fmax(dev, fabs(S[i + i * ld] - 1.0));
    }
    for (int o = 16; o; o >>= 1) {
      dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    }
    if (lane == 0 && !(flags[2] & 1)) {
      int bad2 = bad_final;
      if ((mode & kStrict) && !(dmin >= dmax * kStrictRatio)) bad2 = 1;
      if (s_clamped) flags[16] += 1;   // counter: clamped (rank-deficient) passes
      route_update(flags, md, bad2, needs_dev(md) ? dev : 0.0);
    }
  }
  if (bad_final) return;   // outputs are not used (the route moved on)
  if (Rout)
    for (int c = w; c < n; c += NW)
      for (int r = lane; r < n; r += 32)   // Lout = R^T (lower)
        Rout[r + int64_t(c) * n] = (r >= c) ? S[r + c * ld] : 0.0;
  // (X_kk = L_kk^{-1} of every diagonal block was formed right after its
  // factorisation, parked in the block's upper triangle, diagonal in rdiag)
  __syncthreads();
  CHOL_PROF(3);
  // ---- X = L^{-1} in place, block columns right to left
#pragma unroll 1
  for (int k = nb - 1; k >= 0; --k) {
    const int k0 = 32 * k, kb = min(32, n - k0);
    const int r0 = k0 + kb;
    if (r0 < n) {
      // tiles of A21: rows [r0, n8) x the 32 block columns; <= 4 per warp
      const int tb = r0 / 8, nrt = nt8 - tb, ntiles = nrt * 4;
      double acc[4][2];
      // I1: A21 <- X22 A21, X22(r, t) = 0 for t > r (parked data is masked)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[q][0] = acc[q][1] = 0.0;
        const int tt = w + NW * q;
        if (tt < ntiles) {
          const int R = 8 * (tb + tt / 4), C = k0 + 8 * (tt % 4);
          const int kend = min(n8, R + 8);
          // two accumulators (k-steps alternate): half the dependent DMMA chain
          double e0 = 0.0, e1 = 0.0;
          int t0 = r0;
#pragma unroll 1
          for (; t0 + 4 < kend; t0 += 8) {
            const int tc0 = t0 + t4, tc1 = t0 + 4 + t4;
            const double a0 = (tc0 <= R + g) ? S[(R + g) + tc0 * ld] : 0.0;
            const double a1 = (tc1 <= R + g) ? S[(R + g) + tc1 * ld] : 0.0;
            dmma884(acc[q][0], acc[q][1], a0, S[tc0 + (C + g) * ld]);
            dmma884(e0, e1, a1, S[tc1 + (C + g) * ld]);
          }
          if (t0 < kend) {
            const int tc0 = t0 + t4;
            const double a0 = (tc0 <= R + g) ? S[(R + g) + tc0 * ld] : 0.0;
            dmma884(acc[q][0], acc[q][1], a0, S[tc0 + (C + g) * ld]);
          }
          acc[q][0] += e0;
          acc[q][1] += e1;
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tt = w + NW * q;
        if (tt < ntiles) {
          const int R = 8 * (tb + tt / 4), C = k0 + 8 * (tt % 4);
          const int r = R + g, cA = C + 2 * t4;
          if (r < n) {
            S[r + cA * ld] = acc[q][0];
            S[r + (cA + 1) * ld] = acc[q][1];
          }
        }
      }
      __syncthreads();
      // I2: A21 <- -A21 X11, X11(t, c) = 0 for t < c, rdiag on the diagonal,
      // parked at (c, t) below it
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[q][0] = acc[q][1] = 0.0;
        const int tt = w + NW * q;
        if (tt < ntiles) {
          const int R = 8 * (tb + tt / 4), cb = 8 * (tt % 4);   // block-local columns
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int tl = 4 * kk + t4;   // A fragment column (block-local t)
            const double av = S[(R + g) + (k0 + tl) * ld];
            const int cl = cb + g;   // B fragment: X11(tl, cl)
            const double bv = (tl < cl) ? 0.0
                              : (tl == cl ? rdiag[k0 + cl] : S[(k0 + cl) + (k0 + tl) * ld]);
            dmma884(acc[q][0], acc[q][1], av, bv);
          }
        }
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tt = w + NW * q;
        if (tt < ntiles) {
          const int R = 8 * (tb + tt / 4), C = k0 + 8 * (tt % 4);
          const int r = R + g, cA = C + 2 * t4;
          if (r < n) {
            S[r + cA * ld] = -acc[q][0];
            S[r + (cA + 1) * ld] = -acc[q][1];
          }
        }
      }
      __syncthreads();
    }
    // I3: X11 into the lower triangle of the diagonal block
    double v[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = tid + kBlkThreads * q;   // 1024 = 32 x 32 slots
      const int a = e % 32, b = e / 32;      // X(a, b), a >= b
      v[q] = 0.0;
      if (a < kb && b < kb && a >= b)
        v[q] = (a == b) ? rdiag[k0 + a] : S[(k0 + b) + (k0 + a) * ld];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int e = tid + kBlkThreads * q;
      const int a = e % 32, b = e / 32;
      if (a < kb && b < kb && a >= b) S[(k0 + a) + (k0 + b) * ld] = v[q];
    }
    __syncthreads();
  }
  for (int c = w; c < n; c += NW)
    for (int r = lane; r < n; r += 32)   // Rinv(r, c) = X(c, r), c >= r
      Rinv[r + int64_t(c) * n] = (c >= r) ? S[c + r * ld] : 0.0;
  CHOL_PROF(4);
}

// ------------------------------------------------------------------------
// Look-ahead blocked Cholesky + inverse (n <= 32*NB; one CTA of 16 warps).  Same
// contract, modes and status words as chol_blk_kernel.  X = L^{-1} lives in the
// upper triangle (X(r, c), r > c, at (c, r); diagonal in rdiag), so L stays in
// the lower triangle and both can be built concurrently.  Per 32-column block k:
//  F(k)  warp 0 factors the diagonal block in registers (lane = row) and streams
//        every group of 4 factored columns (+ 1/L_jj) through a 2-slot shared ring
//        (named barriers FULL / EMPTY) to P <= 4 panel warps, which run the same
//        eliminations on the rows below the block, so the panel L_ik is finished
//        with the diagonal block (no panel product, no X_kk on the critical path).
//        At the same time the other warps finish the trailing update of block
//        column k-1 beyond block column k, form X_{k-1,k-1} and the inverse's
//        block row X_{k-1,<k-1} = -X_{k-1,k-1} (L_{k-1,<k-1} X_{<k-1,<k-1}).
//  T(k)  all warps: trailing update of block column k+1 only (look-ahead).
// The pivot chain of F is the critical path; everything else hides behind it.
constexpr int kLaBarFull = 1, kLaBarEmpty = 3, kLaBarRest = 5;
// panel warps 1, 2, 3, 5: off SM sub-partition 0 (warp 0's)
__device__ __forceinline__ int la_panel_warp(int p) { return p < 3 ? p + 1 : 5; }

__device__ __forceinline__ void nbar_sync(int id, int cnt) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}
__device__ __forceinline__ void nbar_arrive(int id, int cnt) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(cnt) : "memory");
}

// role of warp w in F(k) with P panel warps: 0 diagonal, 1 panel (idx), 2 rest
// (idx), 3 idle (the other warps of sub-partition 0)
__device__ __forceinline__ int la_role(int w, int P, int& idx) {
  idx = 0;
  if (w == 0) return 0;
#pragma unroll
  for (int p = 0; p < 4; ++p)
    if (p < P && w == la_panel_warp(p)) {
      idx = p;
      return 1;
    }
  if ((w & 3) == 0) return 3;
  int r = 0;
  for (int v = 1; v < w; ++v) {
    bool pan = false;
#pragma unroll
    for (int p = 0; p < 4; ++p) pan |= (p < P && v == la_panel_warp(p));
    r += (!pan && (v & 3) != 0);
  }
  idx = r;
  return 2;
}
__device__ __forceinline__ int la_rest_count(int P) { return 12 - P; }

// A(r, c) -= sum_{t in [t0, t0+32)} L(r, t) L(c, t) on the 8x8 tiles (rt, ct),
// ct in [ct_lo, ct_hi), rt in [ct, nt8): tiles widx, widx + nw, ...
__device__ __noinline__ void la_trail(double* S, int ld, int n, int t0, int ct_lo, int ct_hi,
                                         int nt8, int widx, int nw, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  int tot = 0;
  for (int ct = ct_lo; ct < ct_hi; ++ct) tot += nt8 - ct;
#pragma unroll 1
  for (int tt = widx; tt < tot; tt += nw) {
    int ct = ct_lo, rem = tt;
    while (rem >= nt8 - ct) { rem -= nt8 - ct; ++ct; }
    const int rt = ct + rem;
    const int R = 8 * rt, C = 8 * ct;
    double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
    for (int kk = 0; kk < 8; kk += 2) {
      const int ta = t0 + 4 * kk + t4, tb = ta + 4;
      dmma884(c0, c1, S[(R + g) + ta * ld], S[(C + g) + ta * ld]);
      dmma884(e0, e1, S[(R + g) + tb * ld], S[(C + g) + tb * ld]);
    }
    const int r = R + g, cA = C + 2 * t4;
    if (r < n) {
      if (cA < n) S[r + cA * ld] -= c0 + e0;
      if (cA + 1 < n) S[r + (cA + 1) * ld] -= c1 + e1;
    }
  }
}

// X_kk = L_kk^{-1} of the diagonal block at k0 (kb <= 32 columns) by one warp:
// lanes 0-15 / 16-31 invert the 16 x 16 halves by register-resident forward
// substitution, then X21 = -X22 (L21 X11) on DMMA tiles.  X(r, c), r > c, parked
// at (c, r); the diagonal is rdiag.  tmp: 256 doubles of shared scratch.
__device__ __noinline__ void la_form_xkk(double* S, int ld, const double* rdiag, int k0,
                                            int kb, int lane, double* tmp) {
  const int g = lane >> 2, t4 = lane & 3;
  {
    const int h = lane >> 4, c = lane & 15, o = 16 * h;
    double x[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int t = 0; t < r; ++t) {
        const double l = (o + r < kb) ? S[(k0 + o + r) + (k0 + o + t) * ld] : 0.0;
        if (t & 1) s1 = fma(l, x[t], s1);
        else s0 = fma(l, x[t], s0);
      }
      const double rdr = (o + r < kb) ? rdiag[k0 + o + r] : 0.0;
      x[r] = (r < c || o + r >= kb) ? 0.0 : (r == c ? rdr : -rdr * (s0 + s1));
    }
#pragma unroll
    for (int r = 1; r < 16; ++r)
      if (r > c && o + r < kb) S[(k0 + o + c) + (k0 + o + r) * ld] = x[r];
  }
  __syncwarp();
  if (kb <= 16) return;
  auto x11 = [&](int row, int col) -> double {
    return row < col ? 0.0 : (row == col ? rdiag[k0 + row] : S[(k0 + col) + (k0 + row) * ld]);
  };
  auto x22 = [&](int row, int col) -> double {
    if (row < col || 16 + row >= kb) return 0.0;
    return row == col ? rdiag[k0 + 16 + row] : S[(k0 + 16 + col) + (k0 + 16 + row) * ld];
  };
  double tacc[4][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) {   // T = L21 X11
    const int R = 8 * (q >> 1), C = 8 * (q & 1);
    tacc[q][0] = tacc[q][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int kc = 4 * kk + t4;
      const double av = (16 + R + g < kb) ? S[(k0 + 16 + R + g) + (k0 + kc) * ld] : 0.0;
      dmma884(tacc[q][0], tacc[q][1], av, x11(kc, C + g));
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int R = 8 * (q >> 1), C = 8 * (q & 1);
    tmp[(R + g) + 16 * (C + 2 * t4)] = tacc[q][0];
    tmp[(R + g) + 16 * (C + 2 * t4 + 1)] = tacc[q][1];
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < 4; ++q) {   // X21 = -X22 T
    const int R = 8 * (q >> 1), C = 8 * (q & 1);
    double c0 = 0.0, c1 = 0.0;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int kc = 4 * kk + t4;
      dmma884(c0, c1, x22(R + g, kc), tmp[kc + 16 * (C + g)]);
    }
    const int r = R + g, cA = C + 2 * t4;
    if (16 + r < kb) {
      S[(k0 + cA) + (k0 + 16 + r) * ld] = -c0;
      S[(k0 + cA + 1) + (k0 + 16 + r) * ld] = -c1;
    }
  }
  __syncwarp();
}

// Block row kr of X (rows [kr0, kr0 + kbr), columns [0, kr0)), X_kk already formed:
//   T = L_{kr,<kr} X_{<kr,<kr}, then X_{kr,<kr} = -X_kk T, T staged in the
// destination (upper triangle).  One warp owns a whole 8-column tile column C
// (warps widx of nw take C = 8 widx, 8 (widx + nw), ...): T needs nothing the
// other warps write, and the -X_kk T pass runs over the row tiles bottom-up
// (tile R reads T rows <= R + 7 only), so it runs in place with no barrier.
// Rolled loops: the kernel's code stays small (it runs cold after the GEMMs).
__device__ __noinline__ void la_inverse_row(double* S, int ld, const double* rdiag, int kr0,
                                               int kbr, int widx, int nw, int lane) {
  const int g = lane >> 2, t4 = lane & 3;
  const int nrt = (kbr + 7) / 8, nct = kr0 / 8;
  const int rend = kr0 + kbr;
#pragma unroll 1
  for (int ct = widx; ct < nct; ct += nw) {
    const int C = 8 * ct, j = C + g;
    // stage 1: T(R.., C..) for every row tile; X(t, j) = 0 for t < j, so the k
    // range starts at C and only its first 8 steps (X's diagonal tile) need selects
#pragma unroll 1
    for (int rt = 0; rt < nrt; ++rt) {
      const int R = kr0 + 8 * rt;
      const double* arow = S + (R + g);
      double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
      {
        const int ta = C + t4, tb = C + 4 + t4;
        const double ba = ta > j ? S[j + ta * ld] : (ta == j ? rdiag[j] : 0.0);
        const double bb = tb > j ? S[j + tb * ld] : (tb == j ? rdiag[j] : 0.0);
        dmma884(c0, c1, arow[ta * ld], ba);
        dmma884(e0, e1, arow[tb * ld], bb);
      }
#pragma unroll 1
      for (int t = C + 8; t < kr0; t += 8) {
        const int t0 = t + t4;
        dmma884(c0, c1, arow[t0 * ld], S[j + t0 * ld]);
        dmma884(e0, e1, arow[(t0 + 4) * ld], S[j + (t0 + 4) * ld]);
      }
      const int r = R + g, cA = C + 2 * t4;
      if (r < rend) {
        S[cA + r * ld] = c0 + e0;
        S[(cA + 1) + r * ld] = c1 + e1;
      }
    }
    __syncwarp();
    // stage 2: X_{kr,<kr} = -X_kk T, bottom-up; X_kk(i, t) = 0 for t > i, parked
    // at (t, i) below its diagonal tile (selects only there)
#pragma unroll 1
    for (int rt = nrt - 1; rt >= 0; --rt) {
      const int R = kr0 + 8 * rt, i = R + g;
      const bool iv = i < rend;
      double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll 1
      for (int t = kr0; t < R; t += 8) {
        const int t0 = t + t4;
        dmma884(c0, c1, iv ? S[t0 + i * ld] : 0.0, S[j + t0 * ld]);
        dmma884(e0, e1, iv ? S[(t0 + 4) + i * ld] : 0.0, S[j + (t0 + 4) * ld]);
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int tc = R + 4 * kk + t4;
        const double av = (iv && tc <= i) ? (tc == i ? rdiag[i] : S[tc + i * ld]) : 0.0;
        const double bv = tc < rend ? S[j + tc * ld] : 0.0;
        dmma884(c0, c1, av, bv);
      }
      __syncwarp();   // every lane has read rows R.. of T before they are overwritten
      const int cA = C + 2 * t4;
      if (iv) {
        S[cA + i * ld] = -(c0 + e0);
        S[(cA + 1) + i * ld] = -(c1 + e1);
      }
      __syncwarp();
    }
  }
}

template <int NB>
__global__ void __launch_bounds__(kBlkThreads, 1)
    chol_la_kernel(const double* __restrict__ G, int n, int64_t m, int mode,
                   double* __restrict__ Rinv, double* __restrict__ Rout,
                   int* __restrict__ flags, const int* gate, int gate_val) {
  if (gate && *gate != gate_val) return;
  extern __shared__ double S[];
  __shared__ double rdiag[32 * NB];
  __shared__ __align__(16) double ring[2][4][64];   // factored columns, doubled (see F)
  __shared__ double ring_rd[2][4];
  __shared__ double ttmp[256];
  __shared__ double s_tr, s_dmax;
  __shared__ int s_bad, s_zero, s_clamped;
  const int ld = chol_ld(n);
  const int n8 = (n + 7) & ~7, nt8 = n8 / 8;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nb = (n + 31) / 32;
  const int md = mode & 0xff;
  if (tid == 0) { s_bad = 0; s_zero = 0; s_clamped = 0; }
  if (tid < 32) {
    double tr = 0.0, dmax = 0.0;
    for (int i = tid; i < n; i += 32) {
      const double gi = G[i + int64_t(i) * n];
      tr += gi;
      dmax = fmax(dmax, gi);
    }
    for (int o = 16; o; o >>= 1) {
      tr += __shfl_xor_sync(0xffffffffu, tr, o);
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    if (tid == 0) {
      if (!isfinite(tr)) atomicOr(&flags[3], 4);   // NaN/Inf in the input (TT_ERR_NONFINITE)
      if (!(tr > 0.0)) {
        if (tr == 0.0) { atomicOr(&flags[2], 1); s_zero = 1; }   // Y_n == 0: zero sum (R16)
        s_bad = 1;
      }
      s_tr = tr;
      s_dmax = dmax;
    }
  }
  __syncthreads();
  const bool shifted = md == CH_SHIFT || md == CH_SHIFT2 || md == CH_SHIFT1B || md == CH_RSHIFT;
  const double shift = shifted ? 11.0 * (double(m) * n + double(n) * (n + 1)) * 0x1p-53 * s_tr : 0.0;
  const bool clamp = md == CH_RCLAMP;
  const double tau = 64.0 * n * 0x1p-53 * s_dmax;
#ifdef TTR_CHOL_PROF
  long long prof_t = clock64();
#endif
  for (int j = w; j < n8; j += 16) {
#pragma unroll 4
    for (int i = lane; i < ld; i += 32)
      S[i + j * ld] = (i < n && j < n && i >= j) ? G[i + int64_t(j) * n] + ((i == j) ? shift : 0.0)
                                                 : 0.0;
  }
  __syncthreads();
  CHOL_PROF(5);
#pragma unroll 1
  for (int k = 0; k < nb; ++k) {
    const int k0 = 32 * k, kb = min(32, n - k0);
    const int r0 = k0 + kb;                         // first row below the block
    const int P = r0 < n ? (n - r0 + 31) / 32 : 0;  // panel warps
    const int cnt = 32 * (1 + P);
    const int ng = (kb + 3) >> 2;
    int idx;
    const int role = la_role(w, P, idx);
    if (role <= 1) {
      // ---- F(k).  Diagonal warp (role 0): lane i keeps the not yet eliminated
      // part of row k0 + i in registers (a[q] = A(i, j0 + q)), pivots in groups
      // of 4 with static register offsets, then a shift by 4.  The pivot step
      // is branch-free (clamping and the finiteness test are selects; 1/L_jj =
      // MUFU rsqrt + two Newton steps).  Factored column j goes to the ring slot
      // of its group, doubled (colb[i] = colb[i + 32] = L_ij) so that every load
      // of the update is [base + constant]; updates of the upper slots are
      // harmless.  Panel warps (role 1): the same eliminations on rows
      // r0 + 32 idx + lane with the ring's columns and 1/L_jj -- one shared
      // code path for the update, so the kernel's code stays small.
      const bool diag = role == 0;
      const int i = lane;
      const int ip = diag ? k0 + lane : r0 + 32 * idx + lane;   // absolute row
      const bool live = diag ? lane < kb : ip < n;
      double a[32];
#pragma unroll
      for (int q = 0; q < 32; ++q)
        a[q] = (live && q < kb && (!diag || q <= i)) ? S[ip + (k0 + q) * ld] : 0.0;
      int bad = 0, nclamp = 0;
#pragma unroll 1
      for (int grp = 0; grp < ng; ++grp) {
        const int sl = grp & 1;
        if (!diag) nbar_sync(kLaBarFull + sl, cnt);
        if (diag && P > 0 && grp >= 2) {   // panel done with grp - 2
#ifdef TTR_CHOL_PROF
          const long long tw0 = clock64();
#endif
          nbar_sync(kLaBarEmpty + sl, cnt);
#ifdef TTR_CHOL_PROF
          if (threadIdx.x == 0) atomicAdd(&flags[33], int((clock64() - tw0) >> 6));
#endif
        }
#pragma unroll
        for (int sft = 0; sft < 4; ++sft) {
          const int j = 4 * grp + sft;
          double* cb0 = ring[sl][sft];
          double l;
          if (diag) {
            double piv = __shfl_sync(0xffffffffu, a[sft], j);
            piv = (j < kb) ? piv : 1.0;                       // padding pivot
            const bool fin = fabs(piv) <= 1.79e308;           // false for inf / nan
            const bool cl = clamp && fin && !(piv > tau);     // numerically null direction
            piv = cl ? tau : piv;
            nclamp += cl;
            const bool ok = fin && piv > 0.0;
            bad |= !ok;
            const double pv = ok ? piv : 1.0;
            double rd;
            asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(rd) : "d"(pv));
            rd = rd * fma(-0.5 * pv * rd, rd, 1.5);           // Newton steps for 1/sqrt
            rd = rd * fma(-0.5 * pv * rd, rd, 1.5);
            l = (i > j) ? a[sft] * rd : (i == j ? pv * rd : 0.0);
            if (j < kb && i >= j && i < kb) S[(k0 + i) + (k0 + j) * ld] = l;
            if (i == j && j < kb) rdiag[k0 + j] = rd;
            cb0[i] = l;
            cb0[i + 32] = l;
            if (i == 0) ring_rd[sl][sft] = rd;
            __syncwarp();
          } else {
            l = a[sft] * ring_rd[sl][sft];
            if (live && j < kb) S[ip + (k0 + j) * ld] = l;
          }
          const double* cb = cb0 + j;
#pragma unroll
          for (int qq = 1; qq < 32 - sft; ++qq) a[sft + qq] = fma(-l, cb[qq], a[sft + qq]);
        }
#pragma unroll
        for (int q = 0; q < 28; ++q) a[q] = a[q + 4];
        a[28] = a[29] = a[30] = a[31] = 0.0;
        if (diag) {
          if (P > 0) nbar_arrive(kLaBarFull + sl, cnt);
        } else if (grp + 2 < ng) {
          nbar_arrive(kLaBarEmpty + sl, cnt);   // warp 0 reuses the slot
        }
      }
      if (diag) {
        if (lane == 0) {
          if (bad) s_bad = 1;
          if (nclamp) s_clamped += nclamp;
        }
        CHOL_PROF(6);
      }
    } else if (role == 2 && k > 0) {
      // ---- behind F(k): finish block column k-1 (its trailing update beyond
      // block column k, X_{k-1,k-1}, the inverse's block row k-1)
      const int R = la_rest_count(P), rc = 32 * R;
      const int kp0 = k0 - 32;
      // (columns from k0 + 32 on: block column k itself was updated by T(k-1))
      if (idx == 0) la_form_xkk(S, ld, rdiag, kp0, 32, lane, ttmp);
      else if (k0 + 32 < n)
        la_trail(S, ld, n, kp0, (k0 + 32) / 8, nt8, nt8, idx - 1, R - 1, lane);
      nbar_sync(kLaBarRest, rc);
      if (kp0 > 0) la_inverse_row(S, ld, rdiag, kp0, 32, idx, R, lane);
    }
    __syncthreads();
    CHOL_PROF(0);
    if (s_bad) break;
    // ---- T(k): trailing update of block column k+1 (look-ahead)
    if (r0 < n) {
      la_trail(S, ld, n, k0, r0 / 8, min(r0 / 8 + 4, nt8), nt8, w, 16, lane);
      __syncthreads();
    }
    CHOL_PROF(2);
  }
  __syncthreads();
  const bool bad_final = s_bad;
  if (!bad_final) {
    // the last block: X_kk, then its block row of X (whole CTA)
    const int kl0 = 32 * (nb - 1), kbl = n - kl0;
    if (w == 0) la_form_xkk(S, ld, rdiag, kl0, kbl, lane, ttmp);
    __syncthreads();
    if (kl0 > 0) la_inverse_row(S, ld, rdiag, kl0, kbl, w, 16, lane);
  }
  CHOL_PROF(3);
  if (w == 0 && !s_zero) {   // route checks on diag(L), warp-parallel
    double dev = 0.0, dmin = INFINITY, dmax = 0.0;
    for (int i = lane; i < n; i += 32) {
      const double d = fabs(S[i + i * ld]);
      dmin = fmin(dmin, d);
      dmax = fmax(dmax, d);
      dev = fmax(dev, fabs(S[i + i * ld] - 1.0));
    }
    for (int o = 16; o; o >>= 1) {
      dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
      dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
      dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, o));
    }
    if (lane == 0 && !(flags[2] & 1)) {
      int bad2 = bad_final;
      if ((mode & kStrict) && !(dmin >= dmax * kStrictRatio)) bad2 = 1;
      if (s_clamped) flags[16] += 1;   // counter: clamped (rank-deficient) passes
      route_update(flags, md, bad2, needs_dev(md) ? dev : 0.0);
    }
  }
  if (bad_final) return;   // outputs are not used (the route moved on)
  __syncthreads();
  for (int c = w; c < n; c += 16)
    for (int r = lane; r < n; r += 32) {
      // Rinv(r, c) = X(c, r) (c > r: stored at (r, c)); Lout = R^T (lower)
      Rinv[r + int64_t(c) * n] = (c > r) ? S[r + c * ld] : (c == r ? rdiag[r] : 0.0);
      if (Rout) Rout[r + int64_t(c) * n] = (r >= c) ? S[r + c * ld] : 0.0;
    }
  CHOL_PROF(4);
}

__global__ void route_start_kernel(int* flags) { flags[0] = flags[0] >= 1 ? 1 : 0; }

// Cholesky factor of a Gram G = I + E that is the identity to working accuracy
// (the truncation's last CholeskyQR pass: its input is already orthonormal to
// O(u)): R = I + U with U = triu(E) and U_ii = E_ii / 2, so that
// R^T R = G + U^T U = G + O(||E||^2).  flags[slot] = 1 (-> the full Cholesky runs,
// gated) when max |E| > thr, where the first-order factor is not exact enough.
__global__ void __launch_bounds__(1024)
    near_identity_chol_kernel(const double* __restrict__ G, int n, double* __restrict__ R,
                              int* __restrict__ flags, int slot, double thr) {
  __shared__ double red[32];
  double mx = 0.0;
  // 2-D loop (no division per element), loads batched 4 deep: the Gram sits in
  // L2 and the kernel is bound by load latency
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = w; j < n; j += nw) {
#pragma unroll 4
    for (int i = lane; i < n; i += 32) {
      const double g = G[(i >= j) ? i + int64_t(j) * n : j + int64_t(i) * n];   // lower triangle holds G
      const double x = g - (i == j ? 1.0 : 0.0);
      mx = fmax(mx, fabs(x));
      R[i + int64_t(j) * n] = (i > j) ? x : (i == j ? 1.0 + 0.5 * x : 0.0);   // L = R^T
    }
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[w] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int q = 0; q < nw; ++q) m = fmax(m, red[q]);
    flags[slot] = (m > thr || !(m == m)) ? 1 : 0;
  }
}

__global__ void route_fail_kernel(int* flags) {
  if (flags[0] == 3) atomicOr(&flags[3], 1);
}

__global__ void gated_set_kernel(int* flag, int from, int to) {
  if (*flag == from) *flag = to;
}

// dst = src^T (n x n), iff *gate == gate_val
__global__ void gated_transpose_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                       int n, const int* gate, int gate_val) {
  if (gate && *gate != gate_val) return;
  const int64_t nn = int64_t(n) * n;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nn;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = e % n, j = e / n;
    dst[e] = src[j + i * n];
  }
}

__global__ void gated_copy_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                  int64_t n, const int* gate, int gate_val) {
  if (gate && *gate != gate_val) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    dst[i] = src[i];
}

// ---------------------------------------------------------- Householder fallback
// Single CTA; runs only if every CholeskyQR route broke down (route state 3).  A (m x n) is copied to
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
  if (flags[0] != 3) return;
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
    flags[11] += 1;            // route counter: Householder
  }
}

}  // namespace

// ---------------------------------------------------------- TSQR (R only)
// Rank-deficiency-proof R factor of a tall m x n (n <= 160) matrix op(A): the
// fallback of the R-only QR when both CholeskyQR routes fail (numerically rank-
// deficient bond matrices of the truncation).  Householder on
// row blocks (one CTA per block, block in shared memory), then a binary tree of
// merges of two upper triangles [R1; R2] (packed, both in shared memory).
// Packed upper triangle: element (r, c), r <= c, at c(c+1)/2 + r.
__device__ __forceinline__ int pk(int r, int c) { return c * (c + 1) / 2 + r; }

__global__ void __launch_bounds__(1024, 1)
    tsqr_leaf_kernel(const double* __restrict__ A, int64_t lda, bool trans, int64_t m, int n,
                     int br, double* __restrict__ Rp, const int* gate, int gate_val) {
  if (gate && *gate != gate_val) return;
  extern __shared__ double B[];        // rows x n, ld br
  __shared__ double red[32];
  __shared__ double s_tau;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t r0 = int64_t(blockIdx.x) * br;
  const int rows = int((m - r0) < br ? (m - r0) : int64_t(br));
  for (int e = tid; e < rows * n; e += 1024) {
    int i, j;
    if (trans) { j = e % n; i = e / n; } else { i = e % rows; j = e / rows; }
    const int64_t gi = r0 + i;
    B[i + j * br] = trans ? A[j + gi * lda] : A[gi + int64_t(j) * lda];
  }
  __syncthreads();
  const int steps = min(rows, n);
  for (int j = 0; j < steps; ++j) {
    if (warp == 0) {
      double ss = 0.0;
      for (int i = j + 1 + lane; i < rows; i += 32) ss += B[i + j * br] * B[i + j * br];
      for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      const double alpha = B[j + j * br];
      double tau = 0.0, beta = alpha, scal = 0.0;
      if (ss > 0.0) {
        const double nrm = sqrt(alpha * alpha + ss);
        beta = (alpha >= 0.0) ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      __syncwarp();
      if (ss > 0.0)
        for (int i = j + 1 + lane; i < rows; i += 32) B[i + j * br] *= scal;
      if (lane == 0) {
        s_tau = tau;
        red[0] = beta;
      }
    }
    __syncthreads();
    const double tau = s_tau;
    if (tau != 0.0) {
      for (int k = j + 1 + warp; k < n; k += 32) {
        double wsum = (lane == 0) ? B[j + k * br] : 0.0;
        for (int i = j + 1 + lane; i < rows; i += 32) wsum += B[i + j * br] * B[i + k * br];
        for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
        wsum *= tau;
        if (lane == 0) B[j + k * br] -= wsum;
        for (int i = j + 1 + lane; i < rows; i += 32) B[i + k * br] -= wsum * B[i + j * br];
      }
    }
    if (tid == 0) B[j + j * br] = red[0];
    __syncthreads();
  }
  double* out = Rp + int64_t(blockIdx.x) * (int64_t(n) * (n + 1) / 2);
  for (int c = warp; c < n; c += 32)
    for (int r = lane; r <= c; r += 32) out[pk(r, c)] = (r < rows) ? B[r + c * br] : 0.0;
}

// out[q] = R of [in[2q]; in[2q+1]] (both n x n upper triangles, packed)
__global__ void __launch_bounds__(1024, 1)
    tsqr_merge_kernel(const double* __restrict__ in, int count, int n, double* __restrict__ out,
                      const int* gate, int gate_val) {
  if (gate && *gate != gate_val) return;
  extern __shared__ double T[];        // two packed triangles
  __shared__ double s_tau, s_beta;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t tri = int64_t(n) * (n + 1) / 2;
  const int q = blockIdx.x;
  double* T1 = T;
  double* T2 = T + tri;
  double* o = out + q * tri;
  if (2 * q + 1 >= count) {              // odd one out: copy through
    for (int64_t e = tid; e < tri; e += 1024) o[e] = in[(2 * q) * tri + e];
    return;
  }
  for (int64_t e = tid; e < 2 * tri; e += 1024) T[e] = in[(2 * q) * tri + e];
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    // reflector on x = (T1(j,j), T2(0..j, j))
    if (warp == 0) {
      double ss = 0.0;
      for (int r = lane; r <= j; r += 32) ss += T2[pk(r, j)] * T2[pk(r, j)];
      for (int o2 = 16; o2; o2 >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o2);
      const double alpha = T1[pk(j, j)];
      double tau = 0.0, beta = alpha, scal = 0.0;
      if (ss > 0.0) {
        const double nrm = sqrt(alpha * alpha + ss);
        beta = (alpha >= 0.0) ? -nrm : nrm;
        tau = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      __syncwarp();
      if (ss > 0.0)
        for (int r = lane; r <= j; r += 32) T2[pk(r, j)] *= scal;   // v (below the unit head)
      if (lane == 0) { s_tau = tau; s_beta = beta; }
    }
    __syncthreads();
    const double tau = s_tau;
    if (tau != 0.0) {
      for (int k = j + 1 + warp; k < n; k += 32) {
        double wsum = (lane == 0) ? T1[pk(j, k)] : 0.0;
        for (int r = lane; r <= j; r += 32) wsum += T2[pk(r, j)] * T2[pk(r, k)];
        for (int o2 = 16; o2; o2 >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o2);
        wsum *= tau;
        if (lane == 0) T1[pk(j, k)] -= wsum;
        for (int r = lane; r <= j; r += 32) T2[pk(r, k)] -= wsum * T2[pk(r, j)];
      }
    }
    __syncthreads();
    if (tid == 0) T1[pk(j, j)] = s_beta;
  }
  __syncthreads();
  for (int64_t e = tid; e < tri; e += 1024) o[e] = T1[e];
}

__global__ void unpack_upper_kernel(const double* __restrict__ P, int n, double* __restrict__ R,
                                    const int* gate, int gate_val, int* flags) {
  if (gate && *gate != gate_val) return;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int r = e % n, c = e / n;
    R[e] = (r <= c) ? P[pk(r, c)] : 0.0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) flags[14] += 1;   // route counter: TSQR
}

// R (n x n, ld n) of op(A) by TSQR; gated like the other QR launches.
static int tsqr_r(Ctx& c, int64_t m, int n, const double* A, int64_t lda, bool trans,
                  double* R, const int* gate, int gv, cudaStream_t s) {
  const int br = std::max(n, std::min<int>(int(m), kSmemLimitDoubles / n));
  const int64_t P = (m + br - 1) / br;
  const int64_t tri = int64_t(n) * (n + 1) / 2;
  DBuf W0, W1;
  TTR_TRY(dalloc(W0, size_t(P * tri), s));
  TTR_TRY(dalloc(W1, size_t((P + 1) / 2 * tri), s));
  static std::atomic<bool> attr{false};
  std::unique_lock<std::mutex> init_lock(init_mutex(), std::defer_lock);
  if (!attr) init_lock.lock();
  if (!attr) {
    TTR_CUDA(cudaFuncSetAttribute(tsqr_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimitDoubles * 8));
    TTR_CUDA(cudaFuncSetAttribute(tsqr_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kSmemLimitDoubles * 8));
    attr = true;
  }
  tsqr_leaf_kernel<<<unsigned(P), 1024, size_t(br) * n * 8, s>>>(A, lda, trans, m, n, br, W0.p,
                                                                  gate, gv);
  TTR_TRY(launched());
  double* cur = W0.p;
  double* nxt = W1.p;
  int64_t cnt = P;
  while (cnt > 1) {
    const int64_t half = (cnt + 1) / 2;
    tsqr_merge_kernel<<<unsigned(half), 1024, size_t(2 * tri) * 8, s>>>(cur, int(cnt), n, nxt,
                                                                         gate, gv);
    TTR_TRY(launched());
    std::swap(cur, nxt);
    cnt = half;
  }
  unpack_upper_kernel<<<std::max(1, (n * n + 255) / 256), 256, 0, s>>>(cur, n, R, gate, gv,
                                                                      c.flags.p);
  return launched();
}

bool tsqr_fits(int n) { return n >= 1 && 2 * (int64_t(n) * (n + 1) / 2) <= kSmemLimitDoubles; }

// Launch one Cholesky(+inverse) of the n x n Gram Gm (see chol_blk_kernel).
static int launch_chol(Ctx& c, const double* Gm, int n, int64_t m, int mode, double* Rinv,
                       double* Rk, double* gw, const int* gate, int gv, cudaStream_t s) {
  static std::atomic<bool> attr_done{false};
  std::unique_lock<std::mutex> init_lock(init_mutex(), std::defer_lock);
  if (!attr_done) init_lock.lock();
  if (!attr_done) {
    TTR_CUDA(cudaFuncSetAttribute(chol_inv_kernel<32>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  kCholTsmDoubles * 8));
    TTR_CUDA(cudaFuncSetAttribute(chol_blk_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    TTR_CUDA(cudaFuncSetAttribute(chol_blk_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    TTR_CUDA(cudaFuncSetAttribute(chol_blk_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    TTR_CUDA(cudaFuncSetAttribute(chol_la_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    TTR_CUDA(cudaFuncSetAttribute(chol_la_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  220 * 1024));
    TTR_CUDA(cudaFuncSetAttribute(chol_la_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  210 * 1024));
    attr_done = true;
  }
  const size_t shm = size_t(chol_ld(n)) * ((n + 7) & ~7) * sizeof(double);
  // default: the look-ahead kernel; TTR_CHOL=blk selects the round-1 blocked one (A/B)
  static const bool blk = [] {
    const char* v = getenv("TTR_CHOL");
    return v && strcmp(v, "blk") == 0;
  }();
  if (n <= 32) {
    if (blk) chol_blk_kernel<1><<<1, kBlkThreads, shm, s>>>(Gm, n, m, mode, Rinv, Rk, c.flags.p, gate, gv);
    else chol_la_kernel<1><<<1, kBlkThreads, shm, s>>>(Gm, n, m, mode, Rinv, Rk, c.flags.p, gate, gv);
  } else if (n <= 64) {
    if (blk) chol_blk_kernel<2><<<1, kBlkThreads, shm, s>>>(Gm, n, m, mode, Rinv, Rk, c.flags.p, gate, gv);
    else chol_la_kernel<2><<<1, kBlkThreads, shm, s>>>(Gm, n, m, mode, Rinv, Rk, c.flags.p, gate, gv);
  } else if (n <= 160) {
    if (blk) chol_blk_kernel<5><<<1, kBlkThreads, shm, s>>>(Gm, n, m, mode, Rinv, Rk, c.flags.p, gate, gv);
    else chol_la_kernel<5><<<1, kBlkThreads, shm, s>>>(Gm, n, m, mode, Rinv, Rk, c.flags.p, gate, gv);
  } else {
    const bool big = n * n > kSmemLimitDoubles;
    const size_t tsm = (chol_tsm_doubles(n) <= kCholTsmDoubles) ? size_t(chol_tsm_doubles(n)) * 8 : 0;
    chol_inv_kernel<32><<<1, kCholThreads, big ? tsm : size_t(n) * n * 8, s>>>(
        Gm, n, m, mode, Rinv, Rk, gw, c.flags.p, gate, gv);
  }
  return launched();
}

int qr(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, bool trans, double* Q,
       double* R, cudaStream_t s, bool dist, int64_t mglob, bool robust_q) {
  if (mglob <= 0) mglob = m;
  if ((!dist && m < n) || mglob < n || n < 1 || m < 0) {
    set_error("qr: need m >= n >= 1 (m=%lld n=%lld)", (long long)mglob, (long long)n);
    return TT_ERR_ARG;
  }
  if (n > 1024) {
    set_error("qr: n = %lld > 1024 unsupported", (long long)n);
    return TT_ERR_ARG;
  }
  if (!Q && !R) {
    set_error("qr: nothing to compute");
    return TT_ERR_ARG;
  }
  const int ni = int(n), mi = int(m);
  const bool r_only = (Q == nullptr);
  DBuf T1, T2, Gm, Rinv, Rk, Racc, Rtmp, gw;
  TTR_TRY(dalloc(T1, size_t(m) * n, s));
  TTR_TRY(dalloc(T2, size_t(m) * n, s));
  TTR_TRY(dalloc(Gm, size_t(n) * n, s));
  TTR_TRY(dalloc(Rinv, size_t(n) * n, s));
  if (ni > 160 && ni * ni > kSmemLimitDoubles) TTR_TRY(dalloc(gw, size_t(n) * n, s));
  if (R) {
    TTR_TRY(dalloc(Rk, size_t(n) * n, s));
    TTR_TRY(dalloc(Racc, size_t(n) * n, s));
    TTR_TRY(dalloc(Rtmp, size_t(n) * n, s));
  }
  int* F = c.flags.p;
  // starting route: 0 (CholeskyQR2), or 1 when the previous QR of this call
  // sequence needed a shifted route -- the sweep's sketches Y_n have similar
  // conditioning from bond to bond, so a failed CholeskyQR2 attempt is not
  // repeated at every step (flags are cleared at the start of every rounding)
  route_start_kernel<<<1, 1, 0, s>>>(F);
  TTR_TRY(launched());
  const int copy_blocks = int(std::min<int64_t>((int64_t(m) * n + 255) / 256, c.sm_count * 8));
  double* Rk_p = R ? Rk.p : nullptr;

  // Gram of the input op(A) (A is m x n, or n x m when trans)
  // distributed (mode-slab sharding, NEXT-2): this rank holds m of the mglob
  // rows; every Gram is summed over the ranks (an n x n allreduce), so every rank
  // factors the same Gram and the route flags agree; Q keeps the local rows
  auto reduce_gram = [&]() -> int {
    if (!dist) return TT_OK;
    return allreduce_sum(c, Gm.p, size_t(n) * n);
  };
  auto gram_of_input = [&](const int* gate, int gv) -> int {
    if (mi == 0) {
      TTR_TRY(fill_zero(c, Gm.p, int64_t(ni) * ni, s));
    } else if (trans) {
      TTR_TRY(gemm1(c, false, true, ni, ni, mi, 1.0, A, int(lda), A, int(lda), 0.0, Gm.p, ni, s,
                    gate, gv, kGemmLower));
    } else {
      TTR_TRY(gemm1(c, true, false, ni, ni, mi, 1.0, A, int(lda), A, int(lda), 0.0, Gm.p, ni, s,
                    gate, gv, kGemmLower));
    }
    return reduce_gram();
  };
  auto input_times_rinv = [&](double* dst, const int* gate, int gv) -> int {
    if (trans)
      return gemm1(c, true, false, mi, ni, ni, 1.0, A, int(lda), Rinv.p, ni, 0.0, dst, mi, s,
                   gate, gv, kGemmTriB);
    return gemm1(c, false, false, mi, ni, ni, 1.0, A, int(lda), Rinv.p, ni, 0.0, dst, mi, s,
                 gate, gv, kGemmTriB);
  };
  auto gram = [&](const double* src, const int* gate, int gv) -> int {
    if (mi == 0) TTR_TRY(fill_zero(c, Gm.p, int64_t(ni) * ni, s));
    else TTR_TRY(gemm1(c, true, false, ni, ni, mi, 1.0, src, mi, src, mi, 0.0, Gm.p, ni, s, gate,
                       gv, kGemmLower));
    return reduce_gram();
  };
  auto times_rinv = [&](const double* src, double* dst, const int* gate, int gv) -> int {
    return gemm1(c, false, false, mi, ni, ni, 1.0, src, mi, Rinv.p, ni, 0.0, dst, mi, s, gate,
                 gv, kGemmTriB);
  };
  static const bool dbg = getenv("TTR_QR_DEBUG") != nullptr;
  auto dump = [&](const char* what, const double* p, int64_t cnt) {
    if (!dbg) return;
    cudaStreamSynchronize(s);
    std::vector<double> h(cnt);
    cudaMemcpy(h.data(), p, cnt * 8, cudaMemcpyDeviceToHost);
    int f[16];
    cudaMemcpy(f, F, sizeof f, cudaMemcpyDeviceToHost);
    double ss = 0;
    for (double v : h) ss += v * v;
    fprintf(stderr, "[qr %lldx%d] %s: norm %.6e  [0]=%.6e  route=%d\n", (long long)m, ni, what,
            sqrt(ss), h[0], f[0]);
  };
  auto chol = [&](int mode, const int* gate, int gv) -> int {
    dump("gram", Gm.p, int64_t(ni) * ni);
    int r = launch_chol(c, Gm.p, ni, mglob, mode, Rinv.p, Rk_p, gw.p, gate, gv, s);
    if (Rk_p) dump("Rk", Rk_p, int64_t(ni) * ni);
    return r;
  };
  // Racc <- Rk Racc (gated)
  auto accumulate_r = [&](const int* gate, int gv) -> int {
    if (!R) return TT_OK;
    TTR_TRY(gemm1(c, true, false, ni, ni, ni, 1.0, Rk.p, ni, Racc.p, ni, 0.0, Rtmp.p, ni, s,
                  gate, gv));   // Rk holds L_k = R_k^T
    gated_copy_kernel<<<std::max(1, (ni * ni + 255) / 256), 256, 0, s>>>(Rtmp.p, Racc.p,
                                                                       int64_t(ni) * ni, gate, gv);
    return launched();
  };
  auto copy_r_first = [&](const int* gate, int gv) -> int {
    if (!R) return TT_OK;
    gated_transpose_kernel<<<std::max(1, (ni * ni + 255) / 256), 256, 0, s>>>(Rk.p, Racc.p, ni,
                                                                            gate, gv);
    return launched();
  };
  auto gated_copy = [&](const double* src, double* dst, const int* gate, int gv) -> int {
    gated_copy_kernel<<<copy_blocks, 256, 0, s>>>(src, dst, int64_t(m) * n, gate, gv);
    return launched();
  };
  // one CholeskyQR pass as one persistent launch (cqr.cu): dst = src R^{-1} and
  // its Gram, src = op(A) (first) or a previous Q (m x n, ld m); TTR_NO_CQR=1
  // selects the two-GEMM form (A/B)
  static const bool no_cqr = getenv("TTR_NO_CQR") != nullptr;
  const bool use_cqr = !no_cqr && cqr_fits(ni);
  auto first_pass = [&](double* dst, const int* gate, int gv) -> int {   // Q1 = op(A) R^{-1}, G(Q1)
    if (!use_cqr) {
      TTR_TRY(input_times_rinv(dst, gate, gv));
      return gram(dst, gate, gv);
    }
    TTR_TRY(cqr_pass(c, m, ni, A, lda, trans, Rinv.p, dst, m, Gm.p, s, gate, gv));
    return reduce_gram();
  };
  auto next_pass = [&](const double* src, double* dst, const int* gate, int gv) -> int {
    if (!use_cqr) {
      TTR_TRY(times_rinv(src, dst, gate, gv));
      return gram(dst, gate, gv);
    }
    TTR_TRY(cqr_pass(c, m, ni, src, m, false, Rinv.p, dst, m, Gm.p, s, gate, gv));
    return reduce_gram();
  };
  auto last_q = [&](const double* src, double* dst, const int* gate, int gv) -> int {
    if (!use_cqr) return times_rinv(src, dst, gate, gv);
    return cqr_pass(c, m, ni, src, m, false, Rinv.p, dst, m, nullptr, s, gate, gv);
  };
  auto input_gram = [&](const int* gate, int gv) -> int {
    if (!use_cqr || mi == 0) return gram_of_input(gate, gv);
    TTR_TRY(cqr_pass(c, m, ni, A, lda, trans, nullptr, nullptr, 0, Gm.p, s, gate, gv));
    return reduce_gram();
  };

  // ---- R only, n <= 160 (the truncation): four CholeskyQR passes, no routes.
  // Passes 1-2 are shifted (shift 11(mn + n(n+1)) u tr G, Fukaya et al.), which
  // compresses kappa(op(A)) up to ~1/u; passes 3-4 are plain, so the final Q4
  // is orthonormal and A = Q4 R carries no shift bias; a pivot below
  // tau = 64 n u max(diag G) (a numerically null direction of a rank-deficient
  // bond matrix) is clamped to tau instead of breaking down.  R^T R = A^T A +
  // O(u ||A||^2): singular values/vectors of R are those of op(A) to O(u ||A||)
  // (DESIGN.md §QR).
  if (r_only && ni <= 160) {
    TTR_TRY(input_gram(nullptr, 0));
    TTR_TRY(chol(CH_RSHIFT, nullptr, 0));                   // R1 (shifted)
    TTR_TRY(copy_r_first(nullptr, 0));
    TTR_TRY(first_pass(T1.p, nullptr, 0));                  // Q1 = op(A) R1^{-1}, G(Q1)
    TTR_TRY(chol(CH_RSHIFT, nullptr, 0));                   // R2 (shifted)
    TTR_TRY(accumulate_r(nullptr, 0));
    TTR_TRY(next_pass(T1.p, T2.p, nullptr, 0));             // Q2 = Q1 R2^{-1}, G(Q2)
    TTR_TRY(chol(CH_RCLAMP, nullptr, 0));                   // R3 (plain, clamped)
    TTR_TRY(accumulate_r(nullptr, 0));
    TTR_TRY(next_pass(T2.p, T1.p, nullptr, 0));             // Q3 = Q2 R3^{-1}, G(Q3)
    // R4: Q3 is orthonormal to O(u), so its Gram is I + E with ||E|| = O(u) and
    // the first-order factor I + triu(E) (half diagonal) is exact to O(u^2); the
    // full Cholesky runs only when max |E| > 1e-8 (gated on the device)
    near_identity_chol_kernel<<<1, 1024, 0, s>>>(Gm.p, ni, Rk.p, F, kNearIdFlag, 1e-8);
    TTR_TRY(launched());
    TTR_TRY(chol(CH_RCLAMP, F + kNearIdFlag, 1));           // R4 (plain, clamped), if needed
    TTR_TRY(accumulate_r(nullptr, 0));
    TTR_CUDA(cudaMemcpyAsync(R, Racc.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
    return TT_OK;
  }
  // ---- robust Q (deterministic baseline, see common.cuh): the passes of the
  // R-only path with the full clamped Cholesky for pass 4 and Q = Q3 R4^{-1}
  if (robust_q && !r_only && !dist) {
    if (!R) {
      set_error("qr: robust_q needs R");
      return TT_ERR_ARG;
    }
    TTR_TRY(input_gram(nullptr, 0));
    TTR_TRY(chol(CH_RSHIFT, nullptr, 0));
    TTR_TRY(copy_r_first(nullptr, 0));
    TTR_TRY(first_pass(T1.p, nullptr, 0));
    TTR_TRY(chol(CH_RSHIFT, nullptr, 0));
    TTR_TRY(accumulate_r(nullptr, 0));
    TTR_TRY(next_pass(T1.p, T2.p, nullptr, 0));
    TTR_TRY(chol(CH_RCLAMP, nullptr, 0));
    TTR_TRY(accumulate_r(nullptr, 0));
    TTR_TRY(next_pass(T2.p, T1.p, nullptr, 0));
    TTR_TRY(chol(CH_RCLAMP, nullptr, 0));
    TTR_TRY(accumulate_r(nullptr, 0));
    TTR_TRY(last_q(T1.p, Q, nullptr, 0));
    TTR_CUDA(cudaMemcpyAsync(R, Racc.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
    return TT_OK;
  }
  // ---- route 0: CholeskyQR2, accepted when pass 2 finds Q1 close to
  // orthonormal (|diag R2 - 1| <= kDevTol).  The route state F[0] lives on the
  // device; every launch of an inactive route is a no-op.
  TTR_TRY(input_gram(F, 0));                                // pass 1 on the input
  TTR_TRY(chol(CH_FIRST, F, 0));
  TTR_TRY(copy_r_first(F, 0));
  TTR_TRY(first_pass(T1.p, F, 0));                          // Q1 -> T1, pass 2 Gram
  TTR_TRY(chol(CH_SECOND, F, 0));
  TTR_TRY(accumulate_r(F, 0));
  if (!r_only) TTR_TRY(last_q(T1.p, Q, F, 0));              // Q = Q1 R2^{-1}
  // ---- route 1: shifted CholeskyQR3 (kappa up to ~1e10)
  TTR_TRY(input_gram(F, 1));
  TTR_TRY(chol(CH_SHIFT, F, 1));
  TTR_TRY(copy_r_first(F, 1));
  TTR_TRY(first_pass(T1.p, F, 1));                          // Q1 (shifted) -> T1
  TTR_TRY(chol(CH_SPLAIN | (r_only ? kStrict : 0), F, 1));  // -> route 2 if Q1 is still too ill-conditioned
  TTR_TRY(accumulate_r(F, 1));
  TTR_TRY(next_pass(T1.p, T2.p, F, 1));
  TTR_TRY(chol(CH_SLAST, F, 1));
  TTR_TRY(accumulate_r(F, 1));
  if (!r_only) TTR_TRY(last_q(T2.p, Q, F, 1));
  // ---- route 2: shifted pass on the input, a second shifted pass on its Q1
  // (kappa up to ~1/u), then CholeskyQR2.  Skipped for R-only QRs, whose hard
  // cases are exactly rank-deficient (TSQR).
  if (!r_only) {
    TTR_TRY(input_gram(F, 2));
    TTR_TRY(chol(CH_SHIFT1B, F, 2));
    TTR_TRY(copy_r_first(F, 2));
    TTR_TRY(first_pass(T1.p, F, 2));
    TTR_TRY(chol(CH_SHIFT2, F, 2));
    TTR_TRY(accumulate_r(F, 2));
    TTR_TRY(next_pass(T1.p, T2.p, F, 2));
    TTR_TRY(chol(CH_S2PLAIN, F, 2));
    TTR_TRY(accumulate_r(F, 2));
    TTR_TRY(next_pass(T2.p, T1.p, F, 2));
    TTR_TRY(chol(CH_S2LAST, F, 2));
    TTR_TRY(accumulate_r(F, 2));
    TTR_TRY(last_q(T1.p, Q, F, 2));
  } else {
    gated_set_kernel<<<1, 1, 0, s>>>(F, 2, 3);              // route 2 -> 3 (TSQR)
    TTR_TRY(launched());
  }
  if (R)
    TTR_CUDA(cudaMemcpyAsync(R, Racc.p, sizeof(double) * n * n, cudaMemcpyDeviceToDevice, s));
  // ---- route 3 (all CholeskyQR variants failed): R-only QRs of a numerically
  // rank-deficient matrix go to the Householder TSQR; otherwise Householder.
  // Distributed rows: no Householder fallback -- reported as a breakdown.
  if (dist) {
    route_fail_kernel<<<1, 1, 0, s>>>(F);
    return launched();
  }
  if (r_only && tsqr_fits(ni)) {
    TTR_TRY(tsqr_r(c, m, ni, A, lda, trans, R, F, 3, s));
    return TT_OK;
  }
  DBuf hw, htau;
  TTR_TRY(dalloc(hw, size_t(m) * n, s));
  TTR_TRY(dalloc(htau, size_t(n), s));
  householder_kernel<<<1, kHhThreads, 0, s>>>(A, lda, trans, m, ni, hw.p, htau.p,
                                              r_only ? T1.p : Q, R, F);
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
  __shared__ int s_rot;
  for (int e = tid; e < m * n; e += kJacThreads) {
    const int i = e % m, j = e / m;
    W[e] = A[i + int64_t(j) * lda];
  }
  for (int e = tid; e < n * n; e += kJacThreads) V[e] = ((e % n) == (e / n)) ? 1.0 : 0.0;
  __syncthreads();
  // convergence: all column pairs orthogonal to working precision (m eps; the
  // computed cosine carries ~sqrt(m) eps of rounding noise, so a tighter bar
  // would never be met)
  const double tol = double(m) * 0x1p-52;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    __syncthreads();
    int rotated = 0;
    for (int round = 0; round < np - 1; ++round) {
      for (int pi = warp; pi < np / 2; pi += nw) {
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

// B(:, c) = AV(:, c) / sigma_c^pw for c < k (0 when sigma_c is negligible), so that
// B^T H(X_n) = V_k^T Q^T (pw = 2, see svd_nov) or B = U_k (pw = 1).
__global__ void scale_by_inv_sigma_kernel(const double* __restrict__ AV, int m, int k,
                                          const double* __restrict__ sigma,
                                          double* __restrict__ B, int halfpow, double rel_thr) {
  const double s0 = sigma[0];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * k; e += gridDim.x * blockDim.x) {
    const int c = e / m;
    const double sc = sigma[c];
    double p = (halfpow & 1) ? sqrt(sc) : 1.0;   // sigma^(halfpow/2)
    for (int h = 0; h < (halfpow >> 1); ++h) p *= sc;
    B[e] = (sc > s0 * rel_thr) ? AV[e] / p : 0.0;
  }
}

// columns c with sigma_c <= rel_thr sigma_0 (cut by the pseudo-inverse) become e_c,
// so a QR of the matrix stays full rank and finite (two-sided rounding, R20)
__global__ void unit_cut_columns_kernel(double* __restrict__ A, int m, int n,
                                        const double* __restrict__ sigma, double rel_thr) {
  const double s0 = sigma[0];
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < m * n; e += gridDim.x * blockDim.x) {
    const int c = e / m, i = e - c * m;
    if (!(sigma[c] > s0 * rel_thr)) A[e] = (i == c) ? 1.0 : 0.0;
  }
}

// Q(:, c) *= sign(Q(:, c) . ref(:, c)): a QR's column signs follow its reference
// (the Householder fallback's R may have negative diagonal entries)
__global__ void align_column_signs_kernel(double* __restrict__ Q, const double* __restrict__ ref,
                                          int m) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x)
    acc += Q[int64_t(c) * m + i] * ref[int64_t(c) * m + i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = (threadIdx.x < blockDim.x / 32) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  if (red[0] < 0.0)
    for (int i = threadIdx.x; i < m; i += blockDim.x) Q[int64_t(c) * m + i] = -Q[int64_t(c) * m + i];
}

// deterministic sum of squares: fixed grid, per-block partials in block order
constexpr int kSsqBlocks = 256;
__global__ void sumsq_partial_kernel(const double* __restrict__ x, int64_t n,
                                     double* __restrict__ partial) {
  __shared__ double red[32];
  double acc = 0.0;
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    acc = fma(x[e], x[e], acc);
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];
    partial[blockIdx.x] = t;
  }
}

__global__ void sumsq_final_kernel(const double* __restrict__ partial, int np,
                                   double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < np; ++i) t += partial[i];
    *out = t;
  }
}

__global__ void scale_pow2_kernel(double* __restrict__ x, int64_t n, int shift) {
  for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    x[e] = ldexp(x[e], shift);
}

// x <- 2^{-e} x with e = floor(log2 ||x||) from *ssq = ||x||^2 (every thread
// derives e itself; thread 0 stores it): brings ||x|| into [1, 4) exactly
__global__ void normalize_pow2_kernel(double* __restrict__ x, int64_t n,
                                      const double* __restrict__ ssq, int* __restrict__ e_out) {
  const double q = *ssq;
  const int e = (q > 0.0 && q <= 1.7976931348623157e308) ? ilogb(q) / 2 : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *e_out = e;
  if (e == 0) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    x[i] = ldexp(x[i], -e);
}

__global__ void scale_pow2_dev_kernel(double* __restrict__ x, int64_t n, const int* __restrict__ e,
                                      int sign) {
  const int sh = sign * *e;
  if (sh == 0) return;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    x[i] = ldexp(x[i], sh);
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

__global__ void set_identity_kernel(double* p, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    p[i + i * n] = 1.0;
}

// core(a, i, b) <- d[i] core(a, i, b): a diagonal Kronecker factor in mode 2
__global__ void scale_mode2_kernel(const double* __restrict__ x, int64_t r0, int64_t I,
                                   int64_t r1, const double* __restrict__ dg,
                                   double* __restrict__ y) {
  const int64_t n = r0 * I * r1;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    y[e] = dg[(e / r0) % I] * x[e];
}

__global__ void scale_copy_kernel(const double* __restrict__ x, int64_t n, double a,
                                  double* __restrict__ y) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x)
    y[e] = a * x[e];
}

// M (n x n) += factor: kind 0 identity, 1 diagonal d (n), 2 dense F (n x n, ld n)
__global__ void add_factor_kernel(double* __restrict__ M, int n, int kind,
                                  const double* __restrict__ F) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e % n, j = e / n;
    if (kind == 2) M[e] += F[e];
    else if (i == j) M[e] += (kind == 1 ? F[i] : 1.0);
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
  // W does not fit in shared memory: every pair of a round on its own warp of a
  // cooperative grid instead (same pairs and arithmetic)
  if (m * n > kSmemLimitDoubles) return svd_jacobi_grid(c, m, n, A, lda, AV, V, sigma, s);
  static std::atomic<bool> attr{false};
  std::unique_lock<std::mutex> init_lock(init_mutex(), std::defer_lock);
  if (!attr) init_lock.lock();
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

int scale_by_inv_sigma(Ctx& c, const double* AV, int64_t m, int64_t k, const double* sigma,
                       double* B, int halfpow, double rel_thr, cudaStream_t s) {
  const int blocks = int(std::min<int64_t>((m * k + 255) / 256, c.sm_count * 4));
  scale_by_inv_sigma_kernel<<<std::max(1, blocks), 256, 0, s>>>(AV, int(m), int(k), sigma, B,
                                                               halfpow, rel_thr);
  return launched();
}

// One CholeskyQR pass, Q only, for inputs whose columns are already close to
// orthonormal (kappa - 1 small): Q^T Q = I + O(kappa^2 u).  The two-sided
// rounding's V refinement; n <= 160 (blocked Cholesky), else the routed qr().
// tt_cholesky: one factorisation of the CholeskyQR family (R-only modes)
int cholesky(Ctx& c, int64_t n, const double* G, int64_t m, int shifted, double* Rinv, double* L,
             cudaStream_t s) {
  if (n < 1 || n > 1024 || !G || !Rinv) {
    set_error("tt_cholesky: need 1 <= n <= 1024 and G, Rinv");
    return TT_ERR_ARG;
  }
  DBuf gw;
  if (n > 160 && n * n > kSmemLimitDoubles) TTR_TRY(dalloc(gw, size_t(n) * n, s));
  return launch_chol(c, G, int(n), m, shifted ? CH_RSHIFT : CH_RCLAMP, Rinv, L, gw.p, nullptr, 0,
                     s);
}

int qr_near_orthonormal(Ctx& c, int64_t m, int64_t n, const double* A, int64_t lda, double* Q,
                        cudaStream_t s) {
  if (n > 160 || m < n) return qr(c, m, n, A, lda, false, Q, nullptr, s);
  const int ni = int(n), mi = int(m);
  DBuf Gm, Rinv;
  TTR_TRY(dalloc(Gm, size_t(n) * n, s));
  TTR_TRY(dalloc(Rinv, size_t(n) * n, s));
  TTR_TRY(gemm1(c, true, false, ni, ni, mi, 1.0, A, int(lda), A, int(lda), 0.0, Gm.p, ni, s,
                nullptr, 0, kGemmLower));
  TTR_TRY(launch_chol(c, Gm.p, ni, m, CH_RCLAMP, Rinv.p, nullptr, nullptr, nullptr, 0, s));
  return gemm1(c, false, false, mi, ni, ni, 1.0, A, int(lda), Rinv.p, ni, 0.0, Q, mi, s, nullptr,
               0, kGemmTriB);
}

int unit_cut_columns(Ctx& c, double* A, int64_t m, int64_t n, const double* sigma,
                     double rel_thr, cudaStream_t s) {
  const int blocks = int(std::min<int64_t>((m * n + 255) / 256, c.sm_count * 4));
  unit_cut_columns_kernel<<<std::max(1, blocks), 256, 0, s>>>(A, int(m), int(n), sigma, rel_thr);
  return launched();
}

int align_column_signs(Ctx& c, double* Q, const double* ref, int64_t m, int64_t n,
                       cudaStream_t s) {
  align_column_signs_kernel<<<int(n), 256, 0, s>>>(Q, ref, int(m));
  return launched();
}

int sumsq_det(Ctx& c, const double* x, int64_t n, double* out, double* partial,
              cudaStream_t s) {
  sumsq_partial_kernel<<<kSsqBlocks, 256, 0, s>>>(x, n, partial);
  TTR_TRY(launched());
  sumsq_final_kernel<<<1, 32, 0, s>>>(partial, kSsqBlocks, out);
  return launched();
}

int scale_pow2(Ctx& c, double* x, int64_t n, int shift, cudaStream_t s) {
  const int blocks = int(std::min<int64_t>((n + 255) / 256, c.sm_count * 8));
  scale_pow2_kernel<<<std::max(1, blocks), 256, 0, s>>>(x, n, shift);
  return launched();
}

int normalize_pow2(Ctx& c, double* x, int64_t n, double* ssq, double* partial, int* e_out,
                   cudaStream_t s) {
  TTR_TRY(sumsq_det(c, x, n, ssq, partial, s));
  const int blocks = int(std::min<int64_t>((n + 255) / 256, c.sm_count * 8));
  normalize_pow2_kernel<<<std::max(1, blocks), 256, 0, s>>>(x, n, ssq, e_out);
  return launched();
}

int scale_pow2_dev(Ctx& c, double* x, int64_t n, const int* e, int sign, cudaStream_t s) {
  const int blocks = int(std::min<int64_t>((n + 255) / 256, c.sm_count * 8));
  scale_pow2_dev_kernel<<<std::max(1, blocks), 256, 0, s>>>(x, n, e, sign);
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

int set_identity(Ctx& c, double* p, int64_t n, cudaStream_t s) {
  set_identity_kernel<<<std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 64)), 256, 0, s>>>(p, n);
  return launched();
}

int scale_mode2(Ctx& c, const double* x, int64_t r0, int64_t I, int64_t r1, const double* dg,
                double* y, cudaStream_t s) {
  const int64_t n = r0 * I * r1;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8));
  scale_mode2_kernel<<<std::max(1, blocks), 256, 0, s>>>(x, r0, I, r1, dg, y);
  return launched();
}

int scale_copy(Ctx& c, const double* x, int64_t n, double a, double* y, cudaStream_t s) {
  const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8));
  scale_copy_kernel<<<std::max(1, blocks), 256, 0, s>>>(x, n, a, y);
  return launched();
}

int add_factor(Ctx& c, double* M, int n, int kind, const double* F, cudaStream_t s) {
  add_factor_kernel<<<std::max(1, std::min(c.sm_count * 4, (n * n + 255) / 256)), 256, 0, s>>>(
      M, n, kind, F);
  return launched();
}

// Minv = M^{-1} for a symmetric positive definite M (n x n): Cholesky M = R^T R
// (the CholeskyQR kernels, M as the Gram), then Minv = R^{-1} R^{-T}.
int spd_inverse(Ctx& c, const double* M, int n, double* Minv, cudaStream_t s) {
  DBuf Rinv, gw;
  TTR_TRY(dalloc(Rinv, size_t(n) * n, s));
  if (n > 160 && n * n > kSmemLimitDoubles) TTR_TRY(dalloc(gw, size_t(n) * n, s));
  TTR_TRY(launch_chol(c, M, n, n, CH_RCLAMP, Rinv.p, nullptr, gw.p, nullptr, 0, s));
  return gemm1(c, false, true, n, n, n, 1.0, Rinv.p, n, Rinv.p, n, 0.0, Minv, n, s);
}

int fill_zero(Ctx& c, double* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return TT_OK;
  const int blocks = int(std::min<int64_t>((n + 255) / 256, int64_t(c.sm_count) * 8));
  fill_zero_kernel<<<blocks, 256, 0, s>>>(p, n);
  return launched();
}

}  // namespace ttr
