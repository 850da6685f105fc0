// One CholeskyQR pass of a tall-skinny QR in one persistent launch (round 2):
//
//   Q = op(A) R^{-1}   (R^{-1} upper triangular, from the previous pass's Cholesky)
//   G = Q^T Q          (the Gram the next pass's Cholesky factors)
//
// The CholeskyQR family (CholeskyQR2, shifted CholeskyQR3, the truncation's
// 4-pass R-only QR) used for the thin QR of Alg. 7 line 10
// ([Q_n, R_n] = QR(Y_n)) and for the QR of H(X_n)^T in the truncation
// (Alg. 2 line 4, run on the left-orthogonal result) alternates
// these two products.  As two GEMM launches they read Q_{k-1}, write Q_k, read
// Q_k back, and the Gram (a 144 x 144 output from K = 36864) needs a split-K
// partial buffer plus a reduction launch.  Here every CTA (one per SM) streams
// 32-row chunks of op(A) through shared memory (cp.async, double-buffered): the
// chunk times R^{-1} on DMMA tiles (R^{-1} staged once per CTA in
// fragment-swizzled 8 x 8 tiles, upper tiles only), written back into the chunk
// buffer, then the chunk's contribution to the lower 16 x 16 blocks of the Gram
// accumulated in registers across all of the CTA's chunks, and the chunk of Q
// stored.  Inner loops use 32-bit shared addresses with compile-time offsets
// (a first version with generic pointers and per-tile index arithmetic issued
// ~20 instructions per DMMA and ran at 6 TF/s).  One partial Gram per CTA is summed in CTA order by a second small
// kernel (deterministic; both triangles of G written).
//
// Modes: Rinv == nullptr -> Q = op(A) (Gram only); G == nullptr -> no Gram
// (the final Q of a QR).  n <= 144 (larger n: the two-GEMM form).
//
// FP64 tensor path: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4); fragment layouts:
// A(row = lane>>2, k = lane&3), B(k = lane&3, col = lane>>2),
// D(row = lane>>2, col = 2(lane&3) + {0, 1}).
#include "common.cuh"

namespace ttr {

namespace {

constexpr int kBM = 32;              // rows per chunk
constexpr int kLdc = kBM + 4;        // chunk buffer: column-major, ld 36 = 4 mod 16 doubles
constexpr int kThreads = 512;        // 16 warps: 4 per SM sub-partition
constexpr int kMaxT = 18;            // n <= 144: 18 column tiles of 8
constexpr int kMaxNT = kMaxT * (kMaxT + 1) / 2;   // upper 8 x 8 tiles of R^{-1}
constexpr int kMaxB = 9;                          // 16-column blocks (n <= 144)
constexpr int kMaxNB = kMaxB * (kMaxB + 1) / 2;   // lower 16 x 16 Gram blocks (55)
constexpr int kPart = kMaxNB * 256;               // doubles per CTA partial Gram

struct CqrParams {
  const double* A;
  int64_t lda;
  int64_t m;
  int n, T;            // n, column tiles T = ceil(n / 8)
  const double* Rinv;  // n x n upper (ld n) or nullptr
  double* Q;           // m x n (ld ldq) or nullptr
  int64_t ldq;
  double* ws;          // partial Grams: gridDim.x x kPart
  int64_t nchunks;
  const int* gate;
  int gate_val;
  int vec;             // 16-byte cp.async for the non-transposed load
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts(uint32_t a, double v) {
  asm volatile("st.shared.f64 [%0], %1;\n" ::"r"(a), "d"(v));
}
__device__ __forceinline__ uint32_t saddr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cpa8(uint32_t sa, const double* gmem, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(pred ? 8 : 0));
}
__device__ __forceinline__ void cpa16(uint32_t sa, const double* gmem, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem),
               "r"(bytes));
}

// chunk rows [r0, r0 + 32) of op(A), columns [0, nc) -> buf (column-major, ld 36);
// rows past m and columns past n are zero-filled (nc = 16 * ceil(n / 16): the
// Gram's 16-column blocks read up to there)
template <bool TRANS>
__device__ __forceinline__ void load_chunk(const CqrParams& p, int64_t r0, uint32_t buf, int nc) {
  if (TRANS) {
    // op(A)(r, c) = A[c + r lda]: consecutive threads read consecutive c
    for (int e = threadIdx.x; e < kBM * nc; e += kThreads) {
      const int r = e / nc, c = e - r * nc;
      const bool ok = (r0 + r < p.m) && c < p.n;
      cpa8(buf + 8u * (c * kLdc + r), ok ? p.A + c + (r0 + r) * p.lda : p.A, ok);
    }
  } else if (p.vec) {
    // 16 threads per column, two rows each
    for (int e = threadIdx.x; e < 16 * nc; e += kThreads) {
      const int c = e >> 4, r = 2 * (e & 15);
      const int64_t rem = p.m - (r0 + r);
      const int bytes = (c < p.n) ? (rem >= 2 ? 16 : (rem == 1 ? 8 : 0)) : 0;
      cpa16(buf + 8u * (c * kLdc + r), bytes ? p.A + (r0 + r) + c * p.lda : p.A, bytes);
    }
  } else {
    for (int e = threadIdx.x; e < kBM * nc; e += kThreads) {
      const int c = e >> 5, r = e & 31;
      const bool ok = (r0 + r < p.m) && c < p.n;
      cpa8(buf + 8u * (c * kLdc + r), ok ? p.A + (r0 + r) + c * p.lda : p.A, ok);
    }
  }
}

// column tile of product slot j (increasing in j; -1 = unused slot) for warp
// group G (0..3) of a row tile.  NJ = 3 (T <= 12): {G, 7-G, 8+G}.  NJ = 6
// (T <= 18): a split of tiles 0..17 whose triangular work (tile ct has ct + 1
// k-tiles) is 45/44/44/38 k-tiles -- the slowest group sets the time (a
// {G, 7-G, 8+G, 15-G, 16+G} split with padding tiles was 52 for every group).
__device__ __forceinline__ constexpr int ct_tab(int NJ, int G, int j) {
  constexpr int t6[4][6] = {{-1, -1, 1, 7, 16, 17}, {-1, -1, 3, 8, 14, 15},
                            {-1, -1, 6, 9, 12, 13}, {0, 2, 4, 5, 10, 11}};
  return NJ == 3 ? 8 * (j >> 1) + ((j & 1) ? 7 - G : G) : t6[G][j];
}

// acc(8 rows of row tile rt, column tiles ct_tab(j), j < NJ) = chunk(rt rows, :) R^{-1}.
// R^{-1}(k, c) = 0 for k > c: product tile j needs k-tiles kt <= ct_tab(j).  Since
// ct_tab is increasing, the k-tiles split into compile-time blocks S: kt in
// (ct_tab(S-1), ct_tab(S)] feeds exactly the tiles j >= S -- no predicated DMMA.
// Tiles with ct >= T multiply zero-padded R^{-1} tiles (never stored).
template <int G, int NJ, int S>
__device__ __forceinline__ void trsm_block(uint32_t ap, uint32_t bp, int T,
                                           double (&acc)[NJ][2]) {
  if constexpr (S < NJ) {
    constexpr int lo = (S == 0) ? 0 : ct_tab(NJ, G, S - 1) + 1;
    const int hi = min(ct_tab(NJ, G, S), T - 1);
#pragma unroll 1
    for (int kt = lo; kt <= hi; ++kt) {
      const double a0 = lds(ap + 8u * (8 * kt * kLdc));
      const double a1 = lds(ap + 8u * ((8 * kt + 4) * kLdc));
      const uint32_t bk = bp + 512u * kt;
      double b0[NJ - S], b1[NJ - S];
#pragma unroll
      for (int j = S; j < NJ; ++j) {
        const uint32_t t = bk + 512u * (ct_tab(NJ, G, j) * (ct_tab(NJ, G, j) + 1) / 2);
        b0[j - S] = lds(t);
        b1[j - S] = lds(t + 256u);
      }
      // the a0 products of every tile, then the a1 products: consecutive DMMAs
      // are independent
#pragma unroll
      for (int j = S; j < NJ; ++j) dmma(acc[j][0], acc[j][1], a0, b0[j - S]);
#pragma unroll
      for (int j = S; j < NJ; ++j) dmma(acc[j][0], acc[j][1], a1, b1[j - S]);
    }
    trsm_block<G, NJ, S + 1>(ap, bp, T, acc);
  }
}

// NJ: product column slots per warp (every tile < T covered: NJ = 3 -> T <= 12,
// NJ = 6 -> T <= 18); BPW: Gram blocks per warp (>= ceil(NB / 16))
template <bool TRANS, bool TRSM, bool GRAM, int NJ, int BPW>
__global__ void __launch_bounds__(kThreads, 1) cqr_pass_kernel(const CqrParams p) {
  if (p.gate && *p.gate != p.gate_val) return;
  extern __shared__ __align__(16) double sm[];
  // layout: R^{-1} tiles (TRSM) | chunk buffers A0, A1 | product buffer C (TRSM).
  // Product tiles with ct >= T (a group's slots past the matrix) read "R^{-1}
  // tiles" past the NT stored ones -- inside the allocation (launch_cfg sizes it),
  // values unused: those accumulators are never stored.
  const int T = p.T, NT = T * (T + 1) / 2;
  const int B = (T + 1) / 2, NB = B * (B + 1) / 2, nc = 16 * B;
  const uint32_t sR = saddr(sm);
  const uint32_t sA0 = sR + 8u * (TRSM ? NT * 64 : 0);
  const uint32_t sA1 = sA0 + 8u * (nc * kLdc);
  const uint32_t sCb = sA1 + 8u * (nc * kLdc);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t grid = gridDim.x;
  int64_t chunk = blockIdx.x;

  load_chunk<TRANS>(p, chunk * kBM, sA0, nc);
  asm volatile("cp.async.commit_group;\n" ::);

  if (TRSM) {
    // R^{-1} (upper) into 8 x 8 tiles (kt <= ct < T, tile index ct(ct+1)/2 + kt;
    // zero past n), each as two 4 x 8 halves in B-fragment lane order: lane l of
    // half h holds (k = 8kt + 4h + (l & 3), col = 8ct + (l >> 2)); a warp writes
    // one half-tile
    // (asynchronous: cp.async with zero fill, overlapped with the first chunk)
    int hidx = 0;
    for (int ct = 0; ct < T; ++ct)
      for (int kt = 0; kt <= ct; ++kt)
        for (int h = 0; h < 2; ++h, ++hidx) {
          if ((hidx & 15) != w) continue;
          const int k = 8 * kt + 4 * h + (lane & 3), col = 8 * ct + (lane >> 2);
          const bool ok = k <= col && col < p.n;
          cpa8(sR + 8u * ((ct * (ct + 1) / 2 + kt) * 64 + h * 32 + lane),
               ok ? p.Rinv + k + int64_t(col) * p.n : p.Rinv, ok);
        }
    asm volatile("cp.async.commit_group;\n" ::);
  }

  // Gram blocks of this warp: 16 x 16 blocks (I >= J) numbered row-major, a run
  // [b0, b1) per warp; packed byte offsets of columns 16I and 16J in the chunk
  const int bpw = (NB + 15) / 16;
  const int b0 = min(NB, w * bpw), b1 = min(NB, b0 + bpw);
  uint32_t boff[BPW];
  {
    int I = 0;
    while ((I + 1) * (I + 2) / 2 <= b0) ++I;
    int J = b0 - I * (I + 1) / 2;
#pragma unroll
    for (int q = 0; q < BPW; ++q) {
      boff[q] = uint32_t(16 * I * kLdc * 8) | (uint32_t(16 * J * kLdc * 8) << 16);
      if (++J > I) { ++I; J = 0; }
    }
  }
  double gacc[BPW][4][2];
#pragma unroll
  for (int q = 0; q < BPW; ++q)
#pragma unroll
    for (int t = 0; t < 4; ++t) gacc[q][t][0] = gacc[q][t][1] = 0.0;

  const int rt = w & 3, grp = w >> 2;

  // per chunk: wait for it (and, before the barrier, nothing else is in flight),
  // barrier (every warp is done with the previous chunk), prefetch the next chunk
  // into the other buffer, R^{-1} product into C, barrier, Gram of C, Q stored
  for (int it = 0; chunk < p.nchunks; ++it, chunk += grid) {
    const uint32_t cur = (it & 1) ? sA1 : sA0;
    const uint32_t nxt = (it & 1) ? sA0 : sA1;
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    if (chunk + grid < p.nchunks) load_chunk<TRANS>(p, (chunk + grid) * kBM, nxt, nc);
    asm volatile("cp.async.commit_group;\n" ::);
    uint32_t cbuf = cur;

    if (TRSM) {
      double acc[NJ][2];
#pragma unroll
      for (int j = 0; j < NJ; ++j) acc[j][0] = acc[j][1] = 0.0;
      const uint32_t ap = cur + 8u * ((lane & 3) * kLdc + 8 * rt + (lane >> 2));
      const uint32_t bp = sR + 8u * lane;
      switch (grp) {
        case 0: trsm_block<0, NJ, 0>(ap, bp, T, acc); break;
        case 1: trsm_block<1, NJ, 0>(ap, bp, T, acc); break;
        case 2: trsm_block<2, NJ, 0>(ap, bp, T, acc); break;
        default: trsm_block<3, NJ, 0>(ap, bp, T, acc); break;
      }
      const uint32_t dp = sCb + 8u * ((2 * (lane & 3)) * kLdc + 8 * rt + (lane >> 2));
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int ct = grp == 0 ? ct_tab(NJ, 0, j) : grp == 1 ? ct_tab(NJ, 1, j)
                       : grp == 2 ? ct_tab(NJ, 2, j) : ct_tab(NJ, 3, j);
        if (ct >= 0 && ct < T) {
          sts(dp + 8u * (8 * ct * kLdc), acc[j][0]);
          sts(dp + 8u * ((8 * ct + 1) * kLdc), acc[j][1]);
        }
      }
      __syncthreads();
      cbuf = sCb;
    }

    if (GRAM) {
      // block (I, J): G(16I + a, 16J + b) += sum_r C(r, 16I + a) C(r, 16J + b);
      // fragment F(c0) = C(4kk + (l & 3), c0 + (l >> 2)) is A (c0 = 16I, 16I + 8)
      // and B (c0 = 16J, 16J + 8)
      const uint32_t fp = cbuf + 8u * ((lane >> 2) * kLdc + (lane & 3));
      if (b1 - b0 == BPW) {
#pragma unroll 1
        for (int kk = 0; kk < kBM / 4; ++kk) {
          const uint32_t f = fp + 32u * kk;
          double fa[BPW][2], fb[BPW][2];   // every fragment of the k-step first
#pragma unroll
          for (int q = 0; q < BPW; ++q) {
            const uint32_t oa = f + (boff[q] & 0xffffu), ob = f + (boff[q] >> 16);
            fa[q][0] = lds(oa);
            fa[q][1] = lds(oa + 8u * 8 * kLdc);
            fb[q][0] = lds(ob);
            fb[q][1] = lds(ob + 8u * 8 * kLdc);
          }
#pragma unroll
          for (int q = 0; q < BPW; ++q) {
            dmma(gacc[q][0][0], gacc[q][0][1], fa[q][0], fb[q][0]);
            dmma(gacc[q][1][0], gacc[q][1][1], fa[q][0], fb[q][1]);
            dmma(gacc[q][2][0], gacc[q][2][1], fa[q][1], fb[q][0]);
            dmma(gacc[q][3][0], gacc[q][3][1], fa[q][1], fb[q][1]);
          }
        }
      } else {   // the last warps of a ragged split
#pragma unroll 1
        for (int kk = 0; kk < kBM / 4; ++kk) {
          const uint32_t f = fp + 32u * kk;
#pragma unroll
          for (int q = 0; q < BPW; ++q) {
            if (b0 + q < b1) {
              const uint32_t oa = f + (boff[q] & 0xffffu), ob = f + (boff[q] >> 16);
              const double a0 = lds(oa), a1 = lds(oa + 8u * 8 * kLdc);
              const double c0 = lds(ob), c1 = lds(ob + 8u * 8 * kLdc);
              dmma(gacc[q][0][0], gacc[q][0][1], a0, c0);
              dmma(gacc[q][1][0], gacc[q][1][1], a0, c1);
              dmma(gacc[q][2][0], gacc[q][2][1], a1, c0);
              dmma(gacc[q][3][0], gacc[q][3][1], a1, c1);
            }
          }
        }
      }
    }

    if (p.Q) {
      const int64_t r0 = chunk * kBM;
      const double* cb = sm + (cbuf - sR) / 8;
      for (int e = tid; e < kBM * p.n; e += kThreads) {
        const int c = e >> 5, r = e & 31;
        if (r0 + r < p.m) p.Q[(r0 + r) + c * p.ldq] = cb[c * kLdc + r];
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);

  if (GRAM) {
    // partial block q, sub-tile t (t = 2 (a-half) + (b-half)), lane layout
    double* out = p.ws + int64_t(blockIdx.x) * kPart;
#pragma unroll
    for (int q = 0; q < BPW; ++q)
      if (b0 + q < b1)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          out[(b0 + q) * 256 + t * 64 + 2 * lane] = gacc[q][t][0];
          out[(b0 + q) * 256 + t * 64 + 2 * lane + 1] = gacc[q][t][1];
        }
  }
}

// G = sum over the CTAs' partial Grams, in CTA order; both triangles written
__global__ void cqr_gram_reduce_kernel(const double* __restrict__ ws, int nparts, int n, int B,
                                       double* __restrict__ G, const int* gate, int gate_val) {
  if (gate && *gate != gate_val) return;
  const int NB = B * (B + 1) / 2;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= NB * 256) return;
  const int b = e >> 8, t = (e >> 6) & 3, x = e & 63;
  int I = 0;
  while ((I + 1) * (I + 2) / 2 <= b) ++I;
  const int J = b - I * (I + 1) / 2;
  const int l = x >> 1;
  const int row = 16 * I + 8 * (t >> 1) + (l >> 2), col = 16 * J + 8 * (t & 1) + 2 * (l & 3) + (x & 1);
  double s = 0.0;
  for (int k = 0; k < nparts; ++k) s += ws[int64_t(k) * kPart + e];
  if (row < n && col < n && row >= col) {
    G[row + int64_t(col) * n] = s;
    G[col + int64_t(row) * n] = s;
  }
}

template <bool TRANS, bool TRSM, bool GRAM, int NJ, int BPW>
int launch_cfg(Ctx& c, const CqrParams& p, int grid, cudaStream_t s) {
  auto kern = cqr_pass_kernel<TRANS, TRSM, GRAM, NJ, BPW>;
  static std::atomic<bool> attr[64];
  const size_t maxshm = 227 * 1024;
  std::unique_lock<std::mutex> lk(init_mutex(), std::defer_lock);
  if (!attr[c.device & 63]) lk.lock();
  if (!attr[c.device & 63]) {
    TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(maxshm)));
    attr[c.device & 63] = true;
  }
  const int T = p.T, NT = T * (T + 1) / 2, B = (T + 1) / 2;
  size_t shm = size_t((TRSM ? NT * 64 : 0) + (TRSM ? 3 : 2) * 16 * B * kLdc) * sizeof(double);
  if (TRSM) {
    // the padded slots' reads (ct up to the groups' largest tile, kt < T) stay inside
    int ctmax = 0;
    for (int g = 0; g < 4; ++g)
      for (int j = 0; j < NJ; ++j) ctmax = std::max(ctmax, ct_tab(NJ, g, j));
    shm = std::max(shm, size_t(ctmax * (ctmax + 1) / 2 + T) * 512 + 512);
  }
  if (shm > maxshm) {
    set_error("cqr_pass: %zu bytes of shared memory needed", shm);
    return TT_ERR_ARG;
  }
  kern<<<grid, kThreads, shm, s>>>(p);
  return launched();
}

// (NJ, BPW): T <= 12 -> (3, 2); T <= 18 -> (6, 3)
template <bool TRANS, bool TRSM, bool GRAM>
int launch(Ctx& c, const CqrParams& p, int grid, cudaStream_t s) {
  if (p.T <= 12) return launch_cfg<TRANS, TRSM, GRAM, 3, 2>(c, p, grid, s);
  return launch_cfg<TRANS, TRSM, GRAM, 6, 3>(c, p, grid, s);
}

}  // namespace

bool cqr_fits(int64_t n) { return n >= 1 && n <= 8 * kMaxT; }

int cqr_pass(Ctx& c, int64_t m, int n, const double* A, int64_t lda, bool trans,
             const double* Rinv, double* Q, int64_t ldq, double* G, cudaStream_t s,
             const int* gate, int gate_val) {
  if (!cqr_fits(n) || m < 0 || (!Q && !G)) {
    set_error("cqr_pass: unsupported shape (m=%lld n=%d)", (long long)m, n);
    return TT_ERR_ARG;
  }
  if (m == 0) {
    if (gate) {
      set_error("cqr_pass: m = 0 with a gate");
      return TT_ERR_ARG;
    }
    if (G) TTR_TRY(fill_zero(c, G, int64_t(n) * n, s));
    return TT_OK;
  }
  CqrParams p;
  p.A = A;
  p.lda = lda;
  p.m = m;
  p.n = n;
  p.T = (n + 7) / 8;
  p.Rinv = Rinv;
  p.Q = Q;
  p.ldq = ldq;
  p.nchunks = (m + kBM - 1) / kBM;
  p.gate = gate;
  p.gate_val = gate_val;
  p.vec = !trans && !(reinterpret_cast<uintptr_t>(A) & 15) && !(lda & 1);
  const int grid = int(std::min<int64_t>(p.nchunks, grid_sms(c)));
  p.ws = nullptr;
  if (G) {
    const size_t need = size_t(c.sm_count) * kPart;
    if (c.cqr_ws.n < need) {
      if (c.capturing) {
        set_error("cqr workspace must be sized before graph capture");
        return TT_ERR_ARG;
      }
      TTR_TRY(dalloc(c.cqr_ws, need, s));
    }
    p.ws = c.cqr_ws.p;
  }
  int rc;
  if (Rinv) {
    if (G) rc = trans ? launch<true, true, true>(c, p, grid, s) : launch<false, true, true>(c, p, grid, s);
    else rc = trans ? launch<true, true, false>(c, p, grid, s) : launch<false, true, false>(c, p, grid, s);
  } else {
    rc = trans ? launch<true, false, true>(c, p, grid, s) : launch<false, false, true>(c, p, grid, s);
  }
  TTR_TRY(rc);
  if (G) {
    const int B = (p.T + 1) / 2, NB = B * (B + 1) / 2;
    cqr_gram_reduce_kernel<<<NB, 256, 0, s>>>(p.ws, grid, n, B, G, gate, gate_val);
    TTR_TRY(launched());
  }
  return TT_OK;
}

}  // namespace ttr
