// FP64 tensor-core GEMM for sm_100a: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4),
// operands staged global -> shared memory by a multi-stage cp.async pipeline.
//
// Every contraction of the hot path (Alg. 3 lines 2/4/5, Alg. 7 lines 9/11/13/14,
// the Gram/R^{-1} products of the QR and the truncation products) is a
// column-major C = alpha*op(A)*op(B) + beta*C launched through gemm() below,
// batched over summands with per-entry pointers/shapes, and split along K with
// a fixed-order (deterministic) reduction when M*N alone cannot fill 148 SMs.
//
// On B200 tcgen05.mma has no f64 kind (ptxas rejects .kind::f64), so the
// warp-level DMMA is the FP64 tensor path; see DESIGN.md §Kernels.
#include "common.cuh"
#include "dmma_tma.cuh"

namespace ttr {

namespace {

constexpr int pad_for(int x) { return (20 - (x % 16)) % 16; }  // leading dim ≡ 4 (mod 16) doubles

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool pred) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, int bytes) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

struct GemmParams {
  GemmDesc d[kMaxGemmBatch];
  int nbatch;
  int tiles_m, tiles_n;
  int kslices;
  int kchunk;        // K per slice (multiple of BK)
  double alpha, beta;
  double* ws;        // split-K partials (kslices > 1)
  const int* gate;   // device-side predicate: run iff gate == nullptr || *gate == gate_val
  int gate_val;
  int vec;           // 1: every A/B 16-byte aligned with even leading dimensions
  int flags;         // kGemmTriB / kGemmLower (common.cuh)
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB>
struct Cfg {
  static constexpr int NT = WM * WN * 32;
  static constexpr int TM = BM / WM, TN = BN / WN;
  static constexpr int FM = TM / 8, FN = TN / 8;
  static constexpr int LDA = TA ? (BK + pad_for(BK)) : (BM + pad_for(BM));
  static constexpr int AEL = TA ? BM * LDA : BK * LDA;
  static constexpr int LDB = TB ? (BN + pad_for(BN)) : (BK + pad_for(BK));
  static constexpr int BEL = TB ? BK * LDB : BN * LDB;
  static constexpr int SEL = AEL + BEL;
  static constexpr size_t SMEM = size_t(STAGES) * SEL * sizeof(double);
  static_assert(TM % 8 == 0 && TN % 8 == 0, "warp tile must be a multiple of 8");
  static_assert(BK % 4 == 0, "BK multiple of 4");
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB>
__global__ void __launch_bounds__(WM* WN * 32)
    dgemm_kernel(const __grid_constant__ GemmParams P) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, TA, TB>;
  extern __shared__ __align__(16) double smem[];
  if (P.gate && *P.gate != P.gate_val) return;

  const int tn = blockIdx.x, tm = blockIdx.y;
  const int b = blockIdx.z % P.nbatch;
  const int ks = blockIdx.z / P.nbatch;
  const GemmDesc& D = P.d[b];
  const int m0 = tm * BM, n0 = tn * BN;
  // kGemmLower: only tiles meeting the lower triangle (the Cholesky reads no more)
  if ((P.flags & kGemmLower) && m0 + BM <= n0) return;
  const bool tile_live = (m0 < D.M) && (n0 < D.N);
  if (!tile_live && P.kslices == 1) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % WM) * C::TM;
  const int wn0 = (warp / WM) * C::TN;

  const int kbeg = ks * P.kchunk;
  // kGemmTriB: B upper triangular (B(k, n) = 0 for k > n): columns < n0 + BN
  // need k < n0 + BN only
  const int kend = min(min(D.K, kbeg + P.kchunk), (P.flags & kGemmTriB) ? n0 + BN : D.K);
  const int KT = (tile_live && kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;

  const double* __restrict__ A = D.A;
  const double* __restrict__ B = D.B;
  const int64_t lda = D.lda, ldb = D.ldb;

  auto load_tile = [&](int slot, int k0) {
    double* sA = smem + slot * C::SEL;
    double* sB = sA + C::AEL;
#pragma unroll 4
    for (int idx = tid; idx < BM * BK; idx += C::NT) {
      int m, k;
      if (TA) { k = idx % BK; m = idx / BK; } else { m = idx % BM; k = idx / BM; }
      const int gm = m0 + m, gk = k0 + k;
      const bool p = (gm < D.M) && (gk < kend);
      const double* src = p ? (TA ? A + gk + int64_t(gm) * lda : A + gm + int64_t(gk) * lda) : A;
      double* dst = TA ? sA + m * C::LDA + k : sA + k * C::LDA + m;
      cp_async8(dst, src, p);
    }
#pragma unroll 4
    for (int idx = tid; idx < BN * BK; idx += C::NT) {
      int n, k;
      if (TB) { n = idx % BN; k = idx / BN; } else { k = idx % BK; n = idx / BK; }
      const int gn = n0 + n, gk = k0 + k;
      const bool p = (gn < D.N) && (gk < kend);
      const double* src = p ? (TB ? B + gn + int64_t(gk) * ldb : B + gk + int64_t(gn) * ldb) : B;
      double* dst = TB ? sB + k * C::LDB + n : sB + n * C::LDB + k;
      cp_async8(dst, src, p);
    }
  };

  // 16-byte path (P.vec): each thread's cp.async sources are computed once and
  // advanced by one k-tile per load; vectors run along the contiguous dimension
  // of each operand (m or k for A, k or n for B); a vector straddling the M/N
  // edge or the end of the K slice copies 8 bytes and zero-fills the rest
  constexpr int AVn = BM * BK / 2, BVn = BN * BK / 2;
  constexpr int NAL = (AVn + C::NT - 1) / C::NT, NBL = (BVn + C::NT - 1) / C::NT;
  const double* a_ptr[NAL];
  const double* b_ptr[NAL > NBL ? NAL : NBL];
  int a_dst[NAL], b_dst[NBL], a_k[NAL], b_k[NBL];
  bool a_ok[NAL], b_ok[NBL];
  int a_full[NAL], b_full[NBL];
  if (P.vec) {
#pragma unroll
    for (int i = 0; i < NAL; ++i) {
      const int v = tid + i * C::NT;
      int m, k;
      if (TA) { k = 2 * (v % (BK / 2)); m = v / (BK / 2); }
      else { m = 2 * (v % (BM / 2)); k = v / (BM / 2); }
      const bool in = v < AVn;
      a_ok[i] = in && (m0 + m < D.M);
      a_full[i] = TA ? 16 : ((m0 + m + 1 < D.M) ? 16 : 8);
      a_k[i] = k;
      a_dst[i] = TA ? m * C::LDA + k : k * C::LDA + m;
      a_ptr[i] = a_ok[i] ? (TA ? A + (kbeg + k) + int64_t(m0 + m) * lda
                               : A + (m0 + m) + int64_t(kbeg + k) * lda) : A;
    }
#pragma unroll
    for (int i = 0; i < NBL; ++i) {
      const int v = tid + i * C::NT;
      int n, k;
      if (TB) { n = 2 * (v % (BN / 2)); k = v / (BN / 2); }
      else { k = 2 * (v % (BK / 2)); n = v / (BK / 2); }
      const bool in = v < BVn;
      b_ok[i] = in && (n0 + n < D.N);
      b_full[i] = TB ? ((n0 + n + 1 < D.N) ? 16 : 8) : 16;
      b_k[i] = k;
      b_dst[i] = TB ? k * C::LDB + n : n * C::LDB + k;
      b_ptr[i] = b_ok[i] ? (TB ? B + (n0 + n) + int64_t(kbeg + k) * ldb
                               : B + (kbeg + k) + int64_t(n0 + n) * ldb) : B;
    }
  }
  auto load_tile_vec = [&](int slot, int kt) {
    double* sA = smem + slot * C::SEL;
    double* sB = sA + C::AEL;
    const int k0 = kbeg + kt * BK;
#pragma unroll
    for (int i = 0; i < NAL; ++i) {
      if (tid + i * C::NT < AVn) {
        const int rem = kend - (k0 + a_k[i]);   // K left from this vector's first k
        int bytes = a_ok[i] ? (TA ? (rem >= 2 ? 16 : (rem == 1 ? 8 : 0)) : (rem >= 1 ? a_full[i] : 0)) : 0;
        const double* src = a_ptr[i] + (TA ? int64_t(kt) * BK : int64_t(kt) * BK * lda);
        cp_async16(sA + a_dst[i], bytes ? src : A, bytes);
      }
    }
#pragma unroll
    for (int i = 0; i < NBL; ++i) {
      if (tid + i * C::NT < BVn) {
        const int rem = kend - (k0 + b_k[i]);
        int bytes = b_ok[i] ? (TB ? (rem >= 1 ? b_full[i] : 0) : (rem >= 2 ? 16 : (rem == 1 ? 8 : 0))) : 0;
        const double* src = b_ptr[i] + (TB ? int64_t(kt) * BK * ldb : int64_t(kt) * BK);
        cp_async16(sB + b_dst[i], bytes ? src : B, bytes);
      }
    }
  };

  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) {
      if (P.vec) load_tile_vec(s, s);
      else load_tile(s, kbeg + s * BK);
    }
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int nk = kt + STAGES - 1;
    if (nk < KT) {
      if (P.vec) load_tile_vec(nk % STAGES, nk);
      else load_tile(nk % STAGES, kbeg + nk * BK);
    }
    cp_async_commit();

    const double* sA = smem + (kt % STAGES) * C::SEL;
    const double* sB = sA + C::AEL;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[C::FM], bf[C::FN];
#pragma unroll
      for (int i = 0; i < C::FM; ++i) {
        const int m = wm0 + i * 8 + g;
        af[i] = TA ? sA[m * C::LDA + kk + t] : sA[(kk + t) * C::LDA + m];
      }
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int n = wn0 + j * 8 + g;
        bf[j] = TB ? sB[(kk + t) * C::LDB + n] : sB[n * C::LDB + kk + t];
      }
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  if (P.kslices == 1) {
    const double alpha = P.alpha, beta = P.beta;
    double* Cp = D.C;
    const int64_t ldc = D.ldc;
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int m = m0 + wm0 + i * 8 + g;
      if (m >= D.M) continue;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + j * 8 + 2 * t + e;
          if (n < D.N) {
            double* cp = Cp + m + int64_t(n) * ldc;
            double v = alpha * acc[i][j][e];
            if (beta != 0.0) v += beta * *cp;
            *cp = v;
          }
        }
      }
    }
  } else {
    // partial tile -> workspace [ks][b][tm][tn][BM x BN] (column-major in the tile)
    const size_t tile = ((size_t(ks) * P.nbatch + b) * P.tiles_m + tm) * P.tiles_n + tn;
    double* W = P.ws + tile * (BM * BN);
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int ml = wm0 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int nl = wn0 + j * 8 + 2 * t;
        W[ml + nl * BM] = acc[i][j][0];
        W[ml + (nl + 1) * BM] = acc[i][j][1];
      }
    }
  }
}

// ------------------------------------------------------------------ TMA-fed variant
// The same tiles, warp layout, k order and epilogue as dgemm_kernel (so the
// results are bit-identical), but every operand tile is moved global -> shared
// by the Tensor Memory Accelerator: one elected thread issues a 2-D
// cp.async.bulk.tensor per operand per stage, completion is tracked by one
// mbarrier per stage (expect-tx bytes), and no thread computes a global address.
// The box of a tile is its padded shared-memory footprint (leading dimension
// LD = tile + 4 doubles, ≡ 4 mod 16: conflict-free fragment loads), i.e. TMA
// over-fetches 4 rows that the fragments never read; rows/columns past the
// matrix edge are zero-filled by the TMA unit (the cp.async path's predicate).
constexpr int kMaxTmaBatch = 32;

struct TmaParams {
  GemmParams g;
  alignas(64) CUtensorMap tm[2 * kMaxTmaBatch];   // [2b] = A of entry b, [2b+1] = B
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB>
struct TmaCfg {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, TA, TB>;
  static constexpr int AB = ((C::AEL * 8 + 127) / 128) * 128;   // bytes, 128-aligned
  static constexpr int BB = ((C::BEL * 8 + 127) / 128) * 128;
  static constexpr int SB = AB + BB;
  static constexpr size_t SMEM = size_t(STAGES) * SB + 128 + 8 * STAGES;
  static constexpr uint32_t TX = uint32_t(C::AEL + C::BEL) * 8;   // full boxes, OOB included
};

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB>
__global__ void __launch_bounds__(WM* WN * 32)
    dgemm_tma_kernel(const __grid_constant__ TmaParams T) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, TA, TB>;
  using X = TmaCfg<BM, BN, BK, WM, WN, STAGES, TA, TB>;
  extern __shared__ __align__(128) unsigned char tsm[];
  const GemmParams& P = T.g;
  if (P.gate && *P.gate != P.gate_val) return;
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tsm) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + STAGES * X::SB);

  const int tn = blockIdx.x, tm = blockIdx.y;
  const int b = blockIdx.z % P.nbatch;
  const int ks = blockIdx.z / P.nbatch;
  const GemmDesc& D = P.d[b];
  const int m0 = tm * BM, n0 = tn * BN;
  if ((P.flags & kGemmLower) && m0 + BM <= n0) return;
  const bool tile_live = (m0 < D.M) && (n0 < D.N);
  if (!tile_live && P.kslices == 1) return;

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % WM) * C::TM;
  const int wn0 = (warp / WM) * C::TN;
  const int kbeg = ks * P.kchunk;
  const int kend = min(min(D.K, kbeg + P.kchunk), (P.flags & kGemmTriB) ? n0 + BN : D.K);
  const int KT = (tile_live && kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;
  const CUtensorMap* mapA = &T.tm[2 * b];
  const CUtensorMap* mapB = &T.tm[2 * b + 1];

  if (tid == 0) {
#pragma unroll
    for (int s2 = 0; s2 < STAGES; ++s2) mbar_init(full + s2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // stage `slot` <- k-tile kt: A box at (row m0, col k0) [or (k0, m0) when
  // transposed], B box at (k0, n0) [or (n0, k0)]; coordinates innermost first
  auto issue = [&](int slot, int kt) {
    unsigned char* sA = base + slot * X::SB;
    unsigned char* sB = sA + X::AB;
    const int k0 = kbeg + kt * BK;
    mbar_expect_tx(full + slot, X::TX);
    if (TA) tma_load_2d(sA, mapA, k0, m0, full + slot);
    else tma_load_2d(sA, mapA, m0, k0, full + slot);
    if (TB) tma_load_2d(sB, mapB, n0, k0, full + slot);
    else tma_load_2d(sB, mapB, k0, n0, full + slot);
  };
  if (tid == 0) {
#pragma unroll
    for (int s2 = 0; s2 < STAGES - 1; ++s2)
      if (s2 < KT) issue(s2, s2);
  }

  double acc[C::FM][C::FN][2];
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int kt = 0; kt < KT; ++kt) {
    mbar_wait(full + kt % STAGES, uint32_t((kt / STAGES) & 1));
    __syncthreads();   // every warp is done with the slot refilled below (used at kt - 1)
    const int nk = kt + STAGES - 1;
    if (tid == 0 && nk < KT) issue(nk % STAGES, nk);
    const double* sA = reinterpret_cast<const double*>(base + (kt % STAGES) * X::SB);
    const double* sB = reinterpret_cast<const double*>(base + (kt % STAGES) * X::SB + X::AB);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[C::FM], bf[C::FN];
#pragma unroll
      for (int i = 0; i < C::FM; ++i) {
        const int m = wm0 + i * 8 + g;
        af[i] = TA ? sA[m * C::LDA + kk + t] : sA[(kk + t) * C::LDA + m];
      }
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int n = wn0 + j * 8 + g;
        bf[j] = TB ? sB[(kk + t) * C::LDB + n] : sB[n * C::LDB + kk + t];
      }
#pragma unroll
      for (int i = 0; i < C::FM; ++i)
#pragma unroll
        for (int j = 0; j < C::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }

  if (P.kslices == 1) {
    const double alpha = P.alpha, beta = P.beta;
    double* Cp = D.C;
    const int64_t ldc = D.ldc;
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int m = m0 + wm0 + i * 8 + g;
      if (m >= D.M) continue;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + j * 8 + 2 * t + e;
          if (n < D.N) {
            double* cp = Cp + m + int64_t(n) * ldc;
            double v = alpha * acc[i][j][e];
            if (beta != 0.0) v += beta * *cp;
            *cp = v;
          }
        }
      }
    }
  } else {
    const size_t tile = ((size_t(ks) * P.nbatch + b) * P.tiles_m + tm) * P.tiles_n + tn;
    double* W = P.ws + tile * (BM * BN);
#pragma unroll
    for (int i = 0; i < C::FM; ++i) {
      const int ml = wm0 + i * 8 + g;
#pragma unroll
      for (int j = 0; j < C::FN; ++j) {
        const int nl = wn0 + j * 8 + 2 * t;
        W[ml + nl * BM] = acc[i][j][0];
        W[ml + (nl + 1) * BM] = acc[i][j][1];
      }
    }
  }
}

// deterministic split-K reduction: slices summed in a fixed order, LANES threads
// per output element (grid: tiles x element chunks): lane q sums slices q,
// q + LANES, ... in index order, the LANES partial sums are combined by a fixed
// butterfly -- several lanes per element when there are many slices (the l x l
// Grams: ~100 slices of few tiles), so enough L2 requests are in flight
template <int BM, int BN, int LANES>
__global__ void __launch_bounds__(256) splitk_reduce(const __grid_constant__ GemmParams P) {
  if (P.gate && *P.gate != P.gate_val) return;
  const int tile_id = blockIdx.x;             // (b, tm, tn)
  const int tn = tile_id % P.tiles_n, tm = (tile_id / P.tiles_n) % P.tiles_m;
  const int b = tile_id / (P.tiles_n * P.tiles_m);
  const GemmDesc& D = P.d[b];
  const int e = (blockIdx.y * 256 + threadIdx.x) / LANES, q0 = threadIdx.x % LANES;
  if ((P.flags & kGemmLower) && tm * BM + BM <= tn * BN) return;
  const int ml = e % BM, nl = e / BM;
  const int m = tm * BM + ml, n = tn * BN + nl;
  const bool live = e < BM * BN && m < D.M && n < D.N;   // (whole lane groups agree)
  const size_t stride = size_t(P.nbatch) * P.tiles_m * P.tiles_n * (BM * BN);
  const double* src = P.ws + ((size_t(b) * P.tiles_m + tm) * P.tiles_n + tn) * (BM * BN) + e;
  double s = 0.0;
  if (live) {
    // loads issued 16 deep so the few threads of a small reduction keep enough
    // L2 requests in flight
    int k = q0;
    for (; k + 15 * LANES < P.kslices; k += 16 * LANES) {
      double v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = __ldcg(src + size_t(k + q * LANES) * stride);
#pragma unroll
      for (int q = 0; q < 16; ++q) s += v[q];
    }
    for (; k + 3 * LANES < P.kslices; k += 4 * LANES) {
      double v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = __ldcg(src + size_t(k + q * LANES) * stride);
#pragma unroll
      for (int q = 0; q < 4; ++q) s += v[q];
    }
    for (; k < P.kslices; k += LANES) s += __ldcg(src + size_t(k) * stride);
  }
#pragma unroll
  for (int o = 1; o < LANES; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (!live || q0 != 0) return;
  double* cp = D.C + m + int64_t(n) * D.ldc;
  double v = P.alpha * s;
  if (P.beta != 0.0) v += P.beta * *cp;
  *cp = v;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES>
struct Shape {
  static constexpr int bm = BM, bn = BN, bk = BK, wm = WM, wn = WN, st = STAGES;
};

// cuTensorMapEncodeTiled from the driver (no link-time dependency on libcuda)
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  });
  return fn;
}

}  // namespace

// 2-D map of a column-major rows x cols fp64 matrix (leading dimension ld) with
// box {box0 (contiguous), box1}; false if TMA cannot address it (dmma_tma.cuh)
bool encode_map(CUtensorMap* m, const double* ptr, int64_t rows, int64_t cols, int64_t ld,
                int box0, int box1) {
  auto enc = tma_encoder();
  if (!enc || rows < 1 || cols < 1) return false;
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld & 1) || ld < rows) return false;
  cuuint64_t dims[2] = {cuuint64_t(rows), cuuint64_t(cols)};
  cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
  cuuint32_t box[2] = {cuuint32_t(box0), cuuint32_t(box1)};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

namespace {

bool tma_disabled() {
  static const bool off = getenv("TTR_NO_TMA") != nullptr;   // A/B switch (diagnostics)
  return off;
}

#ifndef TTR_TMA_STAGES
#define TTR_TMA_STAGES 0   // 0: the shape's own stage count
#endif
template <class S>
constexpr int tma_stages() { return TTR_TMA_STAGES > 0 ? TTR_TMA_STAGES : S::st; }

template <class S, bool TA, bool TB>
int launch_cfg(Ctx& c, GemmParams& P, int maxM, int maxN, int maxK, cudaStream_t s) {
  using C = Cfg<S::bm, S::bn, S::bk, S::wm, S::wn, S::st, TA, TB>;
  constexpr int TS = tma_stages<S>();
  using X = TmaCfg<S::bm, S::bn, S::bk, S::wm, S::wn, TS, TA, TB>;
  auto kern = dgemm_kernel<S::bm, S::bn, S::bk, S::wm, S::wn, S::st, TA, TB>;
  auto tkern = dgemm_tma_kernel<S::bm, S::bn, S::bk, S::wm, S::wn, TS, TA, TB>;
  static std::atomic<bool> attr_set[64];
  static int resident[64] = {0};    // CTAs of this configuration per SM (cp.async kernel)
  static int tresident[64] = {0};   // ... (TMA kernel)
  int dev = c.device;
  std::unique_lock<std::mutex> init_lock(init_mutex(), std::defer_lock);
  if (!attr_set[dev & 63]) init_lock.lock();   // first calls may come from several threads
  if (!attr_set[dev & 63]) {
    TTR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(C::SMEM)));
    int nb = 1;
    TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, C::NT, C::SMEM));
    resident[dev & 63] = std::max(1, nb);
    TTR_CUDA(cudaFuncSetAttribute(tkern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(X::SMEM)));
    nb = 1;
    TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, tkern, C::NT, X::SMEM));
    tresident[dev & 63] = std::max(1, nb);
    attr_set[dev & 63] = true;
  }
  // TMA path when every entry's operands are addressable by a tensor map
  static thread_local TmaParams TP;
  bool use_tma = !tma_disabled() && P.nbatch <= kMaxTmaBatch;
  for (int b = 0; use_tma && b < P.nbatch; ++b) {
    const GemmDesc& D = P.d[b];
    use_tma = (TA ? encode_map(&TP.tm[2 * b], D.A, D.K, D.M, D.lda, C::LDA, S::bm)
                  : encode_map(&TP.tm[2 * b], D.A, D.M, D.K, D.lda, C::LDA, S::bk)) &&
              (TB ? encode_map(&TP.tm[2 * b + 1], D.B, D.N, D.K, D.ldb, C::LDB, S::bk)
                  : encode_map(&TP.tm[2 * b + 1], D.B, D.K, D.N, D.ldb, C::LDB, S::bn));
  }
  P.tiles_m = (maxM + S::bm - 1) / S::bm;
  P.tiles_n = (maxN + S::bn - 1) / S::bn;
  // split-K, wave-aware: pick the slice count whose grid fills the resident CTA
  // slots (SMs x CTAs per SM) best -- a grid of 1.13 waves runs at 57% -- with
  // a small penalty per slice for the extra partial traffic and reduction
  const long slots = long(c.sm_count) * (use_tma ? tresident[dev & 63] : resident[dev & 63]);
  // live tiles: a lower-triangle Gram skips the tiles above the diagonal
  long tiles = long(P.tiles_m) * P.tiles_n * P.nbatch;
  if (P.flags & kGemmLower) {
    long live = 0;
    for (int tm = 0; tm < P.tiles_m; ++tm)
      for (int tn = 0; tn < P.tiles_n; ++tn) live += (tm * S::bm + S::bm > tn * S::bn);
    tiles = live * P.nbatch;
  }
  const int ktiles = (maxK + S::bk - 1) / S::bk;
  int ksl = 1;
  if (tiles < 3 * slots) {
    // (a Gram has a handful of tiles and a long K: up to 256 slices so that its
    // grid fills the GPU)
    const int kmax = std::max(1, std::min((P.flags & kGemmLower) ? 256 : 64, ktiles / 4));
    if (tiles * kmax <= slots) {
      ksl = kmax;   // cannot fill one wave: as many slices as allowed (>= 4 k-tiles each)
    } else {
      double best = -1.0;
      for (int k = 1; k <= kmax; ++k) {
        const long ctas = tiles * k;
        if (ctas < slots && k < kmax) continue;   // at least one full wave
        const long waves = (ctas + slots - 1) / slots;
        const double eff = double(ctas) / double(waves * slots);
        const double score = eff - 0.004 * k;
        if (score > best + 1e-12) { best = score; ksl = k; }
      }
    }
  }
  const int kchunk_tiles = (ktiles + ksl - 1) / ksl;
  ksl = std::max(1, (ktiles + kchunk_tiles - 1) / std::max(1, kchunk_tiles));
  P.kslices = ksl;
  P.kchunk = kchunk_tiles * S::bk;
  if (ksl > 1) {
    const size_t need = size_t(ksl) * P.tiles_m * P.tiles_n * P.nbatch * S::bm * S::bn;
    if (c.gemm_ws.n < need) {
      if (c.capturing) {   // a workspace allocated inside a graph would die with it
        set_error("gemm workspace must be sized before graph capture");
        return TT_ERR_ARG;
      }
      TTR_TRY(dalloc(c.gemm_ws, need + need / 4, s));
    }
    P.ws = c.gemm_ws.p;
  } else {
    P.ws = nullptr;
  }
  dim3 grid(P.tiles_n, P.tiles_m, P.nbatch * ksl);
  if (grid.y > 65535 || grid.z > 65535) {
    set_error("gemm grid too large (%d x %d x %d)", grid.x, grid.y, grid.z);
    return TT_ERR_ARG;
  }
  if (use_tma) {
    TP.g = P;
    tkern<<<grid, C::NT, X::SMEM, s>>>(TP);
  } else {
    kern<<<grid, C::NT, C::SMEM, s>>>(P);
  }
  TTR_TRY(launched());
  if (ksl > 1) {
    const dim3 rg(P.tiles_n * P.tiles_m * P.nbatch, (S::bm * S::bn * (ksl >= 32 ? 4 : 1) + 255) / 256);
    if (ksl >= 32) splitk_reduce<S::bm, S::bn, 4><<<rg, 256, 0, s>>>(P);
    else splitk_reduce<S::bm, S::bn, 1><<<rg, 256, 0, s>>>(P);
    TTR_TRY(launched());
  }
  return TT_OK;
}

// tile shapes (DESIGN.md §Kernels / K2): BM, BN, BK, warps_m, warps_n, stages
using TallS = Shape<128, 48, 32, 4, 2, 2>;   // M >> N ~ l (phase-1 Z, Y_n, Q = Y R^-1)
using WideS = Shape<48, 128, 32, 2, 4, 2>;   // N >> M ~ l (carry M^(j) H(T), projection)
using SqS = Shape<64, 64, 32, 2, 2, 2>;      // general / split-K
using RowS = Shape<64, 48, 32, 4, 2, 3>;     // M = R = 64, N = l = 144 (phase-1 W, split-K)
using GramS = Shape<48, 48, 32, 2, 2, 2>;    // l x l Grams (split-K)
using SmallS = Shape<32, 32, 16, 2, 2, 3>;   // tiny problems
using WideK = Shape<48, 64, 32, 2, 2, 2>;    // short-K wide (carry: K = R = 64), more CTAs/SM

template <bool TA, bool TB>
int dispatch(Ctx& c, GemmParams& P, int maxM, int maxN, int maxK, cudaStream_t s) {
  // the shape that wastes least on ragged edges; ties go to the larger tile
  struct Cand { int bm, bn, id; };
  static constexpr Cand cands[] = {{128, 48, 0}, {48, 128, 1}, {64, 64, 2}, {64, 48, 3},
                                   {48, 48, 4}, {32, 32, 5}};
  auto waste = [&](int bm, int bn) {
    const double tm = double((maxM + bm - 1) / bm) * bm, tn = double((maxN + bn - 1) / bn) * bn;
    return (tm * tn) / (double(maxM) * maxN);
  };
  int best = 5;
  double bw = 1e30;
  for (const Cand& x : cands) {
    // big tiles only where the problem has at least one full tile in each dimension
    if (x.bm > 32 && (maxM < x.bm / 2 || maxN < x.bn / 2)) continue;
    const double wv = waste(x.bm, x.bn) * (1.0 - 1e-3 * (x.bm * x.bn) / 6144.0);
    if (wv < bw) { bw = wv; best = x.id; }
  }
  // short K (phase-1 Z: K = R = 64, four k-tiles): each CTA is mostly load
  // prologue and store epilogue, hidden only by other resident CTAs -- the
  // 64 x 48 tile (80 registers, 57 KB) fits 3 per SM against 2 for 128 x 48
  if (best == 0 && maxK <= 64 && maxM % 64 == 0) best = 3;
  if (best == 1 && maxK <= 64 && maxN % 64 == 0) best = 6;   // the same for wide ones
  switch (best) {
    case 0: return launch_cfg<TallS, TA, TB>(c, P, maxM, maxN, maxK, s);
    case 1: return launch_cfg<WideS, TA, TB>(c, P, maxM, maxN, maxK, s);
    case 2: return launch_cfg<SqS, TA, TB>(c, P, maxM, maxN, maxK, s);
    case 3: return launch_cfg<RowS, TA, TB>(c, P, maxM, maxN, maxK, s);
    case 4: return launch_cfg<GramS, TA, TB>(c, P, maxM, maxN, maxK, s);
    case 6: return launch_cfg<WideK, TA, TB>(c, P, maxM, maxN, maxK, s);
    default: return launch_cfg<SmallS, TA, TB>(c, P, maxM, maxN, maxK, s);
  }
}

}  // namespace

int gemm_impl(Ctx& c, bool ta, bool tb, const GemmDesc* d, int nbatch, double alpha, double beta,
         cudaStream_t s, const int* gate, int gate_val, unsigned flags) {
  int done = 0;
  while (done < nbatch) {
    const int nb = std::min(kMaxGemmBatch, nbatch - done);
    GemmParams P;
    int maxM = 0, maxN = 0, maxK = 0, live = 0;
    for (int i = 0; i < nb; ++i) {
      const GemmDesc& x = d[done + i];
      if (x.M <= 0 || x.N <= 0) continue;
      if (x.K <= 0) {
        // empty contraction (a rank holding no summands in the sharded path):
        // C = beta*C, only beta = 0 is used (C = 0)
        if (beta != 0.0 || gate) {
          set_error("gemm with K = 0 needs beta = 0 and no gate");
          return TT_ERR_ARG;
        }
        TTR_CUDA(cudaMemset2DAsync(x.C, size_t(x.ldc) * sizeof(double), 0,
                                   size_t(x.M) * sizeof(double), size_t(x.N), s));
        continue;
      }
      P.d[live++] = x;
      maxM = std::max(maxM, x.M);
      maxN = std::max(maxN, x.N);
      maxK = std::max(maxK, x.K);
    }
    done += nb;
    if (live == 0) continue;
    P.nbatch = live;
    P.flags = int(flags);
    P.vec = 1;
    for (int i = 0; i < live; ++i) {
      const GemmDesc& x = P.d[i];
      if ((reinterpret_cast<uintptr_t>(x.A) & 15) || (reinterpret_cast<uintptr_t>(x.B) & 15) ||
          (x.lda & 1) || (x.ldb & 1))
        P.vec = 0;
    }
    P.alpha = alpha;
    P.beta = beta;
    P.gate = gate;
    P.gate_val = gate_val;
    int r;
    if (!ta && !tb) r = dispatch<false, false>(c, P, maxM, maxN, maxK, s);
    else if (!ta && tb) r = dispatch<false, true>(c, P, maxM, maxN, maxK, s);
    else if (ta && !tb) r = dispatch<true, false>(c, P, maxM, maxN, maxK, s);
    else r = dispatch<true, true>(c, P, maxM, maxN, maxK, s);
    TTR_TRY(r);
  }
  return TT_OK;
}

}  // namespace ttr
