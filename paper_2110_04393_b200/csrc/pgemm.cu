// Persistent, warp-specialised batched GEMM for SHORT-K products (K <= a few
// hundred): C_j = A_j B_j for every batch entry j, column-major, no transposes.
// Used for Alg. 3 line 4 of phase 1, V(Z_n) = V(Y_n) W_n for every
// summand (K = R_n = 64 on config 5: four k-steps per 128 x 48 tile), where a
// grid of independent CTAs spends most of each CTA in its load prologue and
// store epilogue.  Here one CTA per SM slot walks its tiles (j, tm, tn) in a
// fixed order; a TMA producer warp streams the k-steps of ALL its tiles through a
// 4-slot mbarrier ring (full: expect-tx, empty: one arrive per MMA warp), so the
// next tile's operands arrive while the MMA warps finish the current tile and
// store it.  Same DMMA fragments, k order and fp64 accumulation as
// dgemm_kernel (gemm.cu); results are bit-identical to it.
#include <stdlib.h>

#include "common.cuh"
#include "dmma_tma.cuh"

namespace ttr {

namespace {

#ifndef TTR_PG_STAGES
#define TTR_PG_STAGES 2
#endif
#ifndef TTR_PG_BK
#define TTR_PG_BK 32
#endif
constexpr int pBM = 128, pBN = 48, pBK = TTR_PG_BK, pWM = 4, pWN = 2, pST = TTR_PG_STAGES;
constexpr int pConsumers = pWM * pWN;
constexpr int pThreads = (pConsumers + 1) * 32;
constexpr int pTM = pBM / pWM, pTN = pBN / pWN;      // warp tile 32 x 24
constexpr int pFM = pTM / 8, pFN = pTN / 8;           // 4 x 3 fragments
constexpr int pLda = pBM + 4;                         // A tile [k][m]
constexpr int pLdb = pBK + 4;                         // B tile [n][k]
constexpr int pAEl = pBK * pLda, pBEl = pBN * pLdb;
constexpr int pAB = ((pAEl * 8 + 127) / 128) * 128;
constexpr int pBB = ((pBEl * 8 + 127) / 128) * 128;
constexpr int pSB = pAB + pBB;
constexpr size_t pSmem = size_t(pST) * pSB + 128 + 16 * pST;
constexpr int pMaxB = 32;

struct PGParams {
  CUtensorMap tA[pMaxB];   // A_j: M_j x K_j
  CUtensorMap tB[pMaxB];   // B_j: K_j x N_j
  double* C[pMaxB];
  int64_t ldc[pMaxB];
  int M[pMaxB], N[pMaxB], K[pMaxB];
  int tile0[pMaxB + 1];    // prefix sums of the tiles per entry
  int nb;
};

__device__ __forceinline__ void pg_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ int pg_entry(const PGParams& P, int w) {
  int j = 0;
  while (P.tile0[j + 1] <= w) ++j;
  return j;
}

__global__ void __launch_bounds__(pThreads) pgemm_kernel(const __grid_constant__ PGParams P) {
  extern __shared__ __align__(128) unsigned char raw[];
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + pST * pSB);
  uint64_t* empty = full + pST;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < pST; ++s) {
      mbarrier_init(full + s, 1);
      mbarrier_init(empty + s, pConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int nitems = P.tile0[P.nb];
  constexpr uint32_t tx = uint32_t(pAEl + pBEl) * 8;
  uint32_t pos = 0;   // ring position (k-steps of this CTA so far)
  if (warp == pConsumers) {   // ---- producer (all lanes walk, lane 0 issues)
    for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
      const int j = pg_entry(P, w), tl = w - P.tile0[j];
      const int tiles_n = (P.N[j] + pBN - 1) / pBN;   // n fastest: the A block is reused from L2
      const int m0 = (tl / tiles_n) * pBM, n0 = (tl % tiles_n) * pBN;
      const int KT = (P.K[j] + pBK - 1) / pBK;
      for (int kt = 0; kt < KT; ++kt, ++pos) {
        if (lane == 0) {
          const int slot = int(pos % pST);
          if (pos >= uint32_t(pST)) mbarrier_wait(empty + slot, ((pos / pST) - 1) & 1);
          unsigned char* sA = base + slot * pSB;
          mbarrier_expect_tx(full + slot, tx);
          tma_2d(sA, &P.tA[j], m0, kt * pBK, full + slot);
          tma_2d(sA + pAB, &P.tB[j], kt * pBK, n0, full + slot);
        }
      }
    }
    return;
  }
  // ---- MMA warps
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % pWM) * pTM, wn0 = (warp / pWM) * pTN;
  for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
    const int j = pg_entry(P, w), tl = w - P.tile0[j];
    const int tiles_n = (P.N[j] + pBN - 1) / pBN;
    const int m0 = (tl / tiles_n) * pBM, n0 = (tl % tiles_n) * pBN;
    const int KT = (P.K[j] + pBK - 1) / pBK;
    double acc[pFM][pFN][2];
#pragma unroll
    for (int i = 0; i < pFM; ++i)
#pragma unroll
      for (int jj = 0; jj < pFN; ++jj) acc[i][jj][0] = acc[i][jj][1] = 0.0;
    for (int kt = 0; kt < KT; ++kt, ++pos) {
      const int slot = int(pos % pST);
      mbarrier_wait(full + slot, (pos / pST) & 1);
      const double* sA = reinterpret_cast<const double*>(base + slot * pSB);
      const double* sB = reinterpret_cast<const double*>(base + slot * pSB + pAB);
#pragma unroll
      for (int kk = 0; kk < pBK; kk += 4) {
        double af[pFM], bf[pFN];
#pragma unroll
        for (int i = 0; i < pFM; ++i) af[i] = sA[(kk + t) * pLda + wm0 + i * 8 + g];
#pragma unroll
        for (int jj = 0; jj < pFN; ++jj) bf[jj] = sB[(wn0 + jj * 8 + g) * pLdb + kk + t];
#pragma unroll
        for (int i = 0; i < pFM; ++i)
#pragma unroll
          for (int jj = 0; jj < pFN; ++jj) dmma_884(acc[i][jj][0], acc[i][jj][1], af[i], bf[jj]);
      }
      __syncwarp();
      if (lane == 0) pg_arrive(empty + slot);
    }
    double* Cp = P.C[j];
    const int64_t ldc = P.ldc[j];
#pragma unroll
    for (int i = 0; i < pFM; ++i) {
      const int m = m0 + wm0 + i * 8 + g;
      if (m >= P.M[j]) continue;
#pragma unroll
      for (int jj = 0; jj < pFN; ++jj)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = n0 + wn0 + jj * 8 + 2 * t + e;
          if (n < P.N[j]) Cp[m + int64_t(n) * ldc] = acc[i][jj][e];
        }
    }
  }
}

}  // namespace

// C_j = A_j B_j (column-major, beta = 0) for nb <= 32 entries with short K.
// Returns 1 (nothing launched) when it does not apply (TMA cannot address an
// operand, too many entries, TTR_NO_PGEMM set); the caller then uses gemm().
int pgemm(Ctx& c, const GemmDesc* d, int nb, cudaStream_t s) {
  static const bool off = getenv("TTR_NO_PGEMM") != nullptr || getenv("TTR_NO_TMA") != nullptr;
  if (off || nb < 1 || nb > pMaxB) return 1;
  static thread_local PGParams P;
  int tiles = 0;
  P.tile0[0] = 0;
  for (int j = 0; j < nb; ++j) {
    const GemmDesc& x = d[j];
    if (x.M < 1 || x.N < 1 || x.K < 1 || x.K > 1024) return 1;
    if (!encode_map(&P.tA[j], x.A, x.M, x.K, x.lda, pLda, pBK)) return 1;
    if (!encode_map(&P.tB[j], x.B, x.K, x.N, x.ldb, pLdb, pBN)) return 1;
    P.C[j] = x.C;
    P.ldc[j] = x.ldc;
    P.M[j] = x.M;
    P.N[j] = x.N;
    P.K[j] = x.K;
    tiles += ((x.M + pBM - 1) / pBM) * ((x.N + pBN - 1) / pBN);
    P.tile0[j + 1] = tiles;
  }
  P.nb = nb;
  static std::atomic<bool> attr[64];
  static int resident[64];
  {
    std::unique_lock<std::mutex> lk(init_mutex(), std::defer_lock);
    if (!attr[c.device & 63]) lk.lock();
    if (!attr[c.device & 63]) {
      TTR_CUDA(cudaFuncSetAttribute(pgemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(pSmem)));
      int r = 0;
      TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, pgemm_kernel, pThreads, pSmem));
      resident[c.device & 63] = r;
      attr[c.device & 63] = true;
    }
  }
  const int grid = std::min(tiles, grid_sms(c) * std::max(1, resident[c.device & 63]));
  if (grid < 1) return 1;
  pgemm_kernel<<<grid, pThreads, pSmem, s>>>(P);
  return launched();
}

}  // namespace ttr
