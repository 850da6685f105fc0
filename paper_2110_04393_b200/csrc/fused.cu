// Fused projection-and-carry of the Alg. 7 sweep (north-star item 4; SURVEY §8a
// rows a5-a6): for one sweep step n < N-1, in ONE cooperative launch,
//
//   line 11:  [M^(1) ... M^(s)] = Q_n^T V(X_n)            (l x sum_j R_n^(j))
//   line 13:  H(X_{n+1})[:, block j] = M^(j) H(Y^(j)_{n+1})  for every summand j
//
// Phase A: the projection's output tiles (48 x 128), split along K = l_{n-1} I_n
//          into `ksl` slices, one slice partial per work item, written to a
//          workspace (L2-resident);
// grid barrier;
// Phase B: M = sum of the slice partials in slice order (deterministic, the
//          same order as the unfused split-K reduction), written once;
// grid barrier;
// Phase C: the carry tiles (48 x 128, K = R_n^(j)) of every summand.
//
// Every tile of A and C is an FP64 tensor-core (DMMA m8n8k4) tile fed by TMA:
// one elected thread issues the 2-D tensor copies of each k-step into a
// 4-stage ring tracked by mbarriers whose phase runs on across all the tiles a
// persistent CTA processes.  Versus the unfused path (projection GEMM,
// split-K reduce kernel, batched carry GEMM) this removes two launches, their
// tail/ramp gaps and the carry's per-CTA load prologue (the ring keeps
// streaming across carry tiles).
#include <cooperative_groups.h>
#include <stdlib.h>

#include "common.cuh"
#include "dmma_tma.cuh"

namespace cg = cooperative_groups;

namespace ttr {

namespace {

constexpr int kBM = 48, kBN = 128, kBK = 32, kWM = 2, kWN = 4, kST = 2;
constexpr int kConsumers = kWM * kWN;                  // MMA warps
constexpr int kThreads = (kConsumers + 1) * 32;         // + one TMA producer warp
constexpr int kTM = kBM / kWM, kTN = kBN / kWN;        // warp tile 24 x 32
constexpr int kFM = kTM / 8, kFN = kTN / 8;             // 3 x 4 fragments
constexpr int kLdaT = kBK + 4;                          // A^T tile [m][k] (projection)
constexpr int kLdaN = kBM + 4;                          // A tile [k][m] (carry)
constexpr int kLdb = kBK + 4;                           // B tile [n][k]
constexpr int kAEl = (kBM * kLdaT > kBK * kLdaN) ? kBM * kLdaT : kBK * kLdaN;
constexpr int kBEl = kBN * kLdb;
constexpr int kAB = ((kAEl * 8 + 127) / 128) * 128;
constexpr int kBB = ((kBEl * 8 + 127) / 128) * 128;
constexpr int kSB = kAB + kBB;
constexpr size_t kSmem = size_t(kST) * kSB + 128 + 16 * kST;
constexpr int kMaxPC = 32;

struct PCParams {
  CUtensorMap tQ;              // Q_n: m x l (column-major), read transposed
  CUtensorMap tX;              // V(X_n): m x sumR
  CUtensorMap tM;              // M: l x sumR
  CUtensorMap tY[kMaxPC];      // H(Y^(j)_{n+1}): R_j x N_j
  double* M;                   // l x sumR (ld l)
  double* ws;                  // ksl x tiles_pm x tiles_pn x (48 x 128) partials
  double* X1;                  // H(X_{n+1}) blocks
  int64_t xoff[kMaxPC];        // first element of summand j's block in X1 (ld l)
  int moff[kMaxPC];            // first column of M^(j)
  int Rj[kMaxPC], Nj[kMaxPC];  // K and N of carry j
  int ctile0[kMaxPC + 1];      // prefix sums of the carry tiles per summand
  int l, sumR, S;
  int ksl, kchunk;             // projection split: slices, k-tiles per slice
  int KT_total;                // k-tiles of the projection
  int tiles_pm, tiles_pn;      // projection output tiles
};

struct Ring {
  unsigned char* base;
  uint64_t* full;    // TMA landed (expect-tx), one per slot
  uint64_t* empty;   // every MMA warp is done with the slot (count kConsumers)
  uint32_t it;       // ring position (k-steps of this CTA so far), same in every thread
};

static __device__ __forceinline__ void mbarrier_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(bar)) : "memory");
}

// A phase of 48 x 128 output tiles processed by a persistent CTA: work items
// w = blockIdx.x, blockIdx.x + gridDim.x, ...; item w needs nkt(w) k-steps whose
// operand boxes are coords(w, kt, &a0, &a1, &b0, &b1, &bj) (B map mBs + bj).
// Warp-specialised: the producer warp (one elected lane) streams the k-steps of
// ALL the CTA's items through the kST-slot ring, waiting only for a slot to be
// released (`empty`), so the next item's operands arrive while the current one
// is finishing; the kConsumers MMA warps wait for `full`, multiply, and release
// the slot -- no CTA-wide barrier per k-step.  epi(w, acc, ...) stores an item.
// TA: A is read as a K x M matrix (the projection's Q); else M x K.
template <bool TA, class NKT, class COORDS, class EPI>
__device__ __forceinline__ void run_phase(Ring& R, const CUtensorMap* mA,
                                          const CUtensorMap* mBs, int nitems,
                                          NKT nkt, COORDS coords, EPI epi) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr uint32_t tx = uint32_t((TA ? kBM * kLdaT : kBK * kLdaN) + kBEl) * 8;
  if (warp == kConsumers) {   // ---- producer
    for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
      const int KT = nkt(w);
      for (int kt = 0; kt < KT; ++kt) {
        const uint32_t pos = R.it++;
        if (lane == 0) {
          const int slot = int(pos % kST);
          if (pos >= uint32_t(kST)) mbarrier_wait(R.empty + slot, ((pos / kST) - 1) & 1);
          unsigned char* sA = R.base + slot * kSB;
          int a0, a1, b0, b1, bj;
          coords(w, kt, a0, a1, b0, b1, bj);
          mbarrier_expect_tx(R.full + slot, tx);
          tma_2d(sA, mA, a0, a1, R.full + slot);
          tma_2d(sA + kAB, mBs + bj, b0, b1, R.full + slot);
        }
      }
    }
    return;
  }
  // ---- MMA warps
  const int g = lane >> 2, t = lane & 3;
  const int wm0 = (warp % kWM) * kTM, wn0 = (warp / kWM) * kTN;
  double acc[kFM][kFN][2];
  for (int w = blockIdx.x; w < nitems; w += gridDim.x) {
#pragma unroll
    for (int i = 0; i < kFM; ++i)
#pragma unroll
      for (int j = 0; j < kFN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const int KT = nkt(w);
    for (int kt = 0; kt < KT; ++kt) {
      const uint32_t pos = R.it++;
      const int slot = int(pos % kST);
      mbarrier_wait(R.full + slot, (pos / kST) & 1);
      const double* sA = reinterpret_cast<const double*>(R.base + slot * kSB);
      const double* sB = reinterpret_cast<const double*>(R.base + slot * kSB + kAB);
#pragma unroll
      for (int kk = 0; kk < kBK; kk += 4) {
        double af[kFM], bf[kFN];
#pragma unroll
        for (int i = 0; i < kFM; ++i) {
          const int m = wm0 + i * 8 + g;
          af[i] = TA ? sA[m * kLdaT + kk + t] : sA[(kk + t) * kLdaN + m];
        }
#pragma unroll
        for (int j = 0; j < kFN; ++j) bf[j] = sB[(wn0 + j * 8 + g) * kLdb + kk + t];
#pragma unroll
        for (int i = 0; i < kFM; ++i)
#pragma unroll
          for (int j = 0; j < kFN; ++j) dmma_884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
      __syncwarp();
      if (lane == 0) mbarrier_arrive(R.empty + slot);
    }
    epi(w, acc, wm0, wn0, g, t);
  }
}

__global__ void __launch_bounds__(kThreads)
    proj_carry_kernel(const __grid_constant__ PCParams P) {
  extern __shared__ __align__(128) unsigned char raw[];
  Ring R;
  R.base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 127) &
                                            ~uintptr_t(127));
  R.full = reinterpret_cast<uint64_t*>(R.base + kST * kSB);
  R.empty = R.full + kST;
  R.it = 0;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < kST; ++s) {
      mbarrier_init(R.full + s, 1);
      mbarrier_init(R.empty + s, kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  cg::grid_group grid = cg::this_grid();

  // ---- phase A: projection slice partials, item w = (slice ks, tile tm, tn)
  const int ptiles = P.tiles_pm * P.tiles_pn;
  {
    run_phase<true>(
        R, &P.tQ, &P.tX, ptiles * P.ksl,
        [&](int w) { return max(0, min(P.kchunk, P.KT_total - (w / ptiles) * P.kchunk)); },
        [&](int w, int kt, int& a0, int& a1, int& b0, int& b1, int& bj) {
          const int tl = w % ptiles, k0 = ((w / ptiles) * P.kchunk + kt) * kBK;
          a0 = k0;
          a1 = (tl / P.tiles_pn) * kBM;
          b0 = k0;
          b1 = (tl % P.tiles_pn) * kBN;
          bj = 0;
        },
        [&](int w, double (&acc)[kFM][kFN][2], int wm0, int wn0, int g, int t) {
          double* W = P.ws + size_t(w) * (kBM * kBN);   // [ks][tm][tn], column-major 48 x 128
#pragma unroll
          for (int i = 0; i < kFM; ++i)
#pragma unroll
            for (int j = 0; j < kFN; ++j) {
              const int ml = wm0 + i * 8 + g, nl = wn0 + j * 8 + 2 * t;
              W[ml + nl * kBM] = acc[i][j][0];
              W[ml + (nl + 1) * kBM] = acc[i][j][1];
            }
        });
  }
  grid.sync();
  // ---- phase B: M = sum_ks partial_ks (slice order, deterministic)
  {
    const size_t tile_el = size_t(kBM) * kBN;
    const size_t stride = size_t(ptiles) * tile_el;
    const size_t total = stride;   // elements of one slice
    for (size_t e = size_t(blockIdx.x) * kThreads + tid; e < total;
         e += size_t(gridDim.x) * kThreads) {
      const size_t tl = e / tile_el, el = e % tile_el;
      const int tm = int(tl / P.tiles_pn), tn = int(tl % P.tiles_pn);
      const int r = tm * kBM + int(el % kBM), c = tn * kBN + int(el / kBM);
      if (r >= P.l || c >= P.sumR) continue;
      const double* src = P.ws + e;
      double s = 0.0;
      int k = 0;
      for (; k + 4 <= P.ksl; k += 4) {
        double v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) v[q] = __ldcg(src + size_t(k + q) * stride);
#pragma unroll
        for (int q = 0; q < 4; ++q) s += v[q];
      }
      for (; k < P.ksl; ++k) s += __ldcg(src + size_t(k) * stride);
      P.M[r + size_t(c) * P.l] = s;
    }
  }
  // M is read back through TMA (the async proxy) in phase C
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
  grid.sync();
  // ---- phase C: carries H(X_{n+1})_j = M^(j) H(Y^(j)_{n+1}), item w = (summand j, tm, tn)
  const int tiles_cm = (P.l + kBM - 1) / kBM;
  auto summand = [&](int w) {
    int j = 0;
    while (P.ctile0[j + 1] <= w) ++j;
    return j;
  };
  {
    run_phase<false>(
        R, &P.tM, P.tY, P.ctile0[P.S],
        [&](int w) { return (P.Rj[summand(w)] + kBK - 1) / kBK; },
        [&](int w, int kt, int& a0, int& a1, int& b0, int& b1, int& bj) {
          const int j = summand(w), tl = w - P.ctile0[j];
          a0 = (tl % tiles_cm) * kBM;
          a1 = P.moff[j] + kt * kBK;
          b0 = kt * kBK;
          b1 = (tl / tiles_cm) * kBN;
          bj = j;
        },
        [&](int w, double (&acc)[kFM][kFN][2], int wm0, int wn0, int g, int t) {
          const int j = summand(w), tl = w - P.ctile0[j];
          const int tm = tl % tiles_cm, tn = tl / tiles_cm;
          double* Cp = P.X1 + P.xoff[j];
#pragma unroll
          for (int i = 0; i < kFM; ++i) {
            const int m = tm * kBM + wm0 + i * 8 + g;
            if (m >= P.l) continue;
#pragma unroll
            for (int jj = 0; jj < kFN; ++jj)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int n = tn * kBN + wn0 + jj * 8 + 2 * t + e;
                if (n < P.Nj[j]) Cp[m + int64_t(n) * P.l] = acc[i][jj][e];
              }
          }
        });
  }
}

}  // namespace

bool proj_carry_enabled() {
  static const bool off = getenv("TTR_NO_FUSE") != nullptr || getenv("TTR_NO_TMA") != nullptr;
  return !off;
}

// Returns TT_OK after launching, or 1 when the fused kernel does not apply (the
// caller then runs the unfused GEMMs); errors as usual.
int proj_carry(Ctx& c, int64_t m, int l, int sumR, const double* Q, const double* Xn, double* M,
               int S, const double* const* Y1, const int64_t* Rj, const int64_t* Nj,
               const int64_t* moff, double* X1, const int64_t* xoff, cudaStream_t s) {
  if (!proj_carry_enabled() || S < 1 || S > kMaxPC || l < 1 || sumR < 1 || m < 1) return 1;
  static thread_local PCParams P;
  if (!encode_map(&P.tQ, Q, m, l, m, kLdaT, kBM)) return 1;
  if (!encode_map(&P.tX, Xn, m, sumR, m, kLdb, kBN)) return 1;
  if (!encode_map(&P.tM, M, l, sumR, l, kLdaN, kBK)) return 1;
  int tiles = 0;
  const int tiles_cm = (l + kBM - 1) / kBM;
  P.ctile0[0] = 0;
  for (int j = 0; j < S; ++j) {
    if (Rj[j] < 1 || Nj[j] < 1) return 1;
    if (!encode_map(&P.tY[j], Y1[j], Rj[j], Nj[j], Rj[j], kLdb, kBN)) return 1;
    P.Rj[j] = int(Rj[j]);
    P.Nj[j] = int(Nj[j]);
    P.moff[j] = int(moff[j]);
    P.xoff[j] = xoff[j];
    tiles += tiles_cm * int((Nj[j] + kBN - 1) / kBN);
    P.ctile0[j + 1] = tiles;
  }
  static std::atomic<bool> attr[64];
  static int resident[64];
  {
    std::unique_lock<std::mutex> lk(init_mutex(), std::defer_lock);
    if (!attr[c.device & 63]) lk.lock();
    if (!attr[c.device & 63]) {
      TTR_CUDA(cudaFuncSetAttribute(proj_carry_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    int(kSmem)));
      int nb = 0;
      TTR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, proj_carry_kernel, kThreads,
                                                             kSmem));
      resident[c.device & 63] = nb;
      attr[c.device & 63] = true;
    }
  }
  const int grid = grid_sms(c) * resident[c.device & 63];
  if (grid < 1) return 1;
  P.M = M;
  P.X1 = X1;
  P.l = l;
  P.sumR = sumR;
  P.S = S;
  P.tiles_pm = (l + kBM - 1) / kBM;
  P.tiles_pn = (sumR + kBN - 1) / kBN;
  P.KT_total = int((m + kBK - 1) / kBK);
  // slices: the item count that fills the grid's waves best (a grid of 1.13
  // waves runs at 57%), at least 8 k-steps per item
  const int ptiles = P.tiles_pm * P.tiles_pn;
  int ksl = 1;
  {
    double best = -1.0;
    const int kmax = std::max(1, std::min(256, P.KT_total / 8));
    for (int k = 1; k <= kmax; ++k) {
      const long items = long(ptiles) * k, waves = (items + grid - 1) / grid;
      const double eff = double(items) / double(waves * grid) - 0.002 * k;
      if (eff > best + 1e-12) { best = eff; ksl = k; }
    }
  }
  P.kchunk = (P.KT_total + ksl - 1) / ksl;
  P.ksl = (P.KT_total + P.kchunk - 1) / P.kchunk;
  const size_t need = size_t(P.ksl) * ptiles * kBM * kBN;
  if (c.gemm_ws.n < need) {
    if (c.capturing) return 1;   // no workspace growth inside a graph: unfused path
    TTR_TRY(dalloc(c.gemm_ws, need + need / 4, s));
  }
  P.ws = c.gemm_ws.p;
  void* args[] = {&P};
  TTR_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<const void*>(proj_carry_kernel),
                                       dim3(grid), dim3(kThreads), args, kSmem, s));
  return launched();
}

}  // namespace ttr
