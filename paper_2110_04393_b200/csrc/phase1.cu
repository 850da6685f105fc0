// Fused phase-1 step (Alg. 3 lines 4-5, inside Alg. 7 lines 3-5):
//
//   W_{n-1}^(j) = H(Z) H(G_n)^T,  V(Z) = V(Y_n^(j)) W_n^(j)
//              = sum_i (Y_i W_n) G_i^T      (Y_i = Y_n(:, i, :), G_i = G_n(:, i, :))
//
// for all summands j in one persistent kernel.  The two-GEMM form writes Z
// (C5: 604 MB per step) to HBM and reads it back, and its first GEMM has K = R
// = 64 (a tile spends most of its life in prologue and epilogue).  Here a CTA
// walks a contiguous run of (summand, i) items; for each item and each 16-wide
// chunk of the sketch rank e it forms Zc = Y_i W(:, chunk) (64 x 16, DMMA) in
// shared memory and immediately accumulates Zc G_i(:, chunk)^T into a 64 x 144
// register tile -- Z never leaves the SM.  W_n^(j) (R x l, 72 KB) stays in
// shared memory while the summand is unchanged; Y_i and the G chunks are
// double-buffered with cp.async, one barrier per chunk.  A CTA's run covers at
// most two summands, whose partial tiles go to a workspace and are summed per
// summand in CTA order by p1_reduce_kernel (deterministic).
#include "common.cuh"

namespace ttr {

namespace {

constexpr int kP1MaxS = 64;      // summands per launch
constexpr int MA = 64;           // rows a (R_{n-1}) padded
constexpr int KB = 64;           // contraction b (R_n) padded
constexpr int EC = 16;           // e chunk (sketch rank l_n)
constexpr int NC = 144;          // columns c (l_{n-1}) padded
constexpr int NCE = 144;         // e extent (l_n) padded
constexpr int LDY = MA + 4, LDW = KB + 4, LDG = NC + 4, LDZ = MA + 4;
constexpr int NT = 256;          // 8 warps: warp w owns rows 8w..8w+7
constexpr int SM_W = NCE * LDW, SM_Y = MA * LDY, SM_G = EC * LDG, SM_Z = EC * LDZ;
constexpr size_t SMEM = size_t(SM_W + 2 * SM_Y + 2 * SM_G + SM_Z) * sizeof(double);

struct P1Params {
  const double* Y[kP1MaxS];   // core n of summand j: R0 x I x R1 (a fastest)
  const double* W[kP1MaxS];   // W_n^(j): R1 x l1, ld ldw
  double* O[kP1MaxS];         // W_{n-1}^(j): R0 x l0, ld ldo
  int R0[kP1MaxS], R1[kP1MaxS];
  const double* G;            // sketch core n: l0 x I x l1 (c fastest)
  double* part;               // [grid][2][MA x NC] partial tiles (col-major, ld MA)
  int S, I, l0, l1, ldw, ldo, per, items;
};

__device__ __forceinline__ void cp16(double* smem, const double* gmem, int bytes) {
  unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit_() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all_() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(NT, 1) phase1_fused_kernel(const __grid_constant__ P1Params P) {
  extern __shared__ __align__(16) double sm[];
  double* sW = sm;                       // [e][b]
  double* sY = sW + SM_W;                // [2][b][a]
  double* sG = sY + 2 * SM_Y;            // [2][e_local][c]
  double* sZ = sG + 2 * SM_G;            // [e_local][a]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int nch = (P.l1 + EC - 1) / EC;
  const int it0 = blockIdx.x * P.per, it1 = min(P.items, it0 + P.per);
  if (it0 >= it1) return;
  const int j_first = it0 / P.I;

  auto load_W = [&](int j) {
    const double* Wj = P.W[j];
    const int R1 = P.R1[j];
    for (int v = tid; v < NCE * (KB / 2); v += NT) {
      const int b = 2 * (v % (KB / 2)), e = v / (KB / 2);
      const int bytes = (e < P.l1 && b < R1) ? 16 : 0;   // R1 even (host check)
      cp16(sW + e * LDW + b, bytes ? Wj + b + int64_t(e) * P.ldw : Wj, bytes);
    }
  };
  auto load_Y = [&](int item, int buf) {
    const int j = item / P.I, i = item % P.I;
    const double* Yj = P.Y[j];
    const int R0 = P.R0[j], R1 = P.R1[j];
    double* dst = sY + buf * SM_Y;
    for (int v = tid; v < KB * (MA / 2); v += NT) {
      const int a = 2 * (v % (MA / 2)), b = v / (MA / 2);
      const int bytes = (a < R0 && b < R1) ? 16 : 0;     // R0 even (host check)
      cp16(dst + b * LDY + a, bytes ? Yj + a + int64_t(R0) * (i + int64_t(P.I) * b) : Yj, bytes);
    }
  };
  auto load_G = [&](int item, int ec, int buf) {
    const int i = item % P.I;
    double* dst = sG + buf * SM_G;
    for (int v = tid; v < EC * (NC / 2); v += NT) {
      const int c = 2 * (v % (NC / 2)), el = v / (NC / 2);
      const int e = ec * EC + el;
      const int bytes = (c < P.l0 && e < P.l1) ? 16 : 0;  // l0 even (host check)
      cp16(dst + el * LDG + c, bytes ? P.G + c + int64_t(P.l0) * (i + int64_t(P.I) * e) : P.G,
           bytes);
    }
  };

  double acc[18][2];
#pragma unroll
  for (int cf = 0; cf < 18; ++cf) acc[cf][0] = acc[cf][1] = 0.0;
  auto flush = [&](int j) {
    const int slot = (j == j_first) ? 0 : 1;
    double* dst = P.part + (size_t(blockIdx.x) * 2 + slot) * (MA * NC);
#pragma unroll
    for (int cf = 0; cf < 18; ++cf) {
      const int a = 8 * warp + g, c = 8 * cf + 2 * t;
      dst[a + MA * c] = acc[cf][0];
      dst[a + MA * (c + 1)] = acc[cf][1];
      acc[cf][0] = acc[cf][1] = 0.0;
    }
  };

  const int s0 = it0 * nch, s1 = it1 * nch;
  int cur_j = j_first;
  load_W(cur_j);
  load_Y(it0, it0 & 1);
  load_G(it0, 0, s0 & 1);
  cp_async_commit_();
  for (int s = s0; s < s1; ++s) {
    const int item = s / nch, ec = s % nch;
    const int j = item / P.I;
    cp_async_wait_all_();
    __syncthreads();                     // step s landed; every warp done with step s-1
    if (j != cur_j) {                    // new summand: flush, then its W (synchronously)
      flush(cur_j);
      cur_j = j;
      load_W(j);
      cp_async_commit_();
      cp_async_wait_all_();
      __syncthreads();
    }
    if (s + 1 < s1) {                    // prefetch step s+1 into the other buffers
      const int item1 = (s + 1) / nch, ec1 = (s + 1) % nch;
      if (ec1 == 0) load_Y(item1, item1 & 1);
      load_G(item1, ec1, (s + 1) & 1);
    }
    cp_async_commit_();
    // Zc = Y_i W(:, chunk): warp w -> rows 8w..8w+7, 16 columns
    const double* Yb = sY + (item & 1) * SM_Y;
    const double* Gb = sG + (s & 1) * SM_G;
    double z0[2] = {0.0, 0.0}, z1[2] = {0.0, 0.0};
    const int kend = (P.R1[j] + 3) & ~3;
#pragma unroll 4
    for (int kk = 0; kk < kend; kk += 4) {
      const double a = Yb[(kk + t) * LDY + 8 * warp + g];
      const double b0 = sW[(ec * EC + g) * LDW + kk + t];
      const double b1 = sW[(ec * EC + 8 + g) * LDW + kk + t];
      dmma(z0[0], z0[1], a, b0);
      dmma(z1[0], z1[1], a, b1);
    }
    // C fragment (row g, cols 2t, 2t+1) -> sZ[e_local][a]
    sZ[(2 * t) * LDZ + 8 * warp + g] = z0[0];
    sZ[(2 * t + 1) * LDZ + 8 * warp + g] = z0[1];
    sZ[(8 + 2 * t) * LDZ + 8 * warp + g] = z1[0];
    sZ[(8 + 2 * t + 1) * LDZ + 8 * warp + g] = z1[1];
    __syncwarp();
    // acc += Zc G_i(:, chunk)^T
#pragma unroll
    for (int kk = 0; kk < EC; kk += 4) {
      const double a = sZ[(kk + t) * LDZ + 8 * warp + g];
#pragma unroll
      for (int cf = 0; cf < 18; ++cf) dmma(acc[cf][0], acc[cf][1], a, Gb[(kk + t) * LDG + 8 * cf + g]);
    }
    __syncwarp();
  }
  flush(cur_j);
}

// W_{n-1}^(j)(a, c) = sum over the CTAs whose run meets summand j, in CTA order
__global__ void p1_reduce_kernel(const __grid_constant__ P1Params P) {
  const int j = blockIdx.x;
  const int b0 = (j * P.I) / P.per, b1 = ((j + 1) * P.I - 1) / P.per;
  const int R0 = P.R0[j];
  for (int e = threadIdx.x; e < R0 * P.l0; e += blockDim.x) {
    const int a = e % R0, c = e / R0;
    double s = 0.0;
    for (int b = b0; b <= b1; ++b) {
      const int slot = (j == (b * P.per) / P.I) ? 0 : 1;
      s += P.part[(size_t(b) * 2 + slot) * (MA * NC) + a + MA * c];
    }
    P.O[j][a + int64_t(P.ldo) * c] = s;
  }
}

}  // namespace

// Returns TT_OK after launching, or 1 when the shapes are outside the fused
// kernel's envelope (the caller then runs the two GEMMs).
int phase1_fused_step(Ctx& c, int S, const double* const* Y, const int64_t* R0,
                      const int64_t* R1, int64_t I, const double* W, int64_t ldw,
                      const int64_t* woff, const double* G, int64_t l0, int64_t l1,
                      double* O, int64_t ldo, const int64_t* ooff, cudaStream_t s) {
  if (S < 1 || S > kP1MaxS || l0 > NC || l1 > NCE || (l0 & 1) || (ldw & 1) || I < 1)
    return 1;
  for (int j = 0; j < S; ++j)
    if (R0[j] > MA || R1[j] > KB || (R0[j] & 1) || (R1[j] & 1) ||
        (reinterpret_cast<uintptr_t>(Y[j]) & 15) ||
        (reinterpret_cast<uintptr_t>(W + woff[j]) & 15))
      return 1;
  if (reinterpret_cast<uintptr_t>(G) & 15) return 1;
  const int64_t items = int64_t(S) * I;
  const int grid = c.sm_count;
  const int64_t per = (items + grid - 1) / grid;
  if (per > I || items < 8 * int64_t(grid)) return 1;   // <= 2 summands per CTA; big enough
  P1Params P;
  for (int j = 0; j < S; ++j) {
    P.Y[j] = Y[j];
    P.W[j] = W + woff[j];
    P.O[j] = O + ooff[j];
    P.R0[j] = int(R0[j]);
    P.R1[j] = int(R1[j]);
  }
  P.G = G;
  P.S = S;
  P.I = int(I);
  P.l0 = int(l0);
  P.l1 = int(l1);
  P.ldw = int(ldw);
  P.ldo = int(ldo);
  P.per = int(per);
  P.items = int(items);
  const size_t need = size_t(grid) * 2 * MA * NC;
  if (c.p1_ws.n < need) TTR_TRY(dalloc(c.p1_ws, need, s));
  P.part = c.p1_ws.p;
  static bool attr[64] = {false};
  if (!attr[c.device & 63]) {
    TTR_CUDA(cudaFuncSetAttribute(phase1_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(SMEM)));
    attr[c.device & 63] = true;
  }
  phase1_fused_kernel<<<grid, NT, SMEM, s>>>(P);
  TTR_TRY(launched());
  p1_reduce_kernel<<<S, 256, 0, s>>>(P);
  return launched();
}

}  // namespace ttr
