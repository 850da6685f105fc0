// Device helpers shared by the DMMA kernels fed by the Tensor Memory Accelerator
// (gemm.cu, fused.cu): the FP64 tensor-core MMA, mbarriers and 2-D TMA loads.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdint.h>

namespace ttr {

// C(8x8) += A(8x4) B(4x8), FP64 on the tensor pipe (SASS DMMA.8x8x4)
static __device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
static __device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
static __device__ __forceinline__ void mbarrier_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(bar)), "r"(count));
}
static __device__ __forceinline__ void mbarrier_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
static __device__ __forceinline__ void mbarrier_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
static __device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                              uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_addr(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// Host: 2-D tensor map of a column-major rows x cols fp64 matrix (leading
// dimension ld, box {box0 contiguous, box1}); false if TMA cannot address it
// (unaligned base, odd ld, driver entry point missing).  gemm.cu.
bool encode_map(CUtensorMap* m, const double* ptr, int64_t rows, int64_t cols, int64_t ld,
                int box0, int box1);

}  // namespace ttr
