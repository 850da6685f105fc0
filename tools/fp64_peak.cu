// FP64 roofline denominators for B200 (sm_100a), measured on the box:
//  * DMMA: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, 512 flop / warp instruction),
//    8 independent accumulators per warp, all SMs, best of 10 launches.
//  * DFMA: plain fp64 FMA pipe, same structure.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
// Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dmma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  double best_dmma = 0, best_dfma = 0;
  for (int warps : {4, 8, 16}) {
    const int blocks = sms * 2, threads = 32 * warps / 2;
    for (int rep = 0; rep < 10; ++rep) {
      cudaEventRecord(e0);
      dmma_loop<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = double(blocks) * (threads / 32) * iters * 8 * 512.0;
      if (rep) best_dmma = fmax(best_dmma, flops / (ms * 1e-3) / 1e12);
      cudaEventRecord(e0);
      dfma_loop<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double f2 = double(blocks) * threads * iters * 8 * 2.0;
      if (rep) best_dfma = fmax(best_dfma, f2 / (ms * 1e-3) / 1e12);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("{\"fp64_dmma_tflops\": %.3f, \"fp64_dfma_tflops\": %.3f, \"sms\": %d, "
         "\"clock_rate_khz\": %d, \"how\": \"best of 10 all-SM launches, 8 independent "
         "DMMA.8x8x4 (512 flop) or DFMA chains per warp\", \"cuda_error\": \"%s\"}\n",
         best_dmma, best_dfma, sms, clk, cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
