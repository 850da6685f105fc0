// DMMA.8x8x4 throughput per SM vs warps per SM and independent chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void kd(double* out, int iters) {
  double c[CH][2];
  for (int i = 0; i < CH; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < CH; ++i) s += c[i][0] + c[i][1];
  if (s == 123.0) out[0] = s;
}
template <int CH> void run(int warps, double* o) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2000; const int blocks = 148;
  kd<CH><<<blocks, 32 * warps>>>(o, 10);
  cudaEventRecord(e0); kd<CH><<<blocks, 32 * warps>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * CH * iters * warps * blocks;
  printf("warps/SM %2d chains %2d: %6.2f TF\n", warps, CH, fl / (ms * 1e-3) / 1e12);
}
int main() {
  double* o; cudaMalloc(&o, 8);
  for (int w : {1, 2, 4, 8, 16}) { run<1>(w, o); run<2>(w, o); run<4>(w, o); run<8>(w, o); run<16>(w, o); }
}
