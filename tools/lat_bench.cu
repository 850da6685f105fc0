// Latency microbenchmark (single warp): dependent chains of fp64 ops, shuffles,
// rsqrt, division, smem round trips, __syncwarp.  cycles per chain step.
#include <cstdio>
#include <cuda_runtime.h>
#define N 1024
__global__ void k(double* out, long long* cyc, double seed) {
  __shared__ double sm[64];
  double x = seed + threadIdx.x * 1e-3, y = 1.0000001;
  long long t0, t1;
  int lane = threadIdx.x;
  sm[lane] = x; __syncwarp();
  // 0: DFMA chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, y, 1e-9);
  t1 = clock64(); cyc[0] = (t1 - t0);
  // 1: DMUL chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = x * y;
  t1 = clock64(); cyc[1] = (t1 - t0);
  // 2: SHFL (double) chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31) * y;
  t1 = clock64(); cyc[2] = (t1 - t0);
  // 3: rsqrt chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = rsqrt(x + 1.0);
  t1 = clock64(); cyc[3] = (t1 - t0);
  // 4: division chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 2.0);
  t1 = clock64(); cyc[4] = (t1 - t0);
  // 5: sqrt chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x + 2.0);
  t1 = clock64(); cyc[5] = (t1 - t0);
  // 6: STS -> syncwarp -> LDS (other lane) chain
  t0 = clock64();
  for (int i = 0; i < N; ++i) { sm[lane] = x; __syncwarp(); x = sm[(lane + 1) & 31] * y; __syncwarp(); }
  t1 = clock64(); cyc[6] = (t1 - t0);
  // 7: float fma chain
  float f = float(x);
  t0 = clock64();
  for (int i = 0; i < N; ++i) f = fmaf(f, 1.0000001f, 1e-9f);
  t1 = clock64(); cyc[7] = (t1 - t0);
  // 8: __syncthreads alone (1 warp)
  t0 = clock64();
  for (int i = 0; i < N; ++i) { __syncthreads(); x += 1e-300; }
  t1 = clock64(); cyc[8] = (t1 - t0);
  out[lane] = x + f;
}
__global__ void kbar(long long* cyc) {   // __syncthreads with 16 warps
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) { __syncthreads(); x = x * 1.0000001; }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = t1 - t0;
  if (x == 0.123) cyc[10] = 1;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 16 * 8);
  k<<<1, 32>>>(o, c, 0.5); kbar<<<1, 512>>>(c); cudaDeviceSynchronize();
  long long h[16]; cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  const char* nm[] = {"dfma", "dmul", "shfl.f64+dmul", "rsqrt(f64)+dadd", "div(f64)+dadd", "sqrt(f64)+dadd",
                      "sts+syncwarp+lds+dmul", "ffma", "syncthreads(1 warp)", "syncthreads(16 warps)+dmul"};
  for (int i = 0; i < 10; ++i) printf("%-28s %7.1f cycles/step\n", nm[i], double(h[i]) / N);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
