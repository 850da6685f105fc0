// Golden-vector writer for the oracle's Philox4x32-10 (tests/test_oracle_philox.py).
// It evaluates NVIDIA's own cuRAND implementation, curand_Philox4x32_10()
// (/usr/local/cuda/include/curand_philox4x32_x.h:171-191), on the HOST, so the
// expected words come from neither the oracle nor this repo's CUDA kernels.
// Build + run (no GPU needed):
//   nvcc -o /tmp/philox_kat tests/golden/philox_kat.cu && /tmp/philox_kat > tests/golden/philox_kat.txt
#define QUALIFIERS static inline __host__ __device__
#include <cstdio>
#include <cstdint>
#include <vector_types.h>
#include <curand_philox4x32_x.h>

int main() {
  const unsigned long long seeds[] = {0ull, 1ull, 0x123456789abcdefull, 0xffffffffffffffffull};
  const unsigned pairs[] = {0u, 1u, 2u, 12345u, 0xfffffffeu};
  const unsigned modes[] = {1u, 2u, 50u};
  const unsigned tags[] = {0u, 3u};
  printf("# seed k n tag x0 x1 x2 x3  (ctr = (k_lo, k_hi, n, tag), key = (seed_lo, seed_hi))\n");
  for (unsigned long long s : seeds)
    for (unsigned k : pairs)
      for (unsigned n : modes)
        for (unsigned t : tags) {
          uint4 c; c.x = k; c.y = 0u; c.z = n; c.w = t;
          uint2 key; key.x = (unsigned)(s & 0xffffffffu); key.y = (unsigned)(s >> 32);
          uint4 r = curand_Philox4x32_10(c, key);
          printf("%llu %u %u %u %u %u %u %u\n", s, k, n, t, r.x, r.y, r.z, r.w);
        }
  // one counter with a non-zero high word of k
  {
    uint4 c; c.x = 7u; c.y = 3u; c.z = 9u; c.w = 0u;
    uint2 key; key.x = 42u; key.y = 0u;
    uint4 r = curand_Philox4x32_10(c, key);
    printf("%llu %llu %u %u %u %u %u %u\n", 42ull, (3ull << 32) | 7ull, 9u, 0u, r.x, r.y, r.z, r.w);
  }
  return 0;
}
