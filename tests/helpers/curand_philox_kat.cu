// Host-side known-answer generator: runs the CUDA toolkit's own
// curand_Philox4x32_10 (curand_philox4x32_x.h) on the CPU for (ctr,key) pairs
// read from stdin.  A library routine used as an independent pin for the
// oracle's Philox (tests/test_oracle_pins.py).  Not part of the product path.
#define QUALIFIERS static __forceinline__ __host__ __device__
#include <cstdio>
#include <cuda_runtime.h>
#include <curand_philox4x32_x.h>
int main() {
  unsigned c0, c1, c2, c3, k0, k1;
  while (std::scanf("%x %x %x %x %x %x", &c0, &c1, &c2, &c3, &k0, &k1) == 6) {
    uint4 c = make_uint4(c0, c1, c2, c3);
    uint2 k = make_uint2(k0, k1);
    uint4 o = curand_Philox4x32_10(c, k);
    std::printf("%08x %08x %08x %08x\n", o.x, o.y, o.z, o.w);
  }
  return 0;
}
