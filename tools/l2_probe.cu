// L2 -> SM read-throughput probe (measurement tool, not part of the library):
// the access pattern of K3d (csr_accumulate_kernel) without its arithmetic —
// every warp gathers whole 1 KB rows (32 lanes x 2 x 16 B, the κ slices of
// k = 512 bf16) at hashed row indices of an L2-resident panel, many rows in
// flight per warp.  The measured bytes/s is the denominator of K3d's L2 view
// in bench.py (DESIGN.md §7 K3).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC \
//        tools/l2_probe.cu -o tools/libl2probe.so
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// rows_per_warp gathers per warp; U rows in flight per lane group
template <int U>
__global__ void __launch_bounds__(256) l2_gather_kernel(const uint4* __restrict__ panel, uint32_t nrows,
                                                        int rows_per_warp, uint32_t salt, uint32_t* out) {
  const int lane = threadIdx.x & 31;
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int i = 0; i < rows_per_warp; i += U) {
    uint4 v[U][2];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t r = mix32(gw * 0x9E3779B9u + (uint32_t)(i + u) + salt) % nrows;
      const uint4* row = panel + (size_t)r * 64;  // 1 KB row = 64 x 16 B
      v[u][0] = __ldg(row + lane);
      v[u][1] = __ldg(row + 32 + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x ^= v[u][0].x ^ v[u][1].x; acc.y ^= v[u][0].y ^ v[u][1].y;
      acc.z ^= v[u][0].z ^ v[u][1].z; acc.w ^= v[u][0].w ^ v[u][1].w;
    }
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) out[0] = gw;  // keeps the loads alive
}

extern "C" int l2_probe_run(const void* panel, uint64_t nrows, int blocks, int rows_per_warp, int u,
                            uint32_t salt, void* out, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const uint4* p = (const uint4*)panel;
  uint32_t* o = (uint32_t*)out;
  switch (u) {
    case 1: l2_gather_kernel<1><<<blocks, 256, 0, st>>>(p, (uint32_t)nrows, rows_per_warp, salt, o); break;
    case 2: l2_gather_kernel<2><<<blocks, 256, 0, st>>>(p, (uint32_t)nrows, rows_per_warp, salt, o); break;
    case 4: l2_gather_kernel<4><<<blocks, 256, 0, st>>>(p, (uint32_t)nrows, rows_per_warp, salt, o); break;
    default: l2_gather_kernel<8><<<blocks, 256, 0, st>>>(p, (uint32_t)nrows, rows_per_warp, salt, o); break;
  }
  return (int)cudaGetLastError();
}
