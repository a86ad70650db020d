// K3: sparse (CSR) one-pass sketch with fused exact column norms (Alg. 1
// line 2; bag-of-words inputs P:9).
//
// Warp-level row processing: a warp owns a group of 4 consecutive rows
// t = 4g..4g+3.  Each lane regenerates Π(κ, t) for its κ values
// κ = 4·lane + 128·q once per group (one Philox call per κ covers the 4 rows
// for the Gaussian stream) — π_t is shared by A's and B's
// row t — then, for every nonzero (t, c, v), adds v·π_t into the fp32
// accumulator row c with vectorised float4 atomics (one 512-byte warp
// transaction per nonzero at k = 512) and v² into the fp64 norm (exact for
// integer counts, so the norms are order-independent and bit-exact).
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

constexpr int CSR_QMAX = 8;  // k <= 4096 -> k/128 <= 32 slots; process in passes of 8

__device__ __forceinline__ void pi_group4(int kind, uint64_t seed, uint32_t kappa, uint64_t tg,
                                          float (&v)[4]) {
  // values of Π(κ, 4·tg + e), e = 0..3
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint64_t t = tg * 4;
  if (kind == PI_GAUSSIAN) {
    const u32x4 w = philox4x32_10((uint32_t)tg, kappa, (uint32_t)(tg >> 32), TAG_GAUSSIAN, k0, k1);
    uint16_t a, b, c, d;
    gauss_pair(w.x, w.y, a, b);
    gauss_pair(w.z, w.w, c, d);
    v[0] = bf16_bits_to_float(a); v[1] = bf16_bits_to_float(b);
    v[2] = bf16_bits_to_float(c); v[3] = bf16_bits_to_float(d);
  } else if (kind == PI_RADEMACHER) {
    const u32x4 w = philox4x32_10((uint32_t)(t >> 7), kappa, (uint32_t)(t >> 39), TAG_RADEMACHER, k0, k1);
    const uint32_t b = (uint32_t)(t & 127);
    const uint32_t wi = b >> 5;
    const uint32_t word = wi == 0 ? w.x : wi == 1 ? w.y : wi == 2 ? w.z : w.w;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t ee = (b & 31) + e;
      const uint32_t pos = (ee >> 1) | ((ee & 1u) << 4);
      v[e] = ((word >> pos) & 1u) ? -1.f : 1.f;
    }
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = (__popcll((unsigned long long)kappa & (t + e)) & 1) ? -1.f : 1.f;
  }
}

__global__ void __launch_bounds__(256)
sketch_csr_kernel(int kind, uint64_t seed, int k, int64_t row0, int64_t rows,
                  const int64_t* __restrict__ arp, const int32_t* __restrict__ acol,
                  const float* __restrict__ aval, float* __restrict__ aacc, double* __restrict__ anrm,
                  const int64_t* __restrict__ brp, const int32_t* __restrict__ bcol,
                  const float* __restrict__ bval, float* __restrict__ bacc, double* __restrict__ bnrm,
                  int q_begin, int q_end, int do_norms) {
  const int lane = threadIdx.x & 31;
  const int64_t g_first = row0 >> 2;                // first 4-row group touching the block
  const int64_t g_last = (row0 + rows - 1) >> 2;
  const int64_t ngroups = g_last - g_first + 1;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t abase = arp[0];
  const int64_t bbase = brp ? brp[0] : 0;
  for (int64_t gi = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); gi < ngroups; gi += nw) {
    const uint64_t tg = (uint64_t)(g_first + gi);
    float pv[CSR_QMAX][4][4];  // [q][row e][κ offset]
#pragma unroll
    for (int q = 0; q < CSR_QMAX; ++q) {
      const int qq = q_begin + q;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int kappa = 4 * lane + 128 * qq + c;
        float v[4] = {0.f, 0.f, 0.f, 0.f};
        if (qq < q_end && kappa < k) pi_group4(kind, seed, (uint32_t)kappa, tg, v);
#pragma unroll
        for (int e = 0; e < 4; ++e) pv[q][e][c] = v[e];
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t t = (int64_t)tg * 4 + e;
      if (t < row0 || t >= row0 + rows) continue;
      const int64_t r = t - row0;
#pragma unroll
      for (int mat = 0; mat < 2; ++mat) {
        const int64_t* rp = mat == 0 ? arp : brp;
        if (!rp) continue;
        const int32_t* col = mat == 0 ? acol : bcol;
        const float* val = mat == 0 ? aval : bval;
        float* acc = mat == 0 ? aacc : bacc;
        double* nrm = mat == 0 ? anrm : bnrm;
        const int64_t base = mat == 0 ? abase : bbase;
        const int64_t p0 = rp[r] - base, p1 = rp[r + 1] - base;
        for (int64_t pp = p0; pp < p1; ++pp) {
          const int64_t c = col[pp];
          const float x = val[pp];
          float* dst = acc + c * k;
#pragma unroll
          for (int q = 0; q < CSR_QMAX; ++q) {
            const int kappa = 4 * lane + 128 * (q_begin + q);
            if (q_begin + q < q_end && kappa < k) {
              if ((k & 3) == 0) {
                atomicAdd(reinterpret_cast<float4*>(dst + kappa),
                          make_float4(x * pv[q][e][0], x * pv[q][e][1], x * pv[q][e][2], x * pv[q][e][3]));
              } else {
#pragma unroll
                for (int c2 = 0; c2 < 4; ++c2)
                  if (kappa + c2 < k) atomicAdd(dst + kappa + c2, x * pv[q][e][c2]);
              }
            }
          }
          if (do_norms && lane == 0) atomicAdd(nrm + c, (double)x * (double)x);
        }
      }
    }
  }
}

cudaError_t launch_sketch_csr(int kind, uint64_t seed, int k, int64_t row0, int64_t rows,
                              const int64_t* a_rowptr, const int32_t* a_col, const float* a_val,
                              int64_t a_n, float* a_acc, double* a_nrm, const int64_t* b_rowptr,
                              const int32_t* b_col, const float* b_val, int64_t b_n, float* b_acc,
                              double* b_nrm, cudaStream_t st) {
  (void)a_n; (void)b_n;
  if (rows <= 0) return cudaSuccess;
  const int qtot = (k + 127) / 128;
  const int64_t ngroups = ((row0 + rows - 1) >> 2) - (row0 >> 2) + 1;
  const int blocks = (int)std::min<int64_t>((ngroups + 7) / 8, 148 * 32);
  for (int q0 = 0; q0 < qtot; q0 += CSR_QMAX) {
    const int q1 = std::min(qtot, q0 + CSR_QMAX);
    sketch_csr_kernel<<<blocks, 256, 0, st>>>(kind, seed, k, row0, rows, a_rowptr, a_col, a_val,
                                              a_acc, a_nrm, b_rowptr, b_col, b_val, b_acc, b_nrm,
                                              q0, q1, q0 == 0 ? 1 : 0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace smp
