// K2 (partial combine), fp32 split planes, K4 (finalize, P:82,
// P:313) and the R5 pairwise Frobenius tree.  All reductions use a fixed
// order so that results are bit-reproducible run to run.
#include <algorithm>
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

// ---------------------------------------------------------------- K2
template <int VEC>
__global__ void reduce_sketch_kernel(const float* __restrict__ part, int splits, int planes,
                                     int64_t n, int k, float* __restrict__ acc,
                                     const int32_t* __restrict__ map) {
  const int64_t total = n * (int64_t)k / VEC;
  const int64_t part_stride = (int64_t)planes * n * k;  // floats per split
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = v * VEC;  // element index c*k + κ
    float s[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) s[q] = 0.f;
    for (int sp = 0; sp < splits; ++sp) {
      for (int pl = 0; pl < planes; ++pl) {
        const float* src = part + sp * part_stride + (int64_t)pl * n * k + e;
        if constexpr (VEC == 4) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(src));
          s[0] += x.x; s[1] += x.y; s[2] += x.z; s[3] += x.w;
        } else {
          s[0] += __ldg(src);
        }
      }
    }
    // output column: c, or map[c] (scattered head columns of the CSR path;
    // added atomically there: K3's tail may add into the same column on
    // another stream — CSR sums are order-dependent anyway)
    const int64_t c = e / k;
    const int64_t eo = map ? (int64_t)map[c] * k + (e - c * k) : e;
    if (map) {
      if constexpr (VEC == 4) {
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(acc + eo), "f"(s[0]), "f"(s[1]),
                     "f"(s[2]), "f"(s[3])
                     : "memory");
      } else {
        atomicAdd(acc + eo, s[0]);
      }
    } else if constexpr (VEC == 4) {
      float4* dst = reinterpret_cast<float4*>(acc + eo);
      float4 a = *dst;
      a.x += s[0]; a.y += s[1]; a.z += s[2]; a.w += s[3];
      *dst = a;
    } else {
      acc[eo] += s[0];
    }
  }
}

cudaError_t launch_reduce_sketch(const float* part, int splits, int planes, int64_t n, int k,
                                 float* acc, cudaStream_t st, const int32_t* map) {
  const int threads = 256;
  if (k % 4 == 0) {
    int64_t tot = n * k / 4;
    int blocks = (int)std::min<int64_t>((tot + threads - 1) / threads, 148 * 16);
    reduce_sketch_kernel<4><<<blocks, threads, 0, st>>>(part, splits, planes, n, k, acc, map);
  } else {
    int64_t tot = n * k;
    int blocks = (int)std::min<int64_t>((tot + threads - 1) / threads, 148 * 16);
    reduce_sketch_kernel<1><<<blocks, threads, 0, st>>>(part, splits, planes, n, k, acc, map);
  }
  return cudaGetLastError();
}

__global__ void reduce_norms_kernel(const double* __restrict__ pnorm, int slots, int64_t n,
                                    double* __restrict__ nacc, const int32_t* __restrict__ map) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    // fixed (sequential) order; 8 independent loads in flight
    double s = 0.0;
    int q = 0;
    for (; q + 8 <= slots; q += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = pnorm[(int64_t)(q + u) * n + c];
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; q < slots; ++q) s += pnorm[(int64_t)q * n + c];
    if (map) atomicAdd(nacc + map[c], s);  // (see reduce_sketch_kernel)
    else nacc[c] += s;
  }
}

cudaError_t launch_reduce_norms(const double* pnorm, int slots, int64_t n, double* nacc,
                                cudaStream_t st, const int32_t* map) {
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
  reduce_norms_kernel<<<blocks, 256, 0, st>>>(pnorm, slots, n, nacc, map);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- exact plane split
// x = p_1 + ... + p_P exactly, every p_q a bf16 number with a limited number
// of significant bits, so that Π·X = Σ_q Π·p_q with every tensor-core
// product short enough to survive the MMA's accumulation (R21):
//   mode 3 (fp32 x, ±1 Π)        : 8 + 8 + 8 bits, exact (products = p_q, ≤ 8 bits)
//   mode 4 (fp32 x, Gaussian Π)  : 4 + 8 + 8 bits, remainder (|r| <= 2^-21 |x|)
//                                  dropped: <= 5e-7 relative per element
//   mode 2 (bf16 x, Gaussian Π)  : 4 + 4 bits, exact
// (Gaussian Π has 8 significant bits; a 16-bit product loses its low bits
// against a large fp32 accumulator inside tcgen05.mma — measured 1.6e-5
// relative column error — while 12-bit products are kept exactly.)
// Round-to-nearest-even to b significant bits, on the fp32 bit pattern.
__device__ __forceinline__ float round_sig(float x, int b) {
  const uint32_t u = __float_as_uint(x);
  if ((u & 0x7F800000u) == 0u) return 0.0f * x;  // zero / subnormal residue: not produced here
  const int drop = 24 - b;
  const uint32_t half = 1u << (drop - 1);
  const uint32_t lsb = (u >> drop) & 1u;
  const uint32_t mag = ((u & 0x7FFFFFFFu) + half - 1u + lsb) & ~((1u << drop) - 1u);
  return __uint_as_float((u & 0x80000000u) | mag);
}

__global__ void split_planes_kernel(const void* __restrict__ Xv, int x_bf16, int64_t ldx, int64_t rows,
                                    int64_t n, int mode, uint16_t* __restrict__ planes, int64_t ldp,
                                    double* __restrict__ pnorm, int seg_rows) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t seg = blockIdx.y;
  if (c >= n) return;
  const int64_t r0 = seg * seg_rows;
  const int64_t r1 = min(rows, r0 + seg_rows);
  int bits[4];
  int np;
  bool exact = true;
  if (mode == 3) { np = 3; bits[0] = 8; bits[1] = 8; bits[2] = 8; bits[3] = 0; }
  else if (mode == 4) { np = 3; bits[0] = 4; bits[1] = 8; bits[2] = 8; bits[3] = 0; exact = false; }
  else { np = 2; bits[0] = 4; bits[1] = 8; bits[2] = 0; bits[3] = 0; }
  double s2 = 0.0;
  for (int64_t t = r0; t < r1; ++t) {
    float x;
    if (x_bf16) x = __uint_as_float((uint32_t)static_cast<const uint16_t*>(Xv)[t * ldx + c] << 16);
    else x = static_cast<const float*>(Xv)[t * ldx + c];
    uint16_t* row = planes + t * ldp;
    float r = x;
    for (int q = 0; q < np; ++q) {
      // the last plane takes the (exactly representable) remainder
      const float p = (q == np - 1 && exact) ? r : round_sig(r, bits[q]);
      row[q * n + c] = (uint16_t)(__float_as_uint(p) >> 16);
      r = __fsub_rn(r, p);
    }
    const double xd = (double)x;
    s2 = fma(xd, xd, s2);
  }
  pnorm[seg * n + c] = s2;
}

// Vectorised variant: thread per 8 consecutive columns (two float4 or one
// uint4 load, one 16-byte store per plane), same arithmetic per element.
__global__ void split_planes_v8_kernel(const void* __restrict__ Xv, int x_bf16, int64_t ldx, int64_t rows,
                                       int64_t n, int mode, uint16_t* __restrict__ planes, int64_t ldp,
                                       double* __restrict__ pnorm, int seg_rows) {
  const int64_t c0 = 8 * (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const int64_t seg = blockIdx.y;
  if (c0 >= n) return;
  const int64_t r0 = seg * seg_rows;
  const int64_t r1 = min(rows, r0 + seg_rows);
  int bits[3];
  int np;
  bool exact = true;
  if (mode == 3) { np = 3; bits[0] = 8; bits[1] = 8; bits[2] = 8; }
  else if (mode == 4) { np = 3; bits[0] = 4; bits[1] = 8; bits[2] = 8; exact = false; }
  else { np = 2; bits[0] = 4; bits[1] = 8; bits[2] = 0; }
  double s2[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) s2[j] = 0.0;
  for (int64_t t = r0; t < r1; ++t) {
    float x[8];
    if (x_bf16) {
      const uint4 v = *reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(Xv) + t * ldx + c0);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) { x[2 * j] = __uint_as_float(w[j] << 16); x[2 * j + 1] = __uint_as_float(w[j] & 0xFFFF0000u); }
    } else {
      const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(Xv) + t * ldx + c0);
      const float4 a = src[0], b = src[1];
      x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w; x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
    }
    uint16_t* row = planes + t * ldp + c0;
    float r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { r[j] = x[j]; s2[j] = fma((double)x[j], (double)x[j], s2[j]); }
    for (int q = 0; q < np; ++q) {
      uint32_t o[4];
#pragma unroll
      for (int j = 0; j < 8; j += 2) {
        const float pa = (q == np - 1 && exact) ? r[j] : round_sig(r[j], bits[q]);
        const float pb = (q == np - 1 && exact) ? r[j + 1] : round_sig(r[j + 1], bits[q]);
        o[j / 2] = (__float_as_uint(pa) >> 16) | (__float_as_uint(pb) & 0xFFFF0000u);
        r[j] = __fsub_rn(r[j], pa);
        r[j + 1] = __fsub_rn(r[j + 1], pb);
      }
      *reinterpret_cast<uint4*>(row + q * n) = make_uint4(o[0], o[1], o[2], o[3]);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) pnorm[seg * n + c0 + j] = s2[j];
}

cudaError_t launch_split_planes(const void* X, int x_bf16, int64_t ldx, int64_t rows, int64_t n,
                                int mode, uint16_t* planes, int64_t ldp, double* pnorm, int seg_rows,
                                cudaStream_t st) {
  const int es = x_bf16 ? 2 : 4;
  const bool vec = (n % 8 == 0) && (ldx % 8 == 0) && (ldp % 8 == 0) &&
                   (reinterpret_cast<uintptr_t>(X) % 16 == 0);
  (void)es;
  if (vec) {
    dim3 grid((unsigned)((n / 8 + 127) / 128), (unsigned)((rows + seg_rows - 1) / seg_rows));
    split_planes_v8_kernel<<<grid, 128, 0, st>>>(X, x_bf16, ldx, rows, n, mode, planes, ldp, pnorm, seg_rows);
  } else {
    dim3 grid((unsigned)((n + 127) / 128), (unsigned)((rows + seg_rows - 1) / seg_rows));
    split_planes_kernel<<<grid, 128, 0, st>>>(X, x_bf16, ldx, rows, n, mode, planes, ldp, pnorm, seg_rows);
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K4
// One warp per column: Ã_c = acc_c * fp32(1/sqrt(k)); ||Ã_c|| in fp64;
// D_c = ||X_c|| / ||Ã_c|| (0 if ||Ã_c|| = 0).
__global__ void finalize_kernel(const float* __restrict__ acc, double* __restrict__ nacc,
                                int64_t n, int k, float scale, float* __restrict__ out,
                                double* __restrict__ sknorm, double* __restrict__ D,
                                int* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t c = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); c < n;
       c += warps) {
    double s2 = 0.0;
    for (int kp = lane; kp < k; kp += 32) {
      const float v = __fmul_rn(acc[c * k + kp], scale);
      out[c * k + kp] = v;
      s2 = fma((double)v, (double)v, s2);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    if (lane == 0) {
      const double sn = sqrt(s2);
      double a2 = nacc[c];
      // R25: norms² below 2^-200 are the exact-zero column (the bf16 norm
      // path maps a zero to 2^-127, whose square is absorbed otherwise)
      if (a2 < 0x1p-200) { a2 = 0.0; nacc[c] = 0.0; }
      sknorm[c] = sn;
      D[c] = sn > 0.0 ? sqrt(a2) / sn : 0.0;
      if (!(a2 == a2) || !(sn == sn) || isinf(a2)) atomicOr(status, 1);
    }
  }
}

cudaError_t launch_finalize(const float* acc, double* nacc, int64_t n, int k, float scale,
                            float* out, double* sknorm, double* D, int* status, cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((n + 7) / 8, 148 * 8);
  if (blocks < 1) blocks = 1;
  finalize_kernel<<<blocks, 256, 0, st>>>(acc, nacc, n, k, scale, out, sknorm, D, status);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- R5 tree
// pad to a power of two with zeros, sum adjacent pairs level by level
// (ping-pong buffers; identical tree to the written definition).
__global__ void pairwise_sum_kernel(const double* __restrict__ x, int64_t n, int64_t p,
                                    double* __restrict__ buf, double* __restrict__ out) {
  double* a = buf;
  double* b = buf + p;
  for (int64_t i = threadIdx.x; i < p; i += blockDim.x) a[i] = i < n ? x[i] : 0.0;
  __syncthreads();
  int64_t len = p;
  while (len > 1) {
    len >>= 1;
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) b[i] = a[2 * i] + a[2 * i + 1];
    __syncthreads();
    double* t = a; a = b; b = t;
  }
  if (threadIdx.x == 0) *out = p > 0 ? a[0] : 0.0;
}

cudaError_t launch_pairwise_sum(const double* x, int64_t n, double* scratch, double* out,
                                cudaStream_t st) {
  int64_t p = 1;
  while (p < n) p <<= 1;
  if (n <= 0) p = 0;
  pairwise_sum_kernel<<<1, 1024, 0, st>>>(x, n, p, scratch, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- combine exchange
// The cross-shard combine (P:145 treeAggregate) is ONE
// all-reduce-sum of a single fp64 buffer [sketch sums (n_tot·k) | norms² (n_tot)]:
// the fp32 sketch partials widened exactly, the fp64 norms copied.  The sum of
// G <= 8 widened fp32 partials in fp64 is exact unless their exponents span
// more than 29 binades, so the reduction order NCCL picks does not change
// the result; the unpack rounds the sketch sum to fp32 once.
__global__ void pack_partials_kernel(const float* __restrict__ sk, int64_t nsk, const double* __restrict__ nrm,
                                     int64_t nn, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nsk + nn;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = i < nsk ? (double)sk[i] : nrm[i - nsk];
}

__global__ void unpack_partials_kernel(const double* __restrict__ in, int64_t nsk, int64_t nn,
                                       float* __restrict__ sk, double* __restrict__ nrm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nsk + nn;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < nsk) sk[i] = __double2float_rn(in[i]);
    else nrm[i - nsk] = in[i];
  }
}

static int exch_blocks(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

cudaError_t launch_pack_partials(const float* sk, int64_t nsk, const double* nrm, int64_t nn, double* out,
                                 cudaStream_t st) {
  pack_partials_kernel<<<exch_blocks(nsk + nn), 256, 0, st>>>(sk, nsk, nrm, nn, out);
  return cudaGetLastError();
}

cudaError_t launch_unpack_partials(const double* in, int64_t nsk, int64_t nn, float* sk, double* nrm,
                                   cudaStream_t st) {
  unpack_partials_kernel<<<exch_blocks(nsk + nn), 256, 0, st>>>(in, nsk, nn, sk, nrm);
  return cudaGetLastError();
}

}  // namespace smp
