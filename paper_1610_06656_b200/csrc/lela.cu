// LELA (Bhojanapalli et al.), the two-pass comparison system of the paper
// (Table 1, runtime P:191-192; SURVEY §8f
// NEXT-3), on the same device data path as SMP-PCA:
//   pass 1: exact column norms only (K_N below; Ω then comes from Eq. 1
//           exactly as for SMP-PCA, smp_sample_estimate);
//   pass 2: the EXACT entries of AᵀB on Ω ("a second pass to compute
//           the sampled entries"): acc[s] += Σ_t A[t, I_s] B[t, J_s].
// Pass 2 streams the row block in chunks of LELA_R rows: each chunk of A and
// B is transposed into an L2-resident column-major fp32 buffer (n × LELA_R;
// K_T), then one thread per sample takes the two contiguous LELA_R-vectors
// and accumulates their products in fp64 (fp32 × fp32 products are exact in
// fp64; K_E).  Samples arrive sorted by (i, j), so a warp's A-vector is
// mostly one L1-resident row and the B-vectors are L2 gathers.
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

constexpr int LELA_R = 64;          // rows per chunk (transposed buffer width)
constexpr int NORM_SEG = 1024;      // rows per norm partial

template <bool BF16>
__device__ __forceinline__ double load_x(const void* X, int64_t idx) {
  if (BF16) return (double)__uint_as_float((uint32_t)static_cast<const uint16_t*>(X)[idx] << 16);
  return (double)static_cast<const float*>(X)[idx];
}

// K_N: pnorm[seg][c] = Σ_{t in segment} X[t, c]² (fp64; squares of bf16 /
// fp32 values are exact in fp64), one column per thread, rows unrolled
template <bool BF16>
__global__ void colnorm_kernel(const void* __restrict__ X, int64_t ldx, int64_t rows, int64_t n,
                               double* __restrict__ pnorm) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * NORM_SEG;
  const int64_t r1 = min(rows, r0 + NORM_SEG);
  if (c >= n) return;
  double acc = 0.0;
  int64_t t = r0;
  for (; t + 8 <= r1; t += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = load_x<BF16>(X, (t + u) * ldx + c);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = fma(v[u], v[u], acc);
  }
  for (; t < r1; ++t) {
    const double v = load_x<BF16>(X, t * ldx + c);
    acc = fma(v, v, acc);
  }
  pnorm[(int64_t)blockIdx.y * n + c] = acc;
}

cudaError_t launch_colnorms(const void* X, int x_bf16, int64_t ldx, int64_t rows, int64_t n, double* pnorm,
                            int* segs, cudaStream_t st) {
  const int64_t nseg = (rows + NORM_SEG - 1) / NORM_SEG;
  *segs = (int)nseg;
  if (nseg == 0 || n == 0) return cudaSuccess;
  if (nseg > 65535) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)nseg);
  if (x_bf16) colnorm_kernel<true><<<grid, 256, 0, st>>>(X, ldx, rows, n, pnorm);
  else colnorm_kernel<false><<<grid, 256, 0, st>>>(X, ldx, rows, n, pnorm);
  return cudaGetLastError();
}

// K_T: out[c · LELA_R + r] = X[r, c] for r < rc (0 for rc <= r < LELA_R),
// 32 × 32 tiles through SMEM (coalesced on both sides)
template <bool BF16>
__global__ void lela_transpose_kernel(const void* __restrict__ X, int64_t ldx, int rc, int64_t n,
                                      float* __restrict__ out) {
  __shared__ float tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32;
  const int r0 = blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int r = r0 + y;
    const int64_t c = c0 + threadIdx.x;
    tile[y][threadIdx.x] = (r < rc && c < n) ? (float)load_x<BF16>(X, (int64_t)r * ldx + c) : 0.0f;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y;
    if (c < n) out[c * LELA_R + r0 + threadIdx.x] = tile[threadIdx.x][y];
  }
}

// K_E: acc[s] += Σ_{r < LELA_R} At[I_s][r] · Bt[J_s][r]  (fp64 accumulation)
__global__ void lela_entries_kernel(const float* __restrict__ At, const float* __restrict__ Bt,
                                    const int32_t* __restrict__ I, const int32_t* __restrict__ J,
                                    int64_t cnt, double* __restrict__ acc) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cnt;
       s += (int64_t)gridDim.x * blockDim.x) {
    const float4* a = reinterpret_cast<const float4*>(At + (int64_t)I[s] * LELA_R);
    const float4* b = reinterpret_cast<const float4*>(Bt + (int64_t)J[s] * LELA_R);
    double x = 0.0, y = 0.0;
#pragma unroll 4
    for (int q = 0; q < LELA_R / 4; ++q) {
      const float4 u = __ldg(a + q), v = __ldcg(b + q);
      x = fma((double)u.x, (double)v.x, x);
      y = fma((double)u.y, (double)v.y, y);
      x = fma((double)u.z, (double)v.z, x);
      y = fma((double)u.w, (double)v.w, y);
    }
    acc[s] += x + y;
  }
}

cudaError_t launch_exact_entries(const void* A, int64_t lda, const void* B, int64_t ldb, int x_bf16,
                                 int64_t rows, int64_t n1, int64_t n2, const int32_t* I, const int32_t* J,
                                 int64_t cnt, double* acc, float* At, float* Bt, int64_t* launches,
                                 cudaStream_t st) {
  const int es = x_bf16 ? 2 : 4;
  const int eb = (int)std::min<int64_t>(std::max<int64_t>((cnt + 255) / 256, 1), 148 * 32);
  for (int64_t r0 = 0; r0 < rows; r0 += LELA_R) {
    const int rc = (int)std::min<int64_t>(LELA_R, rows - r0);
    const uint8_t* Ab = static_cast<const uint8_t*>(A) + r0 * lda * es;
    const uint8_t* Bb = static_cast<const uint8_t*>(B) + r0 * ldb * es;
    dim3 blk(32, 8);
    dim3 ga((unsigned)((n1 + 31) / 32), LELA_R / 32), gb((unsigned)((n2 + 31) / 32), LELA_R / 32);
    if (x_bf16) {
      lela_transpose_kernel<true><<<ga, blk, 0, st>>>(Ab, lda, rc, n1, At);
      lela_transpose_kernel<true><<<gb, blk, 0, st>>>(Bb, ldb, rc, n2, Bt);
    } else {
      lela_transpose_kernel<false><<<ga, blk, 0, st>>>(Ab, lda, rc, n1, At);
      lela_transpose_kernel<false><<<gb, blk, 0, st>>>(Bb, ldb, rc, n2, Bt);
    }
    if (cnt > 0) lela_entries_kernel<<<eb, 256, 0, st>>>(At, Bt, I, J, cnt, acc);
    *launches += 3;
  }
  return cudaGetLastError();
}

int lela_chunk_rows() { return LELA_R; }

}  // namespace smp
