// K5: biased Bernoulli sample Ω (Alg. 1 line 3; Eq. 1,
// P:70-73) and K6: rescaled-JL estimates on Ω (Alg. 1 line 4; Eq. 2,
// P:80-83).
//
//   alpha_i = a2_i / ((2 n2) FA),  beta_j = b2_j / ((2 n1) FB)       (R6)
//   q̂_ij   = min(1, m (alpha_i + beta_j))                            (Eq. 1)
//   (i,j) ∈ Ω  iff  U53(Philox(ctr=(i,j,0,3), key=seed)) 2^-53 < q̂_ij   (§3.4)
//   M̃_ij   = D_A[i] D_B[j] <Ã_i, B̃_j>                               (Eq. 2)
//
// fp64 arithmetic uses explicitly rounded intrinsics (no FMA contraction) so
// q̂ — and therefore Ω — is bit-identical to the written definition.
// Ω is produced in (i,j) order by a count pass, an exclusive scan of block
// counts and a write pass that recomputes the same draws.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

constexpr int OM_THREADS = 256;
constexpr int OM_PER_THREAD = 16;
constexpr int64_t OM_PER_BLOCK = (int64_t)OM_THREADS * OM_PER_THREAD;

__global__ void alpha_beta_kernel(const double* __restrict__ a2, int64_t n1,
                                  const double* __restrict__ b2, int64_t n2,
                                  const double* __restrict__ FAFB, double* __restrict__ alpha,
                                  double* __restrict__ beta) {
  const double da = __dmul_rn(__dmul_rn(2.0, (double)n2), FAFB[0]);
  const double db = __dmul_rn(__dmul_rn(2.0, (double)n1), FAFB[1]);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1 + n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i < n1) alpha[i] = __ddiv_rn(a2[i], da);
    else beta[i - n1] = __ddiv_rn(b2[i - n1], db);
  }
}

cudaError_t launch_alpha_beta(const double* a2, int64_t n1, const double* b2, int64_t n2,
                              const double* FAFB, double* alpha, double* beta, cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((n1 + n2 + 255) / 256, 1024);
  alpha_beta_kernel<<<blocks, 256, 0, st>>>(a2, n1, b2, n2, FAFB, alpha, beta);
  return cudaGetLastError();
}

__device__ __forceinline__ double qhat_of(double m, double al, double be) {
  const double q = __dmul_rn(m, __dadd_rn(al, be));
  return q < 1.0 ? q : 1.0;
}

__device__ __forceinline__ bool draw(uint32_t k0, uint32_t k1, uint32_t i, uint32_t j, double qh) {
  const u32x4 w = philox4x32_10(i, j, 0u, TAG_OMEGA, k0, k1);
  const uint64_t u53 = (((uint64_t)w.y << 32) | (uint64_t)w.x) >> 11;
  const double u = __dmul_rn(__ull2double_rn(u53), 0x1p-53);
  return u < qh;
}

// per-thread bitmask of hits among its 16 consecutive pairs
__device__ __forceinline__ uint32_t thread_hits(const double* __restrict__ alpha,
                                                const double* __restrict__ beta, int64_t n2,
                                                int64_t N, double m, uint32_t k0, uint32_t k1,
                                                int64_t P0) {
  uint32_t mask = 0;
  if (P0 >= N) return 0;
  int64_t i = P0 / n2, j = P0 - i * n2;
  double al = alpha[i];
#pragma unroll 4
  for (int e = 0; e < OM_PER_THREAD; ++e) {
    if (P0 + e < N) {
      const double qh = qhat_of(m, al, beta[j]);
      if (draw(k0, k1, (uint32_t)i, (uint32_t)j, qh)) mask |= 1u << e;
      if (++j == n2) { j = 0; ++i; if (i * n2 < N) al = alpha[i]; }
    }
  }
  return mask;
}

// block-wide exclusive scan of one int per thread; returns the block total
__device__ __forceinline__ int block_excl_scan(int v, int& excl) {
  __shared__ int wsum[OM_THREADS / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int s = lane < OM_THREADS / 32 ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < OM_THREADS / 32) wsum[lane] = s;
  }
  __syncthreads();
  const int wprefix = wid > 0 ? wsum[wid - 1] : 0;
  excl = wprefix + x - v;
  const int total = wsum[OM_THREADS / 32 - 1];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(OM_THREADS)
omega_count_kernel(const double* __restrict__ alpha, const double* __restrict__ beta, int64_t n1,
                   int64_t n2, double m, uint64_t seed, int64_t* __restrict__ blk_counts) {
  const int64_t N = n1 * n2;
  const int64_t P0 = blockIdx.x * OM_PER_BLOCK + (int64_t)threadIdx.x * OM_PER_THREAD;
  const uint32_t mask = thread_hits(alpha, beta, n2, N, m, (uint32_t)seed, (uint32_t)(seed >> 32), P0);
  int excl;
  const int tot = block_excl_scan(__popc(mask), excl);
  if (threadIdx.x == 0) blk_counts[blockIdx.x] = tot;
}

int64_t omega_num_blocks(int64_t n1, int64_t n2) { return (n1 * n2 + OM_PER_BLOCK - 1) / OM_PER_BLOCK; }

cudaError_t launch_omega_count(const double* alpha, const double* beta, int64_t n1, int64_t n2,
                               double m, uint64_t seed, int64_t* blk_counts, cudaStream_t st) {
  const int64_t nb = omega_num_blocks(n1, n2);
  if (nb == 0) return cudaSuccess;
  omega_count_kernel<<<(unsigned)nb, OM_THREADS, 0, st>>>(alpha, beta, n1, n2, m, seed, blk_counts);
  return cudaGetLastError();
}

// single-block exclusive scan of the block counts (in place); *total = sum
__global__ void scan_counts_kernel(int64_t* __restrict__ c, int64_t nblk, int64_t* __restrict__ total) {
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t per = (nblk + 1023) / 1024;
  const int64_t b0 = tid * per, b1 = min(nblk, b0 + per);
  int64_t s = 0;
  for (int64_t b = b0; b < b1; ++b) s += c[b];
  part[tid] = s;
  __syncthreads();
  if (tid == 0) {
    int64_t run = 0;
    for (int q = 0; q < 1024; ++q) { int64_t v = part[q]; part[q] = run; run += v; }
    *total = run;
  }
  __syncthreads();
  int64_t run = part[tid];
  for (int64_t b = b0; b < b1; ++b) { int64_t v = c[b]; c[b] = run; run += v; }
}

cudaError_t launch_scan_counts(int64_t* blk_counts, int64_t nblk, int64_t* total, cudaStream_t st) {
  scan_counts_kernel<<<1, 1024, 0, st>>>(blk_counts, nblk, total);
  return cudaGetLastError();
}

__global__ void __launch_bounds__(OM_THREADS)
omega_write_kernel(const double* __restrict__ alpha, const double* __restrict__ beta, int64_t n1,
                   int64_t n2, double m, uint64_t seed, const int64_t* __restrict__ blk_offsets,
                   const int64_t* __restrict__ total, int64_t cap, int32_t* __restrict__ I,
                   int32_t* __restrict__ J, double* __restrict__ qhat) {
  if (*total > cap) return;  // caller re-calls with a larger buffer
  const int64_t N = n1 * n2;
  const int64_t P0 = blockIdx.x * OM_PER_BLOCK + (int64_t)threadIdx.x * OM_PER_THREAD;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint32_t mask = thread_hits(alpha, beta, n2, N, m, k0, k1, P0);
  int excl;
  block_excl_scan(__popc(mask), excl);
  int64_t pos = blk_offsets[blockIdx.x] + excl;
  uint32_t mm = mask;
  while (mm) {
    const int e = __ffs(mm) - 1;
    mm &= mm - 1;
    const int64_t P = P0 + e;
    const int64_t i = P / n2, j = P - i * n2;
    I[pos] = (int32_t)i;
    J[pos] = (int32_t)j;
    qhat[pos] = qhat_of(m, alpha[i], beta[j]);
    ++pos;
  }
}

cudaError_t launch_omega_write(const double* alpha, const double* beta, int64_t n1, int64_t n2,
                               double m, uint64_t seed, const int64_t* blk_offsets,
                               const int64_t* total, int64_t cap, int32_t* I, int32_t* J,
                               double* qhat, cudaStream_t st) {
  const int64_t nb = omega_num_blocks(n1, n2);
  if (nb == 0) return cudaSuccess;
  omega_write_kernel<<<(unsigned)nb, OM_THREADS, 0, st>>>(alpha, beta, n1, n2, m, seed, blk_offsets,
                                                          total, cap, I, J, qhat);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K6 SDDMM
// one warp per sample; Ω is sorted by i so consecutive warps reuse Ã_i.
__global__ void sddmm_kernel(const float* __restrict__ Ask, const float* __restrict__ Bsk,
                             const double* __restrict__ DA, const double* __restrict__ DB, int k,
                             const int32_t* __restrict__ I, const int32_t* __restrict__ J,
                             const int64_t* __restrict__ total, int64_t cap, int plain,
                             float* __restrict__ val) {
  if (*total > cap) return;  // Ω not written (capacity); nothing to estimate
  const int64_t cnt = *total;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t s = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); s < cnt; s += nw) {
    const int64_t i = I[s], j = J[s];
    const float* a = Ask + i * k;
    const float* b = Bsk + j * k;
    double dot = 0.0;
    for (int kp = lane; kp < k; kp += 32) dot = fma((double)__ldg(a + kp), (double)__ldg(b + kp), dot);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) val[s] = plain ? (float)dot : (float)(__dmul_rn(__dmul_rn(DA[i], DB[j]), dot));
  }
}

cudaError_t launch_sddmm(const float* Ask, const float* Bsk, const double* DA, const double* DB,
                         int k, const int32_t* I, const int32_t* J, const int64_t* total,
                         int64_t cap, int plain, float* val, cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((cap + 7) / 8, 148 * 16);
  if (blocks < 1) blocks = 1;
  sddmm_kernel<<<blocks, 256, 0, st>>>(Ask, Bsk, DA, DB, k, I, J, total, cap, plain, val);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K5m
// Row-multinomial Ω (the paper's appendix sampler, with Alg. 1
// line 3's saturation; R27; NEXT-2): O(n2 log n2 + m log n2) work
// instead of the n1·n2 Bernoulli sweep.  fp64 with explicit rounding (no
// contraction) so that the saturated prefixes, the draw counts and the drawn
// columns are bit-exact with the written definition:
//   σ = columns by β descending (ties: index ascending), Bp = sequential
//   prefix of β_σ; row i: s_i = first p with m(α_i + β_σ(p)) < 1,
//   T_i = (n2 − s_i)α_i + (Btot − Bp[s_i−1]), M_i = floor(m T_i + u_i);
//   draw d: first p >= s_i with (p − s_i + 1)α_i + (Bp[p] − Bp[s_i−1]) > u T_i;
//   Ω = {(i, σ(p)) : p < s_i} ∪ {distinct draws}, q̂ = 1 on the saturated
//   pairs, 1 − (1−π)^F (1 − fπ) on drawn ones (π = (α_i+β_j)/T_i, F = ⌊m T_i⌋).
enum : uint32_t { TAG_MN_COUNT = 8, TAG_MN_DRAW = 9 };

__device__ __forceinline__ double u53_of(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1, uint32_t tag) {
  const u32x4 w = philox4x32_10(c0, c1, 0u, tag, k0, k1);
  const uint64_t v = (((uint64_t)w.y << 32) | (uint64_t)w.x) >> 11;
  return __dmul_rn(__ull2double_rn(v), 0x1p-53);
}

__global__ void mn_iota_kernel(int32_t* __restrict__ p, int64_t n) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    p[j] = (int32_t)j;
}

// Bp[p] = β_σ(0) + ... + β_σ(p), sequential (the definition's order)
__global__ void mn_prefix_kernel(const double* __restrict__ bsorted, int64_t n2, double* __restrict__ bp) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    double acc = 0.0;
    for (int64_t p = 0; p < n2; ++p) { acc = __dadd_rn(acc, bsorted[p]); bp[p] = acc; }
  }
}

// per row: s_i, T_i, and the row's entry count s_i + M_i (-> offsets by scan)
__global__ void mn_rows_kernel(const double* __restrict__ alpha, const double* __restrict__ bsorted,
                               const double* __restrict__ bp, int64_t n1, int64_t n2, double m, uint64_t seed,
                               int64_t* __restrict__ sat, double* __restrict__ Tr, int64_t* __restrict__ counts) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const double btot = n2 > 0 ? bp[n2 - 1] : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n1; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n1) { counts[n1] = 0; continue; }   // -> offs[n1] = total after the scan
    const double ai = alpha[i];
    int64_t lo = 0, hi = n2;                     // first p with q < 1 (q non-increasing in p)
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const double q = __dmul_rn(m, __dadd_rn(ai, bsorted[mid]));
      if (q < 1.0) hi = mid; else lo = mid + 1;
    }
    const double base = lo > 0 ? bp[lo - 1] : 0.0;
    const double T = __dadd_rn(__dmul_rn((double)(n2 - lo), ai), __dadd_rn(btot, -base));
    const int64_t Mi = lo < n2 ? (int64_t)floor(__dadd_rn(__dmul_rn(m, T), u53_of(k0, k1, (uint32_t)i, 0u, TAG_MN_COUNT))) : 0;
    sat[i] = lo;
    Tr[i] = T;
    counts[i] = lo + Mi;
  }
}

// warp per row: the saturated prefix σ(0..s_i), then the row's draws (CDF
// inversion by binary search), into Jtmp[offs[i] ..]
__global__ void mn_fill_kernel(const double* __restrict__ alpha, const int32_t* __restrict__ sig,
                               const double* __restrict__ bp, int64_t n1, int64_t n2, uint64_t seed,
                               const int64_t* __restrict__ sat, const double* __restrict__ Tr,
                               const int64_t* __restrict__ offs, int32_t* __restrict__ Jtmp) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n1; i += nw) {
    const int64_t o0 = offs[i], o1 = offs[i + 1];
    const int64_t s = sat[i];
    const double ai = alpha[i], T = Tr[i];
    const double base = s > 0 ? bp[s - 1] : 0.0;
    for (int64_t p = lane; p < s; p += 32) Jtmp[o0 + p] = sig[p];
    for (int64_t d = lane; d < o1 - o0 - s; d += 32) {
      const double target = __dmul_rn(u53_of(k0, k1, (uint32_t)i, (uint32_t)d, TAG_MN_DRAW), T);
      int64_t lo = s, hi = n2 - 1;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        const double c = __dadd_rn(__dmul_rn((double)(mid - s + 1), ai), __dadd_rn(bp[mid], -base));
        if (c > target) hi = mid; else lo = mid + 1;
      }
      Jtmp[o0 + s + d] = sig[lo];
    }
  }
}

// flag[e] = 1 for the first occurrence of a column in its row's sorted run
__global__ void mn_flag_kernel(const int32_t* __restrict__ Jsrt, const int64_t* __restrict__ offs, int64_t n1,
                               int32_t* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n1; i += nw) {
    const int64_t o0 = offs[i], o1 = offs[i + 1];
    for (int64_t e = o0 + lane; e < o1; e += 32) flag[e] = (e == o0 || Jsrt[e] != Jsrt[e - 1]) ? 1 : 0;
  }
}

__global__ void mn_total_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ pos, int64_t D,
                                int64_t* __restrict__ total) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *total = D > 0 ? (int64_t)pos[D - 1] + flag[D - 1] : 0;
}

__device__ __forceinline__ double mn_qhat_of(double m, double ai, double bj, double T) {
  const double mi = __dmul_rn(m, T);
  const double F = floor(mi);
  const double f = __dadd_rn(mi, -F);
  const double pi = __ddiv_rn(__dadd_rn(ai, bj), T);
  if (!(pi > 0.0)) return 0.0;
  if (pi >= 1.0) return F >= 1.0 ? 1.0 : f;
  return -expm1(__dadd_rn(__dmul_rn(F, log1p(-pi)), log1p(-__dmul_rn(f, pi))));
}

// Ω in (i, j) order: compacted distinct entries with q̂
__global__ void mn_write_kernel(const double* __restrict__ alpha, const double* __restrict__ beta,
                                const int32_t* __restrict__ Jsrt, const int32_t* __restrict__ flag,
                                const int32_t* __restrict__ pos, const int64_t* __restrict__ offs,
                                const double* __restrict__ Tr, int64_t n1, double m, int32_t* __restrict__ I,
                                int32_t* __restrict__ J, double* __restrict__ qhat) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n1; i += nw) {
    const int64_t o0 = offs[i], o1 = offs[i + 1];
    const double ai = alpha[i], T = Tr[i];
    for (int64_t e = o0 + lane; e < o1; e += 32) {
      if (!flag[e]) continue;
      const int32_t j = Jsrt[e];
      const int64_t o = pos[e];
      const double bj = beta[j];
      const double q = __dmul_rn(m, __dadd_rn(ai, bj));
      I[o] = (int32_t)i;
      J[o] = j;
      qhat[o] = q >= 1.0 ? 1.0 : mn_qhat_of(m, ai, bj, T);
    }
  }
}

template <class T>
static cudaError_t mn_ensure(T*& p, int64_t& cap, int64_t need) {
  if (need <= cap) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, (size_t)std::max<int64_t>(need, 1) * sizeof(T));
  if (e == cudaSuccess) cap = std::max<int64_t>(need, 1);
  return e;
}

void mn_workspace_free(MnWorkspace& w) {
  cudaFree(w.sig); cudaFree(w.iota); cudaFree(w.bsorted); cudaFree(w.bp); cudaFree(w.sat); cudaFree(w.Tr);
  cudaFree(w.offs); cudaFree(w.jtmp); cudaFree(w.jsrt); cudaFree(w.flag); cudaFree(w.pos); cudaFree(w.tmp);
  cudaFree(w.total);
  if (w.total_h) cudaFreeHost(w.total_h);
  w = MnWorkspace{};
}

#define MN_TRY(x)                         \
  do {                                    \
    cudaError_t e_ = (x);                 \
    if (e_ != cudaSuccess) return e_;     \
  } while (0)

cudaError_t run_sample_multinomial(MnWorkspace& w, const double* alpha, const double* beta, int64_t n1,
                                   int64_t n2, double m, uint64_t seed, int64_t cap, int32_t* I, int32_t* J,
                                   double* qhat, int64_t* count, int64_t* launches, cudaStream_t st) {
  MN_TRY(mn_ensure(w.sig, w.sig_cap, n2));
  MN_TRY(mn_ensure(w.iota, w.iota_cap, n2));
  MN_TRY(mn_ensure(w.bsorted, w.bsorted_cap, n2));
  MN_TRY(mn_ensure(w.bp, w.bp_cap, n2));
  MN_TRY(mn_ensure(w.sat, w.sat_cap, n1));
  MN_TRY(mn_ensure(w.Tr, w.Tr_cap, n1));
  MN_TRY(mn_ensure(w.offs, w.offs_cap, n1 + 1));
  int64_t one = 0;
  MN_TRY(mn_ensure(w.total, one, 1));
  if (!w.total_h) MN_TRY(cudaMallocHost(&w.total_h, 8));
  const int nb2 = (int)std::max<int64_t>(1, std::min<int64_t>((n2 + 255) / 256, 1024));
  const int nb1 = (int)std::max<int64_t>(1, std::min<int64_t>((n1 + 256) / 256, 1024));
  const int nbw = (int)std::max<int64_t>(1, std::min<int64_t>((n1 + 7) / 8, 148 * 16));
  // σ: stable descending radix sort of β (ties keep index order)
  mn_iota_kernel<<<nb2, 256, 0, st>>>(w.iota, n2);
  size_t need = 0;
  MN_TRY(cub::DeviceRadixSort::SortPairsDescending(nullptr, need, beta, w.bsorted, w.iota, w.sig, (int)n2, 0, 64, st));
  MN_TRY(mn_ensure(w.tmp, w.tmp_cap, (int64_t)need));
  size_t have = (size_t)w.tmp_cap;
  MN_TRY(cub::DeviceRadixSort::SortPairsDescending(w.tmp, have, beta, w.bsorted, w.iota, w.sig, (int)n2, 0, 64, st));
  mn_prefix_kernel<<<1, 32, 0, st>>>(w.bsorted, n2, w.bp);
  mn_rows_kernel<<<nb1, 256, 0, st>>>(alpha, w.bsorted, w.bp, n1, n2, m, seed, w.sat, w.Tr, w.offs);
  launch_scan_counts(w.offs, n1 + 1, w.total, st);  // -> exclusive offsets, offs[n1] = D
  MN_TRY(cudaMemcpyAsync(w.total_h, w.total, 8, cudaMemcpyDeviceToHost, st));
  MN_TRY(cudaStreamSynchronize(st));
  const int64_t D = *w.total_h;
  *launches += 6;
  if (D >= (1ll << 31)) return cudaErrorInvalidValue;
  *count = 0;
  if (D > 0) {
    MN_TRY(mn_ensure(w.jtmp, w.jtmp_cap, D));
    MN_TRY(mn_ensure(w.jsrt, w.jsrt_cap, D));
    MN_TRY(mn_ensure(w.flag, w.flag_cap, D));
    MN_TRY(mn_ensure(w.pos, w.pos_cap, D));
    mn_fill_kernel<<<nbw, 256, 0, st>>>(alpha, w.sig, w.bp, n1, n2, seed, w.sat, w.Tr, w.offs, w.jtmp);
    size_t n_sort = 0, n_scan = 0;
    MN_TRY(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, n_sort, w.jtmp, w.jsrt, (int)D, (int)n1, w.offs,
                                                   w.offs + 1, 0, 32, st));
    MN_TRY(cub::DeviceScan::ExclusiveSum(nullptr, n_scan, w.flag, w.pos, (int)D, st));
    MN_TRY(mn_ensure(w.tmp, w.tmp_cap, (int64_t)std::max(n_sort, n_scan)));
    have = (size_t)w.tmp_cap;
    MN_TRY(cub::DeviceSegmentedRadixSort::SortKeys(w.tmp, have, w.jtmp, w.jsrt, (int)D, (int)n1, w.offs,
                                                   w.offs + 1, 0, 32, st));
    mn_flag_kernel<<<nbw, 256, 0, st>>>(w.jsrt, w.offs, n1, w.flag);
    have = (size_t)w.tmp_cap;
    MN_TRY(cub::DeviceScan::ExclusiveSum(w.tmp, have, w.flag, w.pos, (int)D, st));
    mn_total_kernel<<<1, 32, 0, st>>>(w.flag, w.pos, D, w.total);
    MN_TRY(cudaMemcpyAsync(w.total_h, w.total, 8, cudaMemcpyDeviceToHost, st));
    MN_TRY(cudaStreamSynchronize(st));
    *count = *w.total_h;
    *launches += 5;
    if (*count <= cap) {
      mn_write_kernel<<<nbw, 256, 0, st>>>(alpha, beta, w.jsrt, w.flag, w.pos, w.offs, w.Tr, n1, m, I, J, qhat);
      *launches += 1;
    }
  }
  return cudaGetLastError();
}

}  // namespace smp
