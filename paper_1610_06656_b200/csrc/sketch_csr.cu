// K3: sparse (CSR) one-pass sketch with fused exact column norms (Alg. 1
// line 2; bag-of-words inputs P:9).
//
//   Ã[:, c] += Σ_{(t, c, v) in the block} v · π_t,    a2[c] += Σ v²
//
// A sparse product has no reuse on both sides at once: a row t's π_t is
// shared by the ~100 nonzeros of that row, a column's accumulator by the
// nonzeros of that column.  K3 keeps the ACCUMULATOR in registers (column-
// stationary) and moves π through L2, once per nonzero:
//
//   K3a  generate the Π panel of Rp rows (bf16, Rp x kp, row t contiguous
//        in κ) into an L2-resident buffer — every Π entry is generated once;
//   K3b  key every nonzero of the panel (A and B) as (column << tbits | t);
//   K3c  counting sort by column (SMEM histograms per CTA row range, one
//        exclusive scan over (column, CTA), SMEM-cursor scatter) -> the
//        panel's nonzeros grouped by column (a per-panel CSC transpose);
//        CUB radix sort for more columns than fit a CTA's SMEM histogram;
//   K3d  warps take fixed chunks of the sorted nonzeros (load balance for
//        Zipf-heavy columns): lanes own κ slices, gather π_t (kp bf16) from
//        the panel, FMA v·π_t into fp32 registers, and flush the column's
//        partial with one vector reduction (red.global.add.v4.f32) when the
//        column changes; lane 0 adds v² into the fp64 norm (exact for
//        integer counts: order-independent, bit-exact).
//
// Products v·π are exact in fp32 (integer counts times bf16); the fp32 sums
// are order-dependent across chunks (the reductions race), so CSR sketches
// agree with the oracle to ~1e-7 relative but are not bit-reproducible run
// to run (K3).
#include <algorithm>
#include <utility>
#include <vector>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cstdio>
#include <cstdlib>
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

// ---------------------------------------------------------------- K3a
// pi[(t - t0) * kp + κ] = Π(κ, t) as bf16 bits, κ < k; zero for k <= κ < kp.
// Thread (κ, row group): one Philox call covers 4 rows (Gaussian) or 32 rows
// of one word (Rademacher); a warp writes 32 consecutive κ of a row (64 B).
__global__ void pi_panel_kernel(int kind, uint64_t seed, int k, int kp, int64_t t0, int rows,
                                uint16_t* __restrict__ pi) {
  const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
  const int rpg = kind == PI_RADEMACHER ? 32 : 4;  // rows per generator call
  const int64_t g_first = t0 / rpg, g_last = (t0 + rows - 1) / rpg;
  const int64_t ngroups = g_last - g_first + 1;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const uint32_t total = (uint32_t)(ngroups * kp);  // < 2^32: rows <= 2^15 per panel
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (uint32_t)nthreads) {
    const int kappa = (int)(e % (uint32_t)kp);
    const int64_t g = g_first + (int64_t)(e / (uint32_t)kp);
    const int64_t tb = g * rpg;
    if (kappa >= k) {
      for (int j = 0; j < rpg; ++j) {
        const int64_t t = tb + j;
        if (t >= t0 && t < t0 + rows) pi[(t - t0) * kp + kappa] = 0;
      }
      continue;
    }
    if (kind == PI_GAUSSIAN) {
      const u32x4 w = philox4x32_10((uint32_t)g, (uint32_t)kappa, (uint32_t)(g >> 32), TAG_GAUSSIAN, k0, k1);
      uint16_t z[4];
      gauss_pair(w.x, w.y, z[0], z[1]);
      gauss_pair(w.z, w.w, z[2], z[3]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t t = tb + j;
        if (t >= t0 && t < t0 + rows) pi[(t - t0) * kp + kappa] = z[j];
      }
    } else if (kind == PI_RADEMACHER) {
      // word (t >> 5) & 3 of Philox(ctr = (t >> 7, κ, t >> 39, 1)), DESIGN.md §3.3
      const u32x4 w = philox4x32_10((uint32_t)(tb >> 7), (uint32_t)kappa, (uint32_t)(tb >> 39),
                                    TAG_RADEMACHER, k0, k1);
      const uint32_t wi = (uint32_t)((tb >> 5) & 3);
      const uint32_t word = wi == 0 ? w.x : wi == 1 ? w.y : wi == 2 ? w.z : w.w;
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const int64_t t = tb + j;
        if (t >= t0 && t < t0 + rows) {
          const uint32_t pos = ((uint32_t)j >> 1) | (((uint32_t)j & 1u) << 4);
          pi[(t - t0) * kp + kappa] = ((word >> pos) & 1u) ? (uint16_t)0xBF80 : (uint16_t)0x3F80;
        }
      }
    } else {
      for (int j = 0; j < rpg; ++j) {
        const int64_t t = tb + j;
        if (t >= t0 && t < t0 + rows) pi[(t - t0) * kp + kappa] = pi_bits(kind, seed, (uint32_t)kappa, (uint64_t)t);
      }
    }
  }
}

// K3a' (Gaussian Π with a tensor-core head): one generation of a 64-row ×
// 32-κ tile written in BOTH layouts — row-major for the tail (pi[(t - t0) *
// kp + κ], κ < kp) and κ-major for K1's head panel (kmaj[κ * ld + t_off + t -
// t0], κ < kpad).  Thread (κ, 8-row group): two Philox calls give its 8
// consecutive rows, stored as one 16-byte κ-major vector; the row-major side
// goes through an SMEM tile (one 16-byte store per thread).  t0 % 4 == 0.
constexpr int DUAL_ROWS = 64, DUAL_K = 32;
__global__ void __launch_bounds__(256)
pi_panel_dual_kernel(uint64_t seed, int k, int kp, int kpad, int64_t t0, int rows, uint16_t* __restrict__ pi,
                     uint16_t* __restrict__ kmaj, int64_t ld, int64_t t_off) {
  __shared__ __align__(16) uint16_t tile[DUAL_ROWS][DUAL_K + 8];
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * DUAL_ROWS, c0 = blockIdx.y * DUAL_K;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  const int kq = tid & (DUAL_K - 1), rg = tid >> 5;  // κ within the tile, 8-row group 0..7
  const int kappa = c0 + kq;
  const int rt = r0 + 8 * rg;                        // first of the thread's 8 rows
  uint32_t z[4] = {0u, 0u, 0u, 0u};                  // bf16 pairs: rows (0,1), (2,3), (4,5), (6,7)
  if (kappa < k) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (rt + 4 * h < rows) {
        const uint64_t tq = (uint64_t)(t0 + rt + 4 * h) >> 2;
        const u32x4 w = philox4x32_10((uint32_t)tq, (uint32_t)kappa, (uint32_t)(tq >> 32), TAG_GAUSSIAN, k0, k1);
        z[2 * h] = gauss_pair_bits(w.x, w.y);
        z[2 * h + 1] = gauss_pair_bits(w.z, w.w);
      }
    }
  }
  // κ-major: 8 consecutive rows of one κ
  if (kmaj && kappa < kpad && rt < rows) {
    uint16_t* dst = kmaj + (int64_t)kappa * ld + t_off + rt;
    if (rt + 8 <= rows && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
      *reinterpret_cast<uint4*>(dst) = make_uint4(z[0], z[1], z[2], z[3]);
    } else {
      for (int j = 0; j < 8 && rt + j < rows; ++j) dst[j] = (uint16_t)(z[j >> 1] >> (16 * (j & 1)));
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) tile[8 * rg + j][kq] = (uint16_t)(z[j >> 1] >> (16 * (j & 1)));
  __syncthreads();
  // row-major: 64 rows x 32 κ, one 16-byte store (8 κ) per thread
  {
    const int r = tid >> 2, cq = (tid & 3) * 8;
    const int kb = c0 + cq;
    if (r0 + r < rows && kb < kp) {
      uint16_t* dst = pi + (int64_t)(r0 + r) * kp + kb;
      if (kb + 8 <= kp && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(&tile[r][cq]);
      } else {
        for (int j = 0; j < 8 && kb + j < kp; ++j) dst[j] = tile[r][cq + j];
      }
    }
  }
}

// ---------------------------------------------------------------- K3b
// kv[o] = (key << 32) | bits(v), key = (c_glob << tbits) | (t - p0), for the
// nonzeros of rows [p0, p0 + rows) of one matrix (the packed (value, key)
// pair K3d reads; a radix sort on bits [32, 32 + key bits) orders it); warp
// per row; o = (entry index relative to rowptr[0]) - ebase.
__global__ void csr_keys_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ col,
                                const float* __restrict__ val, int64_t p0, int rows,
                                int64_t ebase, uint32_t cofs, int tbits, int64_t ncols,
                                uint64_t* __restrict__ kv, int* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t base = rowptr[0];  // col/val are indexed from rowptr[0]
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += nw) {
    const int64_t e0 = rowptr[p0 + r] - base, e1 = rowptr[p0 + r + 1] - base;
    for (int64_t e = e0 + lane; e < e1; e += 32) {
      const int32_t c = col[e];
      if (c < 0 || c >= ncols) atomicOr(status, 2);  // out-of-range column
      const uint32_t cg = (uint32_t)(c < 0 ? 0 : (c >= ncols ? 0 : c)) + cofs;
      kv[e - ebase] = ((uint64_t)((cg << tbits) | (uint32_t)r) << 32) | __float_as_uint(val[e]);
    }
  }
}

// ---------------------------------------------------------------- K3d
#ifndef SMP_CSR_U
#define SMP_CSR_U 4
#endif
#ifndef SMP_CSR_CHUNK
#define SMP_CSR_CHUNK 128
#endif
constexpr int CSR_CHUNK = SMP_CSR_CHUNK;  // sorted nonzeros per warp task
constexpr int CSR_U = SMP_CSR_U;          // π rows in flight per lane

__device__ __forceinline__ void red_add_v4(float* addr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

template <int KV>
__device__ __forceinline__ void flush_col(uint32_t c, const float (&acc)[KV][8], double nrm, int k,
                                          float* __restrict__ acc_sk, double* __restrict__ acc_nrm,
                                          int lane, bool do_norms) {
  float* dst = acc_sk + (int64_t)c * k;
#pragma unroll
  for (int i = 0; i < KV; ++i) {
    const int kb = 8 * (lane + 32 * i);
    if ((k & 3) == 0) {
      if (kb < k) red_add_v4(dst + kb, acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
      if (kb + 4 < k) red_add_v4(dst + kb + 4, acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (kb + j < k) atomicAdd(dst + kb + j, acc[i][j]);
    }
  }
  // v² partials live in lanes 0..3 (fast path: lane u takes entry u of a group)
  nrm += __shfl_down_sync(0xFFFFFFFFu, nrm, 2);
  nrm += __shfl_down_sync(0xFFFFFFFFu, nrm, 1);
  if (do_norms && lane == 0) atomicAdd(acc_nrm + c, nrm);
}

// Warps take fixed chunks of CSR_CHUNK sorted entries; lanes own 8·KV κ
// (κ = 8·(lane + 32 i) .. +7), so the panel pitch kp is KV·256 (zero padded)
// and every π load is unconditional.  Entries are taken U at a time: the U
// (value, key) pairs are broadcast loads, their 2·KV π vectors are issued
// together, and when all U belong to the running column and carry
// bf16-exact values (integer counts) the group is 16·KV FHFMA.BF16 per entry
// with no per-entry branch; otherwise entries are taken one by one (column
// change -> flush, general fp32 values).  Lane u < U accumulates v² of entry
// u of each group (fp64); the lanes are summed at the flush.
template <int KV>
#ifndef SMP_CSR_ACC_U
#define SMP_CSR_ACC_U 4
#endif
struct AccU { static constexpr int U = KV <= 2 ? SMP_CSR_ACC_U : (KV <= 4 ? 2 : 1); };

#ifndef SMP_CSR_ACC_MINB
#define SMP_CSR_ACC_MINB 3  // (measured: 1 or 4 blocks per SM are 15-50% slower)
#endif
template <int KV>
__global__ void __launch_bounds__(256, KV <= 2 ? SMP_CSR_ACC_MINB : 1)
csr_accumulate_kernel(const uint2* __restrict__ kv, int64_t n,
                      const uint16_t* __restrict__ pi, int kp, int k, int tbits,
                      float* __restrict__ acc_sk, double* __restrict__ acc_nrm, int do_norms,
                      const uint32_t* __restrict__ seg_beg, const uint32_t* __restrict__ seg_end) {
  constexpr int U = AccU<KV>::U;
  // counting sort: the panel's tail is kv[*seg_beg (0 if null), *seg_end) (n bounds it)
  if (seg_end) {
    const int64_t b = seg_beg ? *seg_beg : 0;
    kv += b;
    n = min(n, (int64_t)*seg_end - b);
  }
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const uint32_t tmask = (1u << tbits) - 1u;
  const uint16_t* pil = pi + 8 * lane;
  for (int64_t task = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
       task * CSR_CHUNK < n; task += nw) {
    const int64_t e0 = task * CSR_CHUNK;
    const int64_t e1 = min(n, e0 + CSR_CHUNK);
    float acc[KV][8];
#pragma unroll
    for (int i = 0; i < KV; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
    double nrm = 0.0;
    uint32_t cur = __ldg(&kv[e0].y) >> tbits;
    for (int64_t eb = e0; eb < e1; eb += U) {
      const int cnt = (int)min((int64_t)U, e1 - eb);
      uint32_t kk[U], vb[U];
      uint4 q[U][KV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        // past the chunk end: repeat the last entry with value 0 (same column, adds nothing)
        const uint2 x = __ldg(&kv[eb + min(u, cnt - 1)]);
        kk[u] = x.y;
        vb[u] = u < cnt ? x.x : 0u;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint16_t* row = pil + (int64_t)(kk[u] & tmask) * kp;
#pragma unroll
        for (int i = 0; i < KV; ++i) q[u][i] = __ldg(reinterpret_cast<const uint4*>(row + 256 * i));
      }
      uint32_t low = 0;
#pragma unroll
      for (int u = 0; u < U; ++u) low |= vb[u];
      if ((kk[0] >> tbits) == cur && (kk[U - 1] >> tbits) == cur && (low & 0xFFFFu) == 0u) {
        // fast path: one column, bf16-exact values: v·π exact, FHFMA.BF16 without unpacking
#pragma unroll
        for (int u = 0; u < U; ++u) {
#pragma unroll
          for (int i = 0; i < KV; ++i) {
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].x, acc[i][0], acc[i][1]);
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].y, acc[i][2], acc[i][3]);
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].z, acc[i][4], acc[i][5]);
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].w, acc[i][6], acc[i][7]);
          }
        }
        if (lane < U) {
          uint32_t mine = vb[0];
#pragma unroll
          for (int u = 1; u < U; ++u) mine = lane == u ? vb[u] : mine;
          const double v = (double)__uint_as_float(mine);
          nrm = fma(v, v, nrm);
        }
        continue;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u >= cnt) break;
        const uint32_t c = kk[u] >> tbits;
        if (c != cur) {
          flush_col<KV>(cur, acc, nrm, k, acc_sk, acc_nrm, lane, do_norms != 0);
#pragma unroll
          for (int i = 0; i < KV; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
          nrm = 0.0;
          cur = c;
        }
        const float v = __uint_as_float(vb[u]);
        if (lane == 0) nrm = fma((double)v, (double)v, nrm);
        if ((vb[u] & 0xFFFFu) == 0u) {
#pragma unroll
          for (int i = 0; i < KV; ++i) {
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].x, acc[i][0], acc[i][1]);
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].y, acc[i][2], acc[i][3]);
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].z, acc[i][4], acc[i][5]);
            fma_bf16s_x2_f32(vb[u] >> 16, q[u][i].w, acc[i][6], acc[i][7]);
          }
        } else {
#pragma unroll
          for (int i = 0; i < KV; ++i) {
            const uint32_t w[4] = {q[u][i].x, q[u][i].y, q[u][i].z, q[u][i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              acc[i][2 * j] = fmaf(v, __uint_as_float(w[j] << 16), acc[i][2 * j]);
              acc[i][2 * j + 1] = fmaf(v, __uint_as_float(w[j] & 0xFFFF0000u), acc[i][2 * j + 1]);
            }
          }
        }
      }
    }
    flush_col<KV>(cur, acc, nrm, k, acc_sk, acc_nrm, lane, do_norms != 0);
  }
}

// ---------------------------------------------------------------- head/tail split
// A nonzero goes to the tensor-core head path iff its column is a head column
// (slot lut[c] != CSR_NO_SLOT) and its value has at most 4 significant bits
// (small integer counts): Gaussian Π (8 bits) times such a value is a 12-bit
// product, which tcgen05 accumulates exactly (R21).  Everything
// else is the tail.
constexpr uint16_t CSR_NO_SLOT = 0xFFFF;
__device__ __forceinline__ bool is_4bit(float v) {
  const uint32_t u = __float_as_uint(v);
  return ((u & 0x7F800000u) != 0x7F800000u) && ((u & 0x000FFFFFu) == 0u);
}

// ---------------------------------------------------------------- K3c counting sort
// One counting sort per GROUP of panels (up to ~2^27 entries) orders the
// nonzeros of the group's rows by (panel, column), so that every panel's tail
// is one contiguous, column-grouped range for K3d.  Each panel is cut into S
// row slices, one CTA per (panel, slice), about one CTA per SM over the
// group: the CTA counts its slice's tail entries per column in SMEM (hist
// pass; counts stored CTA-contiguous), a prefix over the slices of every
// (panel, column) cell plus one scan over the cells' totals give every CTA its
// own base per column, and the scatter pass claims positions from SMEM
// cursors.  A slice's entries are a contiguous range of each matrix, streamed
// coalesced with CSR_MLP loads in flight per thread (the row of an entry,
// needed by the scatter, by binary search in the slice's row offsets staged in
// SMEM); the head slot table sits in SMEM beside the counters.  In the
// scatter a tail entry costs one 8-byte (value, key) store.  Head entries
// (tensor-core path) are not counted; the scatter writes them straight into
// the dense head chunk, whose slice rows the CTA zeroes first (the
// densification of the head is fused into this pass).  The order inside one
// cell follows the SMEM atomics; K3d's fp32 sums are order-dependent anyway
// (DESIGN.md §7).
constexpr int CSR_T_THREADS = 1024;
#ifndef SMP_CSR_MLP
#define SMP_CSR_MLP 4
#endif
#ifndef SMP_CSR_PIPE
#define SMP_CSR_PIPE 1  // (4 pipelined: 0.91 ms per 12 panels; 8 unpipelined 0.98, 8 pipelined 1.05)
#endif
constexpr int CSR_MLP = SMP_CSR_MLP;  // CSR loads in flight per thread (sort passes)

// L2 eviction priorities: the CSR stream is read once (evict_first); the
// sorted (value, key) pairs are written in pieces by many CTAs over the whole
// pass and read back by K3d, so they are kept (evict_last) — a partially
// written 32-byte sector that leaves L2 early costs a DRAM read-modify-write.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int32_t ld_hint_s32(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ float ld_hint_f32(const float* p, uint64_t pol) {
  float v;
  asm volatile("ld.global.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint_v2(uint2* p, uint2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(p), "r"(v.x), "r"(v.y), "l"(pol)
               : "memory");
}


struct CsrSortArgs {
  const int64_t* arp;
  const int32_t* acol;
  const float* aval;
  int64_t a_n;
  const int64_t* brp;
  const int32_t* bcol;
  const float* bval;
  int64_t b_n;
  int64_t pr;               // rowptr index of the group's first row
  int rows;                 // group rows
  int tbits;                // panel rows = 2^tbits
  int ntot;
  int S;                    // slices (CTAs) per panel
  const uint16_t* lut;      // head slot per column (CSR_NO_SLOT: tail), or null
  int lut_smem;             // stage lut in SMEM
  uint32_t* cnt;            // [(p*S + s)*ntot + c]: hist counts; scatter: prefix over earlier slices
  const uint32_t* base;     // scatter: [p*ntot + c] start of cell (p, c) in kv
  uint2* kv;                // scatter: (value bits, key)
  int* status;
  uint16_t* xh;             // dense head chunk (null: no head)
  int64_t ldh, xrow;
  int n_head;
};

constexpr int CSR_SCATTER_RB = 64;        // scatter: rows per batch (head rows zeroed just before their values)
constexpr int CSR_ROWID_CAP = 24 * 1024;  // scatter: SMEM row ids of a batch's entries (else binary search)

// HEAD: 0 no head columns, 1 head slot table staged in SMEM, 2 read from global
template <bool SCATTER, int HEAD>
__global__ void __launch_bounds__(CSR_T_THREADS, 1) csr_sort_pass_kernel(CsrSortArgs a) {
  // SMEM: [ntot] counters | [ntot] u16 head slots (HEAD 1) | 2 x [nr+1] i32 row
  //       offsets (A, B) | scatter: [CSR_ROWID_CAP] u8 batch row of each entry of the batch (A then B)
  extern __shared__ uint32_t sm_cnt[];
  const int p = blockIdx.y, sl = blockIdx.x;
  const int pb = p << a.tbits;
  const int R = min(1 << a.tbits, a.rows - pb);
  const int r0 = pb + (int)(((int64_t)sl * R) / a.S), r1 = pb + (int)(((int64_t)(sl + 1) * R) / a.S);
  const int nr = r1 - r0;
  uint16_t* slut = reinterpret_cast<uint16_t*>(sm_cnt + a.ntot);
  int32_t* srp = reinterpret_cast<int32_t*>(sm_cnt + a.ntot + (HEAD == 1 ? (a.ntot + 1) / 2 : 0));
  uint8_t* rowid = reinterpret_cast<uint8_t*>(srp + 2 * (nr + 1));
  uint32_t* my_cnt = a.cnt + ((int64_t)p * a.S + sl) * a.ntot;
  const uint32_t* my_base = a.base + (int64_t)p * a.ntot;
  {  // counters (scatter: cursor = cell start + earlier slices) and head slots; 4 loads in flight
    for (int c0 = threadIdx.x; c0 < a.ntot; c0 += 4 * blockDim.x) {
      uint32_t x[4];
      uint16_t y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * blockDim.x;
        x[u] = (SCATTER && c < a.ntot) ? my_base[c] + my_cnt[c] : 0u;
        y[u] = (HEAD == 1 && c < a.ntot) ? a.lut[c] : CSR_NO_SLOT;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int c = c0 + u * blockDim.x;
        if (c < a.ntot) {
          sm_cnt[c] = x[u];
          if (HEAD == 1) slut[c] = y[u];
        }
      }
    }
  }
  const uint32_t tbits = (uint32_t)a.tbits, tmask = (1u << a.tbits) - 1u;
  const uint64_t pol_first = l2_policy_evict_first(), pol_last = l2_policy_evict_last();
  const int64_t e0a = a.arp[a.pr + r0] - a.arp[0];
  const int64_t e0b = a.brp ? a.brp[a.pr + r0] - a.brp[0] : 0;
  if (SCATTER) {  // slice row offsets of each matrix, relative to its first entry
    for (int i = threadIdx.x; i <= nr; i += blockDim.x) {
      srp[i] = (int32_t)(a.arp[a.pr + r0 + i] - a.arp[0] - e0a);
      srp[nr + 1 + i] = a.brp ? (int32_t)(a.brp[a.pr + r0 + i] - a.brp[0] - e0b) : 0;
    }
  }
  __syncthreads();
  uint16_t* xh = (SCATTER && HEAD != 0) ? a.xh : nullptr;
  const int nq = (a.n_head + 7) / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int ncols_a = (int)a.a_n, ncols_b = (int)a.b_n;  // counting mode: ntot < 2^16
  uint2* kvp = a.kv;
  // hist: the whole slice in one batch; scatter: batches of at most
  // CSR_SCATTER_RB rows and CSR_ROWID_CAP entries (a longer row is a batch of its own)
  for (int rb = 0; rb < nr;) {
    int re = nr;
    if (SCATTER) {  // largest re <= rb + RB with the batch's entries <= CAP (uniform search)
      int lo = rb + 1, hi = min(nr, rb + CSR_SCATTER_RB);
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((srp[mid] - srp[rb]) + (srp[nr + 1 + mid] - srp[nr + 1 + rb]) <= CSR_ROWID_CAP) lo = mid;
        else hi = mid - 1;
      }
      re = lo;
    }
    const int32_t nba = SCATTER ? srp[re] - srp[rb] : 0;
    const bool single = SCATTER && re == rb + 1;  // one row: no row ids needed
    uint16_t* xb = xh ? xh + ((int64_t)(r0 + rb) + a.xrow) * a.ldh : nullptr;  // the batch's first head row
    if (SCATTER) {
      // row ids of the batch's entries (warp per row), and the head slots of
      // the batch's rows zeroed (coalesced) just before their values
      for (int rr = rb + warp; rr < re; rr += nwarp) {
        if (xb) {
          uint4* row = reinterpret_cast<uint4*>(xb + (int64_t)(rr - rb) * a.ldh);
          for (int q = lane; q < nq; q += 32) row[q] = make_uint4(0u, 0u, 0u, 0u);
        }
        if (!single) {
          for (int e = srp[rr] + lane; e < srp[rr + 1]; e += 32) rowid[e - srp[rb]] = (uint8_t)(rr - rb);
          for (int e = srp[nr + 1 + rr] + lane; e < srp[nr + 1 + rr + 1]; e += 32)
            rowid[nba + e - srp[nr + 1 + rb]] = (uint8_t)(rr - rb);
        }
      }
      __syncthreads();
    }
#pragma unroll 1
    for (int mat = 0; mat < 2; ++mat) {
      const int64_t* rp = mat == 0 ? a.arp : a.brp;
      if (!rp) continue;
      const int64_t e0 = mat == 0 ? e0a : e0b;
      const int32_t* col = (mat == 0 ? a.acol : a.bcol) + e0;
      const float* val = (mat == 0 ? a.aval : a.bval) + e0;
      const int ncols = mat == 0 ? ncols_a : ncols_b;
      const uint32_t cofs = mat == 0 ? 0u : (uint32_t)a.a_n;
      const int32_t* mrp = srp + mat * (nr + 1);
      const int32_t eb0 = SCATTER ? mrp[rb] : 0;
      const int32_t eb1 = SCATTER ? mrp[re] : (int32_t)(rp[a.pr + r1] - rp[0] - e0);
      const uint8_t* mid8 = rowid + (mat == 0 ? 0 : nba) - eb0;  // batch row of entry e: mid8[e]
#if SMP_CSR_PIPE
      // software-pipelined: the next group's loads are issued before this
      // group's entries are processed
      int32_t cn[CSR_MLP];
      float vn[CSR_MLP];
#pragma unroll
      for (int u = 0; u < CSR_MLP; ++u) {
        const int32_t e = eb0 + (int32_t)threadIdx.x + u * (int32_t)blockDim.x;
        cn[u] = e < eb1 ? ld_hint_s32(col + e, pol_first) : 0;
        vn[u] = e < eb1 ? ld_hint_f32(val + e, pol_first) : 0.f;
      }
#endif
      for (int32_t eb = eb0 + (int32_t)threadIdx.x; eb < eb1; eb += CSR_MLP * (int32_t)blockDim.x) {
        int32_t c[CSR_MLP];
        float v[CSR_MLP];
#pragma unroll
        for (int u = 0; u < CSR_MLP; ++u) {
#if SMP_CSR_PIPE
          c[u] = cn[u];
          v[u] = vn[u];
          const int32_t e = eb + (CSR_MLP + u) * (int32_t)blockDim.x;
          cn[u] = e < eb1 ? ld_hint_s32(col + e, pol_first) : 0;
          vn[u] = e < eb1 ? ld_hint_f32(val + e, pol_first) : 0.f;
#else
          const int32_t e = eb + u * (int32_t)blockDim.x;
          c[u] = e < eb1 ? ld_hint_s32(col + e, pol_first) : 0;
          v[u] = e < eb1 ? ld_hint_f32(val + e, pol_first) : 0.f;
#endif
        }
#pragma unroll
        for (int u = 0; u < CSR_MLP; ++u) {
          const int32_t e = eb + u * (int32_t)blockDim.x;
          if (e >= eb1) continue;
          const bool bad = c[u] < 0 || c[u] >= ncols;
          if (SCATTER && bad) atomicOr(a.status, 2);  // out-of-range column
          const uint32_t cg = (uint32_t)(bad ? 0 : c[u]) + cofs;
          bool head = false;
          uint32_t slot = 0;
          if (HEAD != 0) {
            slot = HEAD == 1 ? slut[cg] : __ldg(a.lut + cg);
            head = slot != CSR_NO_SLOT && is_4bit(v[u]);
          }
          if (!SCATTER) {
            if (!head) atomicAdd(&sm_cnt[cg], 1u);
            continue;
          }
          const uint32_t lo = single ? 0u : (uint32_t)mid8[e];  // row within the batch
          if (head) {
            if (xb) xb[lo * (uint32_t)a.ldh + slot] = (uint16_t)(__float_as_uint(v[u]) >> 16);
          } else {
            const uint32_t pos = atomicAdd(&sm_cnt[cg], 1u);
            st_hint_v2(kvp + pos, make_uint2(__float_as_uint(v[u]), (cg << tbits) | ((uint32_t)(r0 + rb) + lo) & tmask),
                       pol_last);
          }
        }
      }
    }
    if (SCATTER) __syncthreads();  // row ids and head rows reused by the next batch
    rb = re;
  }
  if (!SCATTER) {
    __syncthreads();
    for (int c = threadIdx.x; c < a.ntot; c += blockDim.x) my_cnt[c] = sm_cnt[c];
  }
}

// per cell (p, c): cnt[(p*S + s)*ntot + c] <- Σ_{s' < s} (in place), tot[p*ntot + c] = Σ_s.
// Block (32 columns x 32 slice groups) per (p, 32-column chunk): each thread
// sums its group's slices, a 32-step SMEM scan over the groups, then the
// in-place prefixes (all loads of a thread in flight at once).
constexpr int SLICE_SCAN_G = 32;
__global__ void __launch_bounds__(1024) csr_slice_scan_kernel(uint32_t* __restrict__ cnt, int gp, int S, int ntot,
                                                             uint32_t* __restrict__ tot) {
  __shared__ uint32_t part[SLICE_SCAN_G][33];
  const int cchunks = (ntot + 31) / 32;
  const int p = blockIdx.x / cchunks, c = (blockIdx.x % cchunks) * 32 + threadIdx.x;
  const int g = threadIdx.y;
  const int per = (S + SLICE_SCAN_G - 1) / SLICE_SCAN_G;  // slices per group (<= 8 for S <= 256)
  const int s0 = g * per, s1 = min(S, s0 + per);
  uint32_t* q = cnt + (int64_t)p * S * ntot + c;
  uint32_t v[8];
  uint32_t sum = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    v[u] = (c < ntot && s0 + u < s1) ? q[(int64_t)(s0 + u) * ntot] : 0u;
    sum += v[u];
  }
  part[g][threadIdx.x] = sum;
  __syncthreads();
  if (g == 0) {
    uint32_t run = 0;
    for (int i = 0; i < SLICE_SCAN_G; ++i) {
      const uint32_t t = part[i][threadIdx.x];
      part[i][threadIdx.x] = run;
      run += t;
    }
    if (c < ntot) tot[(int64_t)p * ntot + c] = run;
  }
  __syncthreads();
  uint32_t run = part[g][threadIdx.x];
  if (c < ntot) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (s0 + u < s1) {
        q[(int64_t)(s0 + u) * ntot] = run;
        run += v[u];
      }
  }
}

constexpr int CSR_HIST_CTAS = 148;
constexpr int CSR_HIST_MAX_COLS = 40960;  // 160 KB of SMEM counters (+ row ids, row offsets)

template <class T>
static cudaError_t grow(T*& p, int64_t& cap, int64_t need) {
  if (need <= cap) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, (size_t)(need > 0 ? need : 1) * sizeof(T));
  if (e == cudaSuccess) cap = need;
  return e;
}

#define CSR_TRY(x)                    \
  do {                                \
    cudaError_t e_ = (x);             \
    if (e_ != cudaSuccess) return e_; \
  } while (0)

// ---------------------------------------------------------------- tensor-core head
// CTA b owns block rows [b·rows/G, (b+1)·rows/G)
__device__ __forceinline__ void cta_rows(int rows, int& r0, int& r1) {
  r0 = (int)(((int64_t)blockIdx.x * rows) / gridDim.x);
  r1 = (int)(((int64_t)(blockIdx.x + 1) * rows) / gridDim.x);
}

// column counts over a row sample of the block (global column index: A then
// B): the sample is `segs` segments of `seg` rows spaced evenly over the block
// (virtual row v -> block row (v / seg)·stride + v % seg); all rows when the
// block is small.  The head choice only routes columns between two exact
// paths, so a sample serves (K3).
__global__ void __launch_bounds__(CSR_T_THREADS)
csr_colcount_kernel(const int64_t* __restrict__ arp, const int32_t* __restrict__ acol, int64_t a_n,
                    const int64_t* __restrict__ brp, const int32_t* __restrict__ bcol, int64_t b_n,
                    int vrows, int seg, int64_t stride, int ntot, uint32_t* __restrict__ cnt) {
  extern __shared__ uint32_t hist[];
  for (int c = threadIdx.x; c < ntot; c += blockDim.x) hist[c] = 0u;
  __syncthreads();
  int r0, r1;
  cta_rows(vrows, r0, r1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int mat = 0; mat < 2; ++mat) {
    const int64_t* rp = mat == 0 ? arp : brp;
    if (!rp) continue;
    const int32_t* col = mat == 0 ? acol : bcol;
    const int64_t ncols = mat == 0 ? a_n : b_n;
    const uint32_t cofs = mat == 0 ? 0u : (uint32_t)a_n;
    const int64_t base = rp[0];
    for (int v = r0 + warp; v < r1; v += nw) {
      const int64_t r = (int64_t)(v / seg) * stride + v % seg;
      const int64_t e0 = rp[r] - base, e1 = rp[r + 1] - base;
      for (int64_t eb = e0 + lane; eb < e1; eb += 128) {
        int32_t c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) c[u] = eb + 32 * u < e1 ? col[eb + 32 * u] : -1;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (eb + 32 * u < e1 && c[u] >= 0 && c[u] < ncols) atomicAdd(&hist[(uint32_t)c[u] + cofs], 1u);
      }
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < ntot; c += blockDim.x)
    if (hist[c]) atomicAdd(&cnt[c], hist[c]);
}

__global__ void csr_head_flag_kernel(const uint32_t* __restrict__ cnt, int ntot, uint32_t thr,
                                     uint32_t* __restrict__ flag) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ntot; c += gridDim.x * blockDim.x)
    flag[c] = cnt[c] >= thr ? 1u : 0u;
}

// slot = exclusive scan of the flags (column order: deterministic)
__global__ void csr_head_map_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ scan,
                                    int ntot, uint16_t* __restrict__ lut, int32_t* __restrict__ map,
                                    uint32_t* __restrict__ total) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ntot; c += gridDim.x * blockDim.x) {
    // slots < ntot <= CSR_HIST_MAX_COLS < 0xFFFF
    lut[c] = flag[c] ? (uint16_t)scan[c] : CSR_NO_SLOT;
    if (flag[c]) map[scan[c]] = c;
    if (c == ntot - 1) *total = scan[c] + flag[c];
  }
}

cudaError_t csr_select_head(CsrWorkspace& w, const int64_t* a_rowptr, const int32_t* a_col, int64_t a_n,
                            const int64_t* b_rowptr, const int32_t* b_col, int64_t b_n, int64_t rows,
                            double density, int* n_head, cudaStream_t st) {
  *n_head = 0;
  const int64_t ntot = a_n + (b_rowptr ? b_n : 0);
  if (ntot > CSR_HIST_MAX_COLS || rows <= 0 || rows >= (1ll << 31)) return cudaSuccess;
  CSR_TRY(grow(w.head_cnt, w.head_cnt_cap, ntot));
  CSR_TRY(grow(w.head_flag, w.head_flag_cap, 2 * ntot));
  CSR_TRY(grow(w.head_lut, w.head_lut_cap, ntot));
  CSR_TRY(grow(w.head_map, w.head_map_cap, ntot));
  CSR_TRY(cudaMemsetAsync(w.head_cnt, 0, ntot * 4, st));
  static PerDeviceOnce attr;
  if (attr.need())
    CSR_TRY(cudaFuncSetAttribute(csr_colcount_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 CSR_HIST_MAX_COLS * 4));
  // row sample: 64 segments of 4096 rows (all rows up to 2^18)
  const int seg = 4096, segs = 64;
  const bool sample = rows > (int64_t)seg * segs;
  const int vrows = sample ? seg * segs : (int)rows;
  const int64_t stride = sample ? rows / segs : seg;
  csr_colcount_kernel<<<148, CSR_T_THREADS, ntot * 4, st>>>(a_rowptr, a_col, a_n, b_rowptr, b_col, b_n,
                                                           vrows, sample ? seg : (int)rows, sample ? stride : 0,
                                                           (int)ntot, w.head_cnt);
  const uint32_t thr = (uint32_t)std::max(1.0, std::ceil(density * (double)vrows));
  const int blocks = (int)((ntot + 255) / 256);
  csr_head_flag_kernel<<<blocks, 256, 0, st>>>(w.head_cnt, (int)ntot, thr, w.head_flag);
  size_t need = 0;
  CSR_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, w.head_flag, w.head_flag + ntot, (int)ntot, st));
  CSR_TRY(grow(w.head_tmp, w.head_tmp_cap, (int64_t)need));
  size_t tmp = (size_t)w.head_tmp_cap;
  CSR_TRY(cub::DeviceScan::ExclusiveSum(w.head_tmp, tmp, w.head_flag, w.head_flag + ntot, (int)ntot, st));
  CSR_TRY(grow(w.ne_dev, w.ne_cap, 2));
  csr_head_map_kernel<<<blocks, 256, 0, st>>>(w.head_flag, w.head_flag + ntot, (int)ntot, w.head_lut,
                                              w.head_map, w.ne_dev + 1);
  if (!w.head_h) CSR_TRY(cudaMallocHost(&w.head_h, 8));
  CSR_TRY(cudaMemcpyAsync(w.head_h, w.ne_dev + 1, 4, cudaMemcpyDeviceToHost, st));
  CSR_TRY(cudaStreamSynchronize(st));
  *n_head = (int)*reinterpret_cast<uint32_t*>(w.head_h);
  w.launches += 5;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- driver
__global__ void csr_bounds_kernel(const int64_t* __restrict__ arp, const int64_t* __restrict__ brp,
                                  int64_t rbase, int rows, int rp, int npan, int64_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= npan; i += gridDim.x * blockDim.x) {
    const int64_t r = rbase + (i < npan ? (int64_t)i * rp : rows);
    out[i] = arp[r] - arp[0];
    out[npan + 1 + i] = brp ? brp[r] - brp[0] : 0;
  }
}

// out[κ · ld + t_off + t] = pi[t · kp + κ] (κ < k; zero for k <= κ < kpad):
// the row-major K3 panel transposed into the κ-major layout K1 (PANEL) reads,
// so the head and the tail of the CSR sketch share one generation of Π.
__global__ void pi_transpose_kernel(const uint16_t* __restrict__ pi, int kp, int k, int prow, int kpad,
                                    uint16_t* __restrict__ out, int64_t ld, int64_t t_off) {
  __shared__ uint16_t tile[64][66];
  const int t0 = blockIdx.x * 64, c0 = blockIdx.y * 64;
  for (int i = threadIdx.y; i < 64; i += blockDim.y)
    for (int j = threadIdx.x; j < 64; j += blockDim.x) {
      const int t = t0 + i, c = c0 + j;
      tile[i][j] = (t < prow && c < k) ? pi[(int64_t)t * kp + c] : (uint16_t)0;
    }
  __syncthreads();
  for (int i = threadIdx.y; i < 64; i += blockDim.y)
    for (int j = threadIdx.x; j < 64; j += blockDim.x) {
      const int c = c0 + i, t = t0 + j;
      if (c < kpad && t < prow) out[(int64_t)c * ld + t_off + t] = tile[j][i];
    }
}

void csr_workspace_free(CsrWorkspace& w) {
  cudaFree(w.pi); cudaFree(w.kv_in); cudaFree(w.kv_out); cudaFree(w.cub_tmp); cudaFree(w.bounds_d); cudaFree(w.hist); cudaFree(w.offs);
  cudaFree(w.ne_dev); cudaFree(w.head_lut); cudaFree(w.head_map); cudaFree(w.head_cnt); cudaFree(w.head_flag);
  cudaFree(w.xhead); cudaFree(w.head_tmp); cudaFree(w.kmaj); cudaFree(w.xhead1); cudaFree(w.kmaj1);
  for (int b = 0; b < 2; ++b) {
    if (w.ev_tail[b]) cudaEventDestroy(w.ev_tail[b]);
    if (w.ev_head[b]) cudaEventDestroy(w.ev_head[b]);
  }
  if (w.head_h) cudaFreeHost(w.head_h);
  if (w.bounds_h) cudaFreeHost(w.bounds_h);
  w = CsrWorkspace{};
}

static int bits_for(int64_t x) {  // smallest b with 2^b > x
  int b = 0;
  while (b < 62 && ((int64_t)1 << b) <= x) ++b;
  return b;
}

// panel rows = 2^tbits: the 32-bit sort key packs (column << tbits | row);
// at most 2^15 rows (a 32 MB bf16 Π panel at k = 512 stays L2-resident);
// SMP_CSR_PANEL_BITS lowers the cap (tuning only)
static int csr_tbits_cap() {
  const char* e = getenv("SMP_CSR_PANEL_BITS");
  const int v = e ? atoi(e) : 15;  // (values up to 17 accepted for experiments)
  return std::max(8, std::min(17, v));
}

int csr_panel_rows(int64_t ntot) {
  const int cbits = bits_for(ntot - 1 > 0 ? ntot - 1 : 1);
  return 1 << std::max(0, std::min(csr_tbits_cap(), 32 - cbits));
}

cudaError_t csr_bounds(CsrWorkspace& w, const int64_t* a_rowptr, const int64_t* b_rowptr, int64_t ntot,
                       int64_t rows, cudaStream_t st) {
  const int rp = csr_panel_rows(ntot);
  const int npan = (int)((rows + rp - 1) / rp);
  CSR_TRY(grow(w.bounds_d, w.bounds_cap, 2 * (int64_t)(npan + 1)));
  if (w.bounds_hcap < 2 * (int64_t)(npan + 1)) {
    if (w.bounds_h) cudaFreeHost(w.bounds_h);
    w.bounds_h = nullptr;
    w.bounds_hcap = 0;
    CSR_TRY(cudaMallocHost(&w.bounds_h, 2 * (size_t)(npan + 1) * 8));
    w.bounds_hcap = 2 * (int64_t)(npan + 1);
  }
  csr_bounds_kernel<<<(npan + 256) / 256, 256, 0, st>>>(a_rowptr, b_rowptr, 0, (int)rows, rp, npan, w.bounds_d);
  CSR_TRY(cudaMemcpyAsync(w.bounds_h, w.bounds_d, 2 * (size_t)(npan + 1) * 8, cudaMemcpyDeviceToHost, st));
  CSR_TRY(cudaStreamSynchronize(st));
  w.bounds_npan = npan;
  w.bounds_rp = rp;
  w.bounds_pre = true;
  return cudaSuccess;
}


cudaError_t launch_sketch_csr(CsrWorkspace& w, int kind, uint64_t seed, int k, int64_t row0,
                              int64_t rows, const int64_t* a_rowptr, const int32_t* a_col,
                              const float* a_val, int64_t a_n, const int64_t* b_rowptr,
                              const int32_t* b_col, const float* b_val, int64_t b_n, float* acc_sk,
                              double* acc_nrm, int* status, cudaStream_t st, const uint16_t* head_lut,
                              int64_t rbase, uint16_t* kmaj, int64_t kmaj_ld, int kpad, uint16_t* xh,
                              int64_t ldh, int n_head) {
  if (rows <= 0) return cudaSuccess;
  const int64_t ntot = a_n + (b_rowptr ? b_n : 0);
  const int cbits = bits_for(ntot - 1 > 0 ? ntot - 1 : 1);
  if (cbits > 31) return cudaErrorInvalidValue;
  const int tbits = std::min(csr_tbits_cap(), 32 - cbits);
  if (tbits < 6) return cudaErrorInvalidValue;  // more than 2^26 columns
  const int rp = 1 << tbits;                      // panel rows
  // Π panel pitch: the κ slices of K3d's lanes, 256·KV with KV in {1, 2, 4, 8, 16} (zero padded)
  const int kvt = k <= 256 ? 1 : k <= 512 ? 2 : k <= 1024 ? 4 : k <= 2048 ? 8 : 16;
  const int kp = 256 * kvt;
  const int npan = (int)((rows + rp - 1) / rp);
  const int64_t* ab;
  const int64_t* bb;
  if (w.bounds_pre) {
    // boundaries of the whole block, read back once by csr_bounds()
    if (rbase % rp != 0 || w.bounds_rp != rp) return cudaErrorInvalidValue;
    const int64_t pb = rbase / rp;
    ab = w.bounds_h + pb;
    bb = w.bounds_h + (w.bounds_npan + 1) + pb;
  } else {
    // panel entry boundaries (one D2H read per call)
    CSR_TRY(grow(w.bounds_d, w.bounds_cap, 2 * (int64_t)(npan + 1)));
    if (w.bounds_hcap < 2 * (int64_t)(npan + 1)) {
      if (w.bounds_h) cudaFreeHost(w.bounds_h);
      w.bounds_h = nullptr;
      w.bounds_hcap = 0;
      CSR_TRY(cudaMallocHost(&w.bounds_h, 2 * (size_t)(npan + 1) * 8));
      w.bounds_hcap = 2 * (int64_t)(npan + 1);
    }
    csr_bounds_kernel<<<(npan + 256) / 256, 256, 0, st>>>(a_rowptr, b_rowptr, rbase, (int)rows, rp, npan,
                                                         w.bounds_d);
    CSR_TRY(cudaMemcpyAsync(w.bounds_h, w.bounds_d, 2 * (size_t)(npan + 1) * 8, cudaMemcpyDeviceToHost, st));
    CSR_TRY(cudaStreamSynchronize(st));
    ab = w.bounds_h;
    bb = w.bounds_h + npan + 1;
  }
  int64_t max_ent = 0;
  for (int p = 0; p < npan; ++p) max_ent = std::max(max_ent, (ab[p + 1] - ab[p]) + (bb[p + 1] - bb[p]));
  CSR_TRY(grow(w.pi, w.pi_cap, (int64_t)rp * kp));
  const int end_bit = tbits + cbits;
  const bool counting = ntot <= CSR_HIST_MAX_COLS;
  if (!counting) head_lut = nullptr;  // (the caller only selects heads when counting)
  if (!counting) xh = nullptr;
  // diagnostics (SMP_CSR_PROFILE=1): device time per K3 stage, summed over
  // panels — one event per stage boundary, read after the last (no syncs)
  const char* prof_env = getenv("SMP_CSR_PROFILE");
  const bool prof = prof_env && atoi(prof_env);
  std::vector<std::pair<cudaEvent_t, int>> pev;  // (event, slot of the stage it ends)
  float pms[3] = {0.f, 0.f, 0.f};  // sort (+ fused head densify), Π panel, accumulate
  auto lap = [&](int slot) -> cudaError_t {
    if (!prof) return cudaSuccess;
    cudaEvent_t e;
    CSR_TRY(cudaEventCreate(&e));
    CSR_TRY(cudaEventRecord(e, st));
    pev.emplace_back(e, slot);
    return cudaSuccess;
  };
  auto gen_panel = [&](int p, int prow) {
    const int64_t p0 = (int64_t)p * rp;
    if (kind == PI_GAUSSIAN && ((row0 + p0) & 3) == 0 && (kp & 1) == 0) {
      // one generation, both layouts (the head panel when kmaj is given)
      const int kcols = std::max(kp, kmaj ? kpad : 0);
      dim3 dg((unsigned)((prow + DUAL_ROWS - 1) / DUAL_ROWS), (unsigned)((kcols + DUAL_K - 1) / DUAL_K));
      pi_panel_dual_kernel<<<dg, 256, 0, st>>>(seed, k, kp, kmaj ? kpad : 0, row0 + p0, prow, w.pi, kmaj,
                                               kmaj_ld, p0);
    } else {
      const int64_t groups = ((row0 + p0 + prow - 1) / 4 - (row0 + p0) / 4 + 1) * kp;
      const int blocks = (int)std::min<int64_t>((groups + 255) / 256, 148 * 16);
      pi_panel_kernel<<<blocks, 256, 0, st>>>(kind, seed, k, kp, row0 + p0, prow, w.pi);
      if (kmaj) {
        dim3 tg((unsigned)((prow + 63) / 64), (unsigned)((kpad + 63) / 64));
        pi_transpose_kernel<<<tg, dim3(32, 8), 0, st>>>(w.pi, kp, k, prow, kpad, kmaj, kmaj_ld, p0);
        w.launches += 1;
      }
    }
    w.launches += 1;
  };
  auto accumulate = [&](int64_t ne, const uint32_t* sb, const uint32_t* se) -> cudaError_t {
    const int64_t tasks = (ne + CSR_CHUNK - 1) / CSR_CHUNK;
    const int ablocks = (int)std::max<int64_t>(1, std::min<int64_t>((tasks + 7) / 8, 148 * 64));
    const int kvw = kvt;
    const uint2* kv = reinterpret_cast<const uint2*>(w.kv_out);
    if (w.ev_pool) {
      while (w.ev_pool->size() < *w.ev_used + 2) {
        cudaEvent_t ev;
        CSR_TRY(cudaEventCreate(&ev));
        w.ev_pool->push_back(ev);
      }
      CSR_TRY(cudaEventRecord((*w.ev_pool)[*w.ev_used], st));
    }
    switch (kvw) {
      case 1: csr_accumulate_kernel<1><<<ablocks, 256, 0, st>>>(kv, ne, w.pi, kp, k, tbits, acc_sk, acc_nrm, 1, sb, se); break;
      case 2: csr_accumulate_kernel<2><<<ablocks, 256, 0, st>>>(kv, ne, w.pi, kp, k, tbits, acc_sk, acc_nrm, 1, sb, se); break;
      case 3: case 4: csr_accumulate_kernel<4><<<ablocks, 256, 0, st>>>(kv, ne, w.pi, kp, k, tbits, acc_sk, acc_nrm, 1, sb, se); break;
      case 5: case 6: case 7: case 8: csr_accumulate_kernel<8><<<ablocks, 256, 0, st>>>(kv, ne, w.pi, kp, k, tbits, acc_sk, acc_nrm, 1, sb, se); break;
      default: csr_accumulate_kernel<16><<<ablocks, 256, 0, st>>>(kv, ne, w.pi, kp, k, tbits, acc_sk, acc_nrm, 1, sb, se); break;
    }
    CSR_TRY(cudaGetLastError());
    if (w.ev_pool) {
      CSR_TRY(cudaEventRecord((*w.ev_pool)[*w.ev_used + 1], st));
      *w.ev_used += 2;
    }
    w.launches += 1;
    return cudaSuccess;
  };
  CSR_TRY(grow(w.pi, w.pi_cap, (int64_t)rp * kp));
  CSR_TRY(lap(-1));
  if (counting) {
    // groups of consecutive panels with at most max(2^24, largest panel)
    // entries: the group's sorted tail (8 B per entry) then stays L2-resident
    // between the scatter and K3d
    const int64_t cap = std::max<int64_t>(max_ent, 1ll << 24);
    int gmax = 1;
    for (int g0 = 0; g0 < npan;) {
      int g1 = g0 + 1;
      while (g1 < npan && (ab[g1 + 1] - ab[g0]) + (bb[g1 + 1] - bb[g0]) <= cap) ++g1;
      gmax = std::max(gmax, g1 - g0);
      g0 = g1;
    }
    // slices per panel: about one CTA per SM over the group, at most max_nr rows each
    int dev = 0, nsm = 148;
    CSR_TRY(cudaGetDevice(&dev));
    CSR_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    // SMEM: counters (4 B) + head slots (2 B) per column when they fit + slice row offsets
    const bool lut_smem = head_lut && ntot * 6 <= 160 * 1024;
    const int64_t fixed = ntot * 4 + (lut_smem ? ((ntot + 1) / 2) * 4 : 0);
    const int max_nr = (int)std::min<int64_t>(rp, (227 * 1024 - CSR_ROWID_CAP - fixed) / 8 - 2);
    if (max_nr < 64) return cudaErrorInvalidValue;
    auto slices = [&](int gp) { return std::max({1, nsm / gp, (rp + max_nr - 1) / max_nr}); };  // <= 256 (slice scan)
    if (slices(1) > 8 * SLICE_SCAN_G) return cudaErrorInvalidValue;
    int64_t cells_max = 1;
    for (int g = 1; g <= gmax; ++g) cells_max = std::max<int64_t>(cells_max, (int64_t)g * ntot * slices(g));
    const size_t smem_rows = (size_t)(std::min(rp, (rp + slices(gmax) - 1) / slices(gmax) + 1) + 1) * 8;
    const size_t smem = (size_t)fixed + smem_rows;
    const size_t smem_sc = smem + CSR_ROWID_CAP;
    CSR_TRY(grow(w.kv_out, w.ent_cap_ko, cap));
    CSR_TRY(grow(w.hist, w.hist_cap, cells_max));                 // per-slice counts / prefixes
    CSR_TRY(grow(w.offs, w.offs_cap, 2 * ((int64_t)gmax * ntot + 1)));  // cell totals | cell starts
    size_t need = 0;
    CSR_TRY(cub::DeviceScan::ExclusiveSum(nullptr, need, w.offs, w.offs, (int)((int64_t)gmax * ntot + 1), st));
    CSR_TRY(grow(w.cub_tmp, w.cub_cap, (int64_t)need));
    static PerDeviceOnce attr;
    if (attr.need()) {
      const int mx = 227 * 1024;
      CSR_TRY(cudaFuncSetAttribute(csr_sort_pass_kernel<false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      CSR_TRY(cudaFuncSetAttribute(csr_sort_pass_kernel<false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      CSR_TRY(cudaFuncSetAttribute(csr_sort_pass_kernel<false, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      CSR_TRY(cudaFuncSetAttribute(csr_sort_pass_kernel<true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      CSR_TRY(cudaFuncSetAttribute(csr_sort_pass_kernel<true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
      CSR_TRY(cudaFuncSetAttribute(csr_sort_pass_kernel<true, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    }
    const int head_mode = !head_lut ? 0 : (lut_smem ? 1 : 2);
    for (int g0 = 0; g0 < npan;) {
      int g1 = g0 + 1;
      while (g1 < npan && (ab[g1 + 1] - ab[g0]) + (bb[g1 + 1] - bb[g0]) <= cap) ++g1;
      const int gp = g1 - g0;
      const int64_t r0g = (int64_t)g0 * rp;
      const int grows = (int)(std::min<int64_t>((int64_t)g1 * rp, rows) - r0g);
      if ((ab[g1] - ab[g0]) + (bb[g1] - bb[g0]) > 0) {
        CsrSortArgs sa{};
        sa.arp = a_rowptr; sa.acol = a_col; sa.aval = a_val; sa.a_n = a_n;
        sa.brp = b_rowptr; sa.bcol = b_col; sa.bval = b_val; sa.b_n = b_n;
        sa.pr = rbase + r0g;
        sa.rows = grows;
        sa.tbits = tbits;
        sa.ntot = (int)ntot;
        sa.S = slices(gp);
        sa.lut = head_lut;
        sa.lut_smem = lut_smem ? 1 : 0;
        sa.status = status;
        sa.xh = xh;
        sa.ldh = ldh;
        sa.xrow = r0g;
        sa.n_head = n_head;
        const int64_t pc = (int64_t)gp * ntot;  // (panel, column) cells
        uint32_t* tot = w.offs;
        uint32_t* start = w.offs + pc + 1;
        dim3 grid((unsigned)sa.S, (unsigned)gp);
        sa.cnt = w.hist;
        sa.base = start;
        switch (head_mode) {
          case 0: csr_sort_pass_kernel<false, 0><<<grid, CSR_T_THREADS, smem, st>>>(sa); break;
          case 1: csr_sort_pass_kernel<false, 1><<<grid, CSR_T_THREADS, smem, st>>>(sa); break;
          default: csr_sort_pass_kernel<false, 2><<<grid, CSR_T_THREADS, smem, st>>>(sa); break;
        }
        csr_slice_scan_kernel<<<(unsigned)(gp * ((ntot + 31) / 32)), dim3(32, SLICE_SCAN_G), 0, st>>>(
            w.hist, gp, sa.S, (int)ntot, tot);
        CSR_TRY(cudaMemsetAsync(tot + pc, 0, 4, st));  // start[pc] = total
        size_t tmp = (size_t)w.cub_cap;
        CSR_TRY(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tmp, tot, start, (int)(pc + 1), st));
        sa.kv = reinterpret_cast<uint2*>(w.kv_out);
        switch (head_mode) {
          case 0: csr_sort_pass_kernel<true, 0><<<grid, CSR_T_THREADS, smem_sc, st>>>(sa); break;
          case 1: csr_sort_pass_kernel<true, 1><<<grid, CSR_T_THREADS, smem_sc, st>>>(sa); break;
          default: csr_sort_pass_kernel<true, 2><<<grid, CSR_T_THREADS, smem_sc, st>>>(sa); break;
        }
        CSR_TRY(cudaGetLastError());
        w.launches += 5;
        CSR_TRY(lap(0));
        for (int p = g0; p < g1; ++p) {
          const int prow = (int)std::min<int64_t>(rp, rows - (int64_t)p * rp);
          gen_panel(p, prow);
          CSR_TRY(lap(1));
          const int64_t ne = (ab[p + 1] - ab[p]) + (bb[p + 1] - bb[p]);
          if (ne == 0) continue;
          // panel p of the group: kv[start[(p - g0)·ntot], start[(p - g0 + 1)·ntot])
          const int64_t q = (int64_t)(p - g0) * ntot;
          CSR_TRY(accumulate(ne, start + q, start + q + ntot));
          CSR_TRY(lap(2));
        }
      } else {
        if (xh && grows > 0)
          CSR_TRY(cudaMemset2DAsync(xh + r0g * ldh, (size_t)ldh * 2, 0, (size_t)n_head * 2, (size_t)grows, st));
        CSR_TRY(lap(0));
        for (int p = g0; p < g1; ++p) {  // Π panels still feed the head's κ-major panel
          gen_panel(p, (int)std::min<int64_t>(rp, rows - (int64_t)p * rp));
          CSR_TRY(lap(1));
        }
      }
      g0 = g1;
    }
  } else {
    CSR_TRY(grow(w.kv_in, w.ent_cap_ki, max_ent));
    CSR_TRY(grow(w.kv_out, w.ent_cap_ko, max_ent));
    size_t need = 0;
    CSR_TRY(cub::DeviceRadixSort::SortKeys(nullptr, need, w.kv_in, w.kv_out, (int)std::max<int64_t>(max_ent, 1),
                                           32, 32 + end_bit, st));
    CSR_TRY(grow(w.cub_tmp, w.cub_cap, (int64_t)need));
    for (int p = 0; p < npan; ++p) {
      const int64_t p0 = (int64_t)p * rp;
      const int prow = (int)std::min<int64_t>(rp, rows - p0);
      const int64_t na = ab[p + 1] - ab[p], nb = bb[p + 1] - bb[p];
      const int64_t ne = na + nb;
      gen_panel(p, prow);
      CSR_TRY(lap(1));
      if (ne == 0) continue;
      const int64_t pr = rbase + p0;  // rowptr index of the panel's first row
      const int kb_blocks = (int)std::min<int64_t>((prow + 7) / 8, 148 * 16);
      // A: entries ab[p] .. ab[p+1] (relative to a_rowptr[0]) -> kv[0 .. na)
      csr_keys_kernel<<<kb_blocks, 256, 0, st>>>(a_rowptr, a_col, a_val, pr, prow, ab[p], 0u, tbits,
                                                 a_n, w.kv_in, status);
      if (b_rowptr && nb > 0)
        csr_keys_kernel<<<kb_blocks, 256, 0, st>>>(b_rowptr, b_col, b_val, pr, prow, bb[p] - na,
                                                   (uint32_t)a_n, tbits, b_n, w.kv_in, status);
      size_t tmp = (size_t)w.cub_cap;
      CSR_TRY(cub::DeviceRadixSort::SortKeys(w.cub_tmp, tmp, w.kv_in, w.kv_out, (int)ne, 32, 32 + end_bit, st));
      w.launches += 1 + (b_rowptr && nb > 0 ? 1 : 0) + 4;
      CSR_TRY(lap(0));
      CSR_TRY(accumulate(ne, nullptr, nullptr));
      CSR_TRY(lap(2));
    }
  }
  if (prof) {
    if (!pev.empty()) CSR_TRY(cudaEventSynchronize(pev.back().first));
    for (size_t i = 1; i < pev.size(); ++i) {
      float ms = 0.f;
      CSR_TRY(cudaEventElapsedTime(&ms, pev[i - 1].first, pev[i].first));
      if (pev[i].second >= 0) pms[pev[i].second] += ms;
    }
    for (auto& e : pev) cudaEventDestroy(e.first);
    fprintf(stderr, "K3 stages over %d panels: sort%s %.3f ms, pi panel %.3f ms, accumulate %.3f ms\n", npan,
            xh ? " + head densify" : "", pms[0], pms[1], pms[2]);
  }
  return cudaGetLastError();
}

}  // namespace smp
