// K1F: the dense one-pass sketch for FP32 inputs with the exact bf16 plane
// split fused in (Alg. 1 line 2; Step 1; DESIGN.md
// R21).  Reading fp32 once from HBM instead of materialising planes:
//
//   x = p1 + p2 + p3 (bf16 planes; ±1 Π: 8+8+8 bits exact; Gaussian Π: 4+8+8
//   bits, remainder <= 2^-21 |x| dropped), D_q += Π · P_q per plane in its
//   own TMEM accumulator (a single accumulator would swallow the small
//   planes' low bits), fp64 Σx² from the fp32 values.
//
// CTA pair (cluster of 2, tcgen05 cta_group::2) tile: 256 κ × 128 input
// columns (64 per SM).  Per 64-row K-block and SM:
//   * TMA: the fp32 X half tile (2 boxes of 32 columns × 64 rows, 128B
//     swizzle, 16 KB) and this SM's 128 κ × 64 t Π tile from the κ-major
//     panel (16 KB), one 4-stage ring;
//   * 8 converter warps read X from SMEM, write the three bf16 planes in the
//     MMA's B layout (SW128, MN-major, 8 KB each; 2-slot ring) and
//     accumulate the fp64 norms;
//   * one leader thread issues 4 K-steps × 3 planes of M=256, N=128, K=16
//     (A = Π from SMEM, K-major) into TMEM columns [128 q, 128 q + 128);
//   * the converter warps then drain TMEM into part[split][q n + c][κ],
//     the layout K2 reduces (planes summed in fp32, fixed order).
#include <cuda.h>
#include <cudaTypedefs.h>
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

namespace f32k {
constexpr int BK = 64;                      // rows per K-block
constexpr int HALF_N = 64;                  // input columns per SM
#ifndef SMP_F32_NSTG
#define SMP_F32_NSTG 4
#endif
#ifndef SMP_F32_NPL
#define SMP_F32_NPL 3
#endif
constexpr int NSTG = SMP_F32_NSTG;          // X + Π ring
constexpr int X_BYTES = BK * HALF_N * 4;    // 16 KB fp32
constexpr int PI_BYTES = 128 * BK * 2;      // 16 KB
// SPLIT: the fp32 X tile and the Π tile live in rings of their own.  An X
// stage is free as soon as the converters have read it (the MMA never reads
// fp32), so its TMA runs NX K-blocks ahead of the converters instead of being
// tied to the MMA's completion; a Π stage is freed by the MMA's commit.
#ifndef SMP_F32_SPLIT
#define SMP_F32_SPLIT 0
#endif
#ifndef SMP_F32_NPI
#define SMP_F32_NPI 3
#endif
#ifndef SMP_F32_X_PROMO
#define SMP_F32_X_PROMO CU_TENSOR_MAP_L2_PROMOTION_L2_256B
#endif
constexpr bool SPLIT = SMP_F32_SPLIT != 0;
// DIRECT: each converter warp arrives on the LEADER CTA's ready barrier itself
// (release at cluster scope) instead of going through a local barrier and the
// relay thread: one hop less in the per-stage chain that bounds K1F.
#ifndef SMP_F32_DIRECT
#define SMP_F32_DIRECT 0
#endif
constexpr bool DIRECT = SMP_F32_DIRECT != 0 && !SPLIT;
constexpr int NPI = SPLIT ? SMP_F32_NPI : NSTG;          // Π ring stages
constexpr int STG = SPLIT ? X_BYTES : X_BYTES + PI_BYTES;   // bytes per X(+Π) stage
constexpr int PI_RING = SPLIT ? NPI * PI_BYTES : 0;
constexpr int NPL = SMP_F32_NPL;            // plane ring
constexpr int PLANE = BK * HALF_N * 2;      // 8 KB bf16
constexpr int PSLOT = 3 * PLANE;            // 24 KB
#ifndef SMP_F32_NCONV
#define SMP_F32_NCONV 16
#endif
constexpr int NCONV = SMP_F32_NCONV;        // converter warps (8..)
constexpr int RG = 2 * NCONV;               // row groups (32 lanes x NCONV / 16 chunks)
constexpr int ROWS_PT = BK / RG;            // rows per converter thread per K-block
constexpr int RED = RG * HALF_N * 8;        // 8 KB fp64 norm reduction
constexpr int BARS = 2 * NSTG + 3 * NPL + 1 + 2 * NPI;
constexpr int SMEM = NSTG * STG + PI_RING + NPL * PSLOT + RED + BARS * 8 + 16 + 1024;
static_assert(SMEM <= 227 * 1024, "K1F exceeds the SMEM budget");
constexpr int THREADS = 32 * (8 + NCONV);
constexpr int TMEM_COLS = 512;
}  // namespace f32k

// SMP_F32_TRACE (tuning builds only): per-K-block clock64 stamps of one CTA
// pair's pipeline events, read back with smp_debug_k1f_trace
#ifdef SMP_F32_TRACE
__device__ unsigned long long g_k1f_trace[2][8][512];
#define K1F_TR(ev, it)                                                             \
  do {                                                                             \
    if ((blockIdx.x >> 1) == SMP_F32_TRACE && (it) < 512) g_k1f_trace[rank][ev][it] = clock64(); \
  } while (0)
#else
#define K1F_TR(ev, it)
#endif

// round to b significant bits (RNE on the fp32 pattern); see reduce.cu
__device__ __forceinline__ float f32k_round_sig(float x, int b) {
  const uint32_t u = __float_as_uint(x);
  if ((u & 0x7F800000u) == 0u) return 0.0f * x;
  const int drop = 24 - b;
  const uint32_t half = 1u << (drop - 1);
  const uint32_t lsb = (u >> drop) & 1u;
  const uint32_t mag = ((u & 0x7FFFFFFFu) + half - 1u + lsb) & ~((1u << drop) - 1u);
  return __uint_as_float((u & 0x80000000u) | mag);
}

// (hi << 16) | lo of bf16_rne(a) (lo) and bf16_rne(b) (hi): one F2FP instead of
// the 4-instruction integer RNE per value (same bits for finite inputs)
__device__ __forceinline__ uint32_t f32k_bf16x2(float a, float b) {
  uint32_t z;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(z) : "f"(b), "f"(a));
  return z;
}

// (hi, lo) += x² in double-float arithmetic on the fp32 pipe: p + e = x² exactly
// (FMA residual), TwoSum(hi, p) exactly, the small terms gathered in lo.  The
// pair carries ~46 significant bits (relative error < 2^-44 over a CTA's
// K-range); it replaces a F2F.F64.F32 + DFMA per element, which the trace showed
// as +1,100 cycles on every K-block with norm duty.  Valid while x² and its
// residual stay normal fp32 numbers: |x| in [2^-40, 2^41) or x = 0 (subnormal
// x: x² < 2^-252, dropped); other magnitudes take the fp64 path (f32k_sq_fast).
__device__ __forceinline__ bool f32k_sq_fast(float x) {
  const uint32_t t = __float_as_uint(x) & 0x7F800000u;       // biased exponent field
  return t == 0u || (t - 0x2B800000u) <= 0x28000000u;        // exponent in [87, 167]
}
__device__ __forceinline__ void f32k_sq_acc(float x, float& hi, float& lo) {
  const float p = __fmul_rn(x, x);
  const float e = __fmaf_rn(x, x, -p);
  const float s = __fadd_rn(hi, p);
  const float bb = __fsub_rn(s, hi);
  const float err = __fadd_rn(__fsub_rn(hi, __fsub_rn(s, bb)), __fsub_rn(p, bb));
  hi = s;
  lo = __fadd_rn(lo, __fadd_rn(err, e));
}

__global__ void __launch_bounds__(f32k::THREADS, 1)
sketch_tc_f32_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_pi,
                     SketchTCParams p, int mode) {
  using namespace f32k;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* st_s = smem;                                   // [NSTG][X 16 KB | Π 16 KB]
  uint8_t* pi_s = smem + NSTG * STG;                      // SPLIT: [NPI][Π 16 KB]
  uint8_t* pl_s = pi_s + PI_RING;                         // [NPL][3][8 KB]
  double* red = reinterpret_cast<double*>(pl_s + NPL * PSLOT);   // [RG][64]
  uint64_t* xfull = reinterpret_cast<uint64_t*>(pl_s + NPL * PSLOT + RED);
  uint64_t* xempty = xfull + NSTG;
  uint64_t* pfull = xempty + NSTG;    // converters -> relay (this CTA's planes of slot ps)
  uint64_t* pempty = pfull + NPL;     // MMA commit -> converters
  uint64_t* ready = pempty + NPL;     // leader only: both CTAs' slot ps ready
  uint64_t* pifull = ready + NPL;     // SPLIT: Π tile landed
  uint64_t* piempty = pifull + NPI;   // SPLIT: MMA commit -> Π producer
  uint64_t* tmem_full = piempty + NPI;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  int bid = blockIdx.x >> 1;
  const int kt = bid % p.k_tiles; bid /= p.k_tiles;
  const int nt = bid % p.n_tiles; bid /= p.n_tiles;
  const int split = bid;
  const int kb_begin = (int)(((int64_t)split * p.kb_total) / p.splits);
  const int kb_end = (int)(((int64_t)(split + 1) * p.kb_total) / p.splits);
  const int nkb_all = kb_end - kb_begin;
  // ablation (SMP_K1F_DEBUG & 512): the TMA producer alone, consuming its own stages
  const bool tma_solo = (p.debug & 512) != 0;
  const int nkb = tma_solo ? 0 : nkb_all;
  const int n0 = nt * 2 * HALF_N + (int)rank * HALF_N;   // this SM's input columns
  const int kappa0 = kt * 256 + (int)rank * 128;

  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], SPLIT ? NCONV : 1 + NCONV);
    }
    for (int s = 0; s < NPI; ++s) {
      mbar_init(&pifull[s], 1);
      mbar_init(&piempty[s], 1);
    }
    for (int s = 0; s < NPL; ++s) {
      mbar_init(&pfull[s], NCONV);
      mbar_init(&pempty[s], 1);
      mbar_init(&ready[s], DIRECT ? 2 * NCONV : 2);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap_x);
    tma_prefetch_desc(&tmap_pi);
  }
  if (warp == 1) tmem_alloc2(tmem_base_s, TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tmem_base_s;

  if (warp == 0) {
    // ---------------- TMA producer: fp32 X half tile + Π tile per stage
    if (lane == 0) {
      for (int it = 0; it < nkb_all; ++it) {
        const int s = it % NSTG;
        if (!tma_solo) mbar_wait(&xempty[s], ((uint32_t)(it / NSTG) & 1u) ^ 1u);
        else if (it >= NSTG) mbar_wait(&xfull[s], ((uint32_t)(it / NSTG) & 1u) ^ 1u);
        K1F_TR(0, it);
        // ablation (SMP_K1F_DEBUG): 128 = no Π TMA, 256 = no X TMA
        const bool ld_pi = !SPLIT && !(p.debug & 128), ld_x = !(p.debug & 256);
        mbar_arrive_expect_tx(&xfull[s], (ld_x ? X_BYTES : 0) + (ld_pi ? PI_BYTES : 0));
        const int row = (kb_begin + it) * BK;
        if (ld_x) {
          tma_load_2d(st_s + s * STG, &tmap_x, &xfull[s], n0, row);
          tma_load_2d(st_s + s * STG + 8192, &tmap_x, &xfull[s], n0 + 32, row);
        }
        if (ld_pi) tma_load_2d(st_s + s * STG + X_BYTES, &tmap_pi, &xfull[s], row, kappa0);
      }
      if (tma_solo)
        for (int it = nkb_all > NSTG ? nkb_all - NSTG : 0; it < nkb_all; ++it)
          mbar_wait(&xfull[it % NSTG], (uint32_t)(it / NSTG) & 1u);
    }
  } else if (SPLIT && warp == 3) {
    // ---------------- TMA producer of the Π ring (SPLIT)
    if (lane == 0) {
      for (int it = 0; it < nkb; ++it) {
        const int s = it % NPI;
        mbar_wait(&piempty[s], ((uint32_t)(it / NPI) & 1u) ^ 1u);
        mbar_arrive_expect_tx(&pifull[s], PI_BYTES);
        tma_load_2d(pi_s + s * PI_BYTES, &tmap_pi, &pifull[s], (kb_begin + it) * BK, kappa0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread)
    if (rank == 0 && lane == 0) {
      // planes 0 and 1 in one N=256 instruction (each CTA's two 64-column
      // plane tiles are adjacent: LBO = 8 KB), plane 2 in an N=128 one: the
      // Π tile (A) is read twice per K-step instead of three times
      const uint32_t idesc256 = make_idesc_bf16(256, 256, 0, 1);
      const uint32_t idesc128 = make_idesc_bf16(256, 128, 0, 1);
      const uint32_t pl_addr = smem_u32(pl_s);
      const uint32_t a_addr = SPLIT ? smem_u32(pi_s) : smem_u32(st_s) + X_BYTES;
      constexpr int A_STRIDE = SPLIT ? PI_BYTES : STG;
      for (int it = 0; it < nkb; ++it) {
        const int s = it % NSTG, ps = it % NPL, pis = it % NPI;
        mbar_wait(&ready[ps], (uint32_t)(it / NPL) & 1u);
        tc_fence_after();
        K1F_TR(5, it);
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk) {
          const uint64_t adesc = make_sdesc_sw128(a_addr + pis * A_STRIDE + kk * 32, 16, 1024);
          const uint64_t b01 = make_sdesc_sw128(pl_addr + ps * PSLOT + kk * 2048, 8192, 1024);
          const uint64_t b2 = make_sdesc_sw128(pl_addr + ps * PSLOT + 2 * PLANE + kk * 2048, 8192, 1024);
          if (p.debug & 4) continue;   // ablation (SMP_K1F_DEBUG): no MMA
          tc_mma2_ss(tbase, adesc, b01, idesc256, (it | kk) != 0 ? 1u : 0u);
          if (p.debug & 32) continue;  // ablation: no third-plane MMA
          tc_mma2_ss(tbase + 256, adesc, b2, idesc128, (it | kk) != 0 ? 1u : 0u);
        }
        if (SPLIT) tc_commit2(&piempty[pis], 0x3);
        else tc_commit2(&xempty[s], 0x3);
        tc_commit2(&pempty[ps], 0x3);
        K1F_TR(6, it);
      }
      tc_commit2(tmem_full, 0x3);
    }
  } else if (warp == 2) {
    // ---------------- relay: this CTA's planes of slot ps (and its Π) are ready
    if (lane == 0 && !DIRECT) {
      const uint32_t leader_ready = mapa_shared(smem_u32(ready), 0);
      for (int it = 0; it < nkb; ++it) {
        const int ps = it % NPL;
        mbar_wait(&pfull[ps], (uint32_t)(it / NPL) & 1u);
        if (SPLIT) mbar_wait(&pifull[it % NPI], (uint32_t)(it / NPI) & 1u);
        K1F_TR(4, it);
        mbar_arrive_cluster_release(leader_ready + 8u * (uint32_t)ps);
      }
    }
  } else if (warp >= 8) {
    // ---------------- converters (+ fp64 norms), then the TMEM epilogue
    // thread (rg, q): 16-byte fp32 chunk q (box q>>3, chunk q&7: columns
    // 32 box + 4 chunk .. +3) of rows rg, rg + RG, ...
    const int g = tid - 256;
    const int q = g & 15, rg = g >> 4;
    const int box = q >> 3, chunk = q & 7;
    const int c0 = 32 * box + 4 * chunk;   // first of this thread's 4 columns
    float nhi[4] = {0.f, 0.f, 0.f, 0.f}, nlo[4] = {0.f, 0.f, 0.f, 0.f};
    double nacc[4] = {0.0, 0.0, 0.0, 0.0};   // elements outside the fp32-safe range (rare)
    const bool norms_on = p.do_norms != 0 && !(p.debug & 1);
    int duty_ctr = kb_begin % p.k_tiles;
    // first plane: 4 significant bits (Gaussian Π) or 8 (±1 Π), RNE on the
    // fp32 pattern (zero and subnormal patterns round to themselves' prefix,
    // so the remainders stay exact); then bf16 RNE; then the exact (±1) or
    // rounded (Gaussian, remainder dropped) third plane
    const uint32_t conv_ready = mapa_shared(smem_u32(ready), 0);   // DIRECT: the leader's barrier
    const uint32_t rb = mode == 4 ? 20u : 16u;           // dropped bits of plane 1
    const uint32_t rmask = (1u << rb) - 1u, rhalf = (1u << (rb - 1)) - 1u;
    for (int it = 0; it < nkb; ++it) {
      const int s = it % NSTG, ps = it % NPL;
#ifdef SMP_F32_ELECT_POLL
      mbar_wait_warp(&xfull[s], (uint32_t)(it / NSTG) & 1u);
      mbar_wait_warp(&pempty[ps], ((uint32_t)(it / NPL) & 1u) ^ 1u);
#else
      mbar_wait(&xfull[s], (uint32_t)(it / NSTG) & 1u);
      if (tid == 256) K1F_TR(1, it);
      mbar_wait(&pempty[ps], ((uint32_t)(it / NPL) & 1u) ^ 1u);
      if (tid == 256) K1F_TR(2, it);
#endif
      const bool duty = norms_on && duty_ctr == kt;
      if (++duty_ctr == p.k_tiles) duty_ctr = 0;
      const uint8_t* xb = st_s + s * STG + box * 8192;
      uint8_t* pb = pl_s + ps * PSLOT;
      const int pc = c0 >> 3, po = (c0 & 7) * 2;
#pragma unroll
      for (int i = 0; i < ROWS_PT; ++i) {
        if (p.debug & 64) break;     // ablation: no conversion
        const int r = rg + RG * i;
        const float4 v = *reinterpret_cast<const float4*>(xb + r * 128 + ((chunk ^ (r & 7)) << 4));
        const float x[4] = {v.x, v.y, v.z, v.w};
        if (duty) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (f32k_sq_fast(x[j])) f32k_sq_acc(x[j], nhi[j], nlo[j]);
            else nacc[j] = fma((double)x[j], (double)x[j], nacc[j]);
          }
        }
        // plane 1 by the integer RNE (4 or 8 significant bits), planes 2 and 3
        // by packed bf16 RNE converts (plane 3 of a ±1 Π is the exact 8-bit
        // remainder, which the convert leaves unchanged)
        uint32_t b1[4];
        float r1[4], r2[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t u = __float_as_uint(x[j]);
          const uint32_t h = (u + rhalf + ((u >> rb) & 1u)) & ~rmask;
          r1[j] = __fsub_rn(x[j], __uint_as_float(h));
          b1[j] = h;
        }
        const uint32_t p2a = f32k_bf16x2(r1[0], r1[1]), p2b = f32k_bf16x2(r1[2], r1[3]);
        r2[0] = __fsub_rn(r1[0], __uint_as_float(p2a << 16));
        r2[1] = __fsub_rn(r1[1], __uint_as_float(p2a & 0xFFFF0000u));
        r2[2] = __fsub_rn(r1[2], __uint_as_float(p2b << 16));
        r2[3] = __fsub_rn(r1[3], __uint_as_float(p2b & 0xFFFF0000u));
        const uint32_t p3a = f32k_bf16x2(r2[0], r2[1]), p3b = f32k_bf16x2(r2[2], r2[3]);
        // element (r, c) of a 64x64 bf16 SW128 tile: r*128 + ((c>>3) ^ (r&7))*16 + (c&7)*2;
        // this thread's 4 columns share one 16-byte chunk
        const uint32_t off = (uint32_t)(r * 128 + ((pc ^ (r & 7)) << 4) + po);
        *reinterpret_cast<uint2*>(pb + off) =
            make_uint2(__byte_perm(b1[0], b1[1], 0x7632), __byte_perm(b1[2], b1[3], 0x7632));
        *reinterpret_cast<uint2*>(pb + PLANE + off) = make_uint2(p2a, p2b);
        *reinterpret_cast<uint2*>(pb + 2 * PLANE + off) = make_uint2(p3a, p3b);
      }
      fence_proxy_async_smem();   // generic-proxy plane writes -> visible to the tensor core
      __syncwarp();
      if (tid == 256) K1F_TR(3, it);
      if (tid == 32 * (8 + NCONV - 1)) K1F_TR(7, it);
      if (lane == 0) {
        mbar_arrive(&xempty[s]);
        if (DIRECT) mbar_arrive_cluster_release(conv_ready + 8u * (uint32_t)ps);
        else mbar_arrive(&pfull[ps]);
      }
    }
    // norm partials: fixed-order reduction over the 16 row groups
#pragma unroll
    for (int j = 0; j < 4; ++j) red[rg * HALF_N + c0 + j] = ((double)nhi[j] + (double)nlo[j]) + nacc[j];
    named_bar_sync(1, 32 * NCONV);
    const int slot = split * p.k_tiles + kt;
    if (g < HALF_N) {
      double v = red[g];
      for (int w = 1; w < RG; ++w) v += red[w * HALF_N + g];
      if (n0 + g < p.n && p.do_norms) p.pnorm[(int64_t)slot * p.n + n0 + g] = v;
    }
    // TMEM -> part[split][q n + col][κ]: warp quad owns lanes 32 quad..,
    // the NCONV/4 warps of a quad split the 384 accumulator columns
    const int quad = warp & 3;
    const int chalf = (warp - 8) >> 2;
    constexpr int CPW = 12 / (NCONV / 4);   // 32-column chunks per warp
    if (nkb > 0) {
      mbar_wait(tmem_full, 0);
      tc_fence_after();
    }
    const int kappa = kappa0 + 32 * quad + lane;
    const int ncol0 = nt * 2 * HALF_N;
    // TMEM column t: [0, 256) = N=256 MMA over (plane 0 | plane 1) of CTA 0,
    // then of CTA 1 (64 columns each); [256, 384) = plane 2, CTA 0 then CTA 1
    for (int cc = chalf * CPW; cc < chalf * CPW + CPW; ++cc) {
      const int t0c = cc * 32;
      int pq, cbase;
      if (t0c < 256) {
        const int h = t0c >> 7, w = t0c & 127;
        pq = w >> 6;
        cbase = h * 64 + (w & 63);
      } else {
        pq = 2;
        cbase = t0c - 256;
      }
      uint32_t r[32];
      tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * quad) << 16) + t0c, r);
      tc_wait_ld();
      if (nkb == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      }
      if (kappa < p.k) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = ncol0 + cbase + j;
          if (col < p.n)
            p.part[((int64_t)split * 3 * p.n + (int64_t)pq * p.n + col) * p.k + kappa] = __uint_as_float(r[j]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tbase, TMEM_COLS);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 f32k_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

#ifdef SMP_F32_TRACE
extern "C" __attribute__((visibility("default"))) int smp_debug_k1f_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_k1f_trace, sizeof(g_k1f_trace));
}
#endif

int sketch_tc_f32_cols_per_tile() { return 2 * f32k::HALF_N; }

cudaError_t launch_sketch_tc_f32(const float* X, int64_t ldx, SketchTCParams p, int mode, cudaStream_t st) {
  auto enc = f32k_encode_fn();
  if (!enc || !p.pi_panel) return cudaErrorNotSupported;
  CUtensorMap tmap_x, tmap_pi;
  {
    cuuint64_t dims[2] = {(cuuint64_t)p.n, (cuuint64_t)p.rows};
    cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
    cuuint32_t box[2] = {32, 64};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&tmap_x, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, SMP_F32_X_PROMO,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)p.pi_ld, (cuuint64_t)p.k_tiles * 256};
    cuuint64_t strides[1] = {(cuuint64_t)p.pi_ld * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    if (enc(&tmap_pi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(p.pi_panel), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return cudaErrorInvalidValue;
  }
  static PerDeviceOnce attr;
  if (attr.need()) {
    cudaError_t e = cudaFuncSetAttribute(sketch_tc_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         f32k::SMEM);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2u * (unsigned)(p.n_tiles * p.k_tiles * p.splits));
  cfg.blockDim = dim3(f32k::THREADS);
  cfg.dynamicSmemBytes = f32k::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr1[1];
  attr1[0].id = cudaLaunchAttributeClusterDimension;
  attr1[0].val.clusterDim.x = 2;
  attr1[0].val.clusterDim.y = 1;
  attr1[0].val.clusterDim.z = 1;
  cfg.attrs = attr1;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, sketch_tc_f32_kernel, tmap_x, tmap_pi, p, mode);
}

}  // namespace smp
