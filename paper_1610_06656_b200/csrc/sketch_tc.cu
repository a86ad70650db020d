// K1: dense one-pass sketch with fused exact column norms (Alg. 1 line 2,
// PAPER.md P:54; Step 1), on the sm_100a tensor cores.
//
//   part[split][c][κ] = Σ_{t in split's rows} Π(κ, t) · X[t, c]   (fp32, TMEM)
//   pnorm[slot][c]    = Σ_{t in split's rows} X[t, c]^2          (fp64, SIMT)
//
// GEMM view: D (κ × c) += Π (κ × t) · X (t × c), M = κ, N = c, K = t.
// A CTA PAIR (cluster of 2, tcgen05 cta_group::2) owns a 256 κ × 256 column
// tile: each SM holds 128 κ rows of Π (its half of A) and 128 columns of X
// (its half of B); one thread of the leader issues M=256, N=256, K=16 MMAs
// that run on both SMs.  Per SM:
//   * X half tile (64 rows × 128 cols bf16) arrives by TMA as two 64×64
//     128B-swizzled boxes: the B operand, MN-major (8-stage SMEM ring).
//   * Π half tile (128 κ × 64 t) is regenerated from the Philox hash by 2
//     sets of 4 generator warps and written straight into TMEM with tcgen05.st: the A
//     operand lives in TMEM (4-stage ring of 32 columns), so Π costs no SMEM
//     bandwidth and is stored nowhere else.
//   * 8 norm warps read the X stage once from SMEM: exact fp32 squares
//     (bf16 has 8 significant bits) summed over 4-row chunks in fp32, then
//     one fp64 add per chunk (R4): A and B are read from HBM
//     exactly once.
//   * the same 8 warps drain the 128 × 256 fp32 accumulator (tcgen05.ld)
//     into the split's partial slot.
// Per-SM SMEM traffic per 64-row K-block: 16 KB TMA write + 16 KB MMA B read
// + 16 KB norm read = 48 KB per 512 tensor cycles (vs 96 B/cycle for the
// MMA operands alone in the one-SM SMEM-SMEM form).
// Synchronisation (per CTA): xfull (TMA tx) / xempty (MMA commit + norm
// warps); pfull (generator warps) / pempty (MMA commit); a relay thread in
// each CTA forwards "X and Π of stage s ready" to the leader's ready[s]
// (count 2, remote mbarrier arrive for the peer); MMA commits are multicast
// to both CTAs.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdlib>
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

constexpr int TC_BM = 256;                        // κ rows per CTA pair (128 per SM)
constexpr int TC_BN = 256;                        // X columns per CTA pair (128 per SM)
constexpr int HALF_N = TC_BN / 2;
constexpr int TC_BK = 64;                         // X rows per K-block
#ifndef SMP_X_STAGES
#define SMP_X_STAGES 8
#endif
constexpr int X_STAGES = SMP_X_STAGES;            // SMEM ring (HBM latency hiding)
// Π generator warp sets (4 warps each) are a template parameter GS of K1:
// 2 when every CTA pair owns the only κ tile of its X tile (k <= 256: the norm
// warps are on duty for every K-block and the SM's issue slots are shared), 3
// when several κ tiles share an X tile (the generators are then the MMA's
// feeder: cfg2 no-MMA generator throughput 23.7 -> 19.5 ms per launch, full
// kernel 31.0 -> 29.6 ms under the power cap; profiles/round2/k1_gen_sets.log).
constexpr int MAX_GEN_SETS = 4;
constexpr int PI_STAGES = 2 * MAX_GEN_SETS;       // barrier slots; a GS build uses 2*GS TMEM stages
constexpr int X_STAGE = TC_BK * HALF_N * 2;       // 16 KB
constexpr int ACC_COLS = TC_BN;                   // fp32 accumulator columns
constexpr int PI_COLS = TC_BK / 2;                // 64 bf16 per lane = 32 columns
constexpr int TMEM_COLS = 512;
static_assert(ACC_COLS + PI_STAGES * PI_COLS <= TMEM_COLS, "TMEM budget");
// each set takes every GS-th pair of K-blocks; a set may run at most one
// ring phase ahead of the MMA only if the ring holds one pair per set
// (so the TMEM ring is 2*GS stages)
// Warp roles: 0 TMA, 1 MMA (leader) + TMEM alloc, 2 relay, 3 spare,
// 4..7, 16..19 (and 20..23, 24..27 for GEN_SETS = 3, 4) Π generators (one warp
// per TMEM lane quadrant per set; the sets take the pairs of K-blocks round
// robin), 8..15 norm warps + TMEM epilogue.
constexpr int NUM_NORM_WARPS = 8;                 // warps 8..15
constexpr int NORM_RG = (32 * NUM_NORM_WARPS) / 16;   // row groups (16 chunks per row)
constexpr int NORM_ROWS = TC_BK / NORM_RG;        // rows per norm thread per stage
constexpr int NORM_RED = NORM_RG * HALF_N * 8;    // 16 KB
constexpr int TC_BARS = 3 * X_STAGES + 2 * PI_STAGES + 1;
constexpr int TC_SMEM = X_STAGES * X_STAGE + NORM_RED + TC_BARS * 8 + 16 + 1024;
static_assert(TC_SMEM <= 227 * 1024, "K1 exceeds the 227 KB SMEM budget");
// PANEL variant (Gaussian Π read from an L2-resident κ-major panel): each
// stage holds the X half tile AND this SM's 128 κ x 64 t Π tile, both by
// TMA (128B swizzle; the Π box is exactly the K-major SW128 layout of the
// MMA's A operand), and the MMA reads A from SMEM.
constexpr int P_STAGES = 6;
constexpr int PI_TILE = 128 * TC_BK * 2;          // 16 KB
constexpr int P_STAGE = X_STAGE + PI_TILE;        // 32 KB
constexpr int P_BARS = 3 * P_STAGES + 2 * PI_STAGES + 1;
constexpr int P_SMEM = P_STAGES * P_STAGE + NORM_RED + P_BARS * 8 + 16 + 1024;
static_assert(P_SMEM <= 227 * 1024, "K1 (panel) exceeds the 227 KB SMEM budget");
constexpr int tc_threads(int gs) { return 32 * (12 + 4 * gs); }   // sets 2.. at warps 20, 24, ...

struct RadCache {
  uint64_t g;
  uint32_t w0, w1, w2, w3;
};

// Word W (global index over 32-row words) of the Rademacher bit string of
// row κ: group W>>2 = Philox(ctr=(g, κ, g>>32, 1)).
__device__ __forceinline__ uint32_t rad_word(RadCache& c, uint64_t W, uint32_t kappa,
                                             uint32_t k0, uint32_t k1, uint32_t tag = TAG_RADEMACHER) {
  uint64_t g = W >> 2;
  if (g != c.g) {
    u32x4 w = philox4x32_10((uint32_t)g, kappa, (uint32_t)(g >> 32), tag, k0, k1);
    c.g = g; c.w0 = w.x; c.w1 = w.y; c.w2 = w.z; c.w3 = w.w;
  }
  uint32_t i = (uint32_t)(W & 3);
  return i == 0 ? c.w0 : i == 1 ? c.w1 : i == 2 ? c.w2 : c.w3;
}

// Bit position of element e (0..31) inside its 32-row word: even rows use
// bits 0..15, odd rows bits 16..31, so that a bf16 pair
// (rows 2p, 2p+1) is built with one shift and one LOP3.
__device__ __forceinline__ uint32_t rad_pos(uint32_t e) { return (e >> 1) | ((e & 1u) << 4); }

// (a & b) | c in ONE LOP3 with b and c in registers: written as two C
// operators with two immediates the compiler emits two LOP3s per bf16 pair
// (a LOP3 has one immediate slot), i.e. 3 instructions per pair with the
// shift instead of 2 — a quarter of the generator warps' instructions, which
// pace cfg1 (profiles/round2/k1_trace_cfg1.log).
__device__ __forceinline__ uint32_t lop3_and_or(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// a constant the compiler cannot fold back into an immediate
__device__ __forceinline__ uint32_t opaque_u32(uint32_t v) {
  uint32_t d;
  asm volatile("mov.u32 %0, %1;" : "=r"(d) : "r"(v));
  return d;
}

// Half a κ row of the Π tile, rows t0..t0+31: 32 bf16 packed in 16 words
// (word p = rows 2p (low half) and 2p+1 (high half)), the TMEM A layout.
__device__ __forceinline__ void gen_pi_half(int kind, uint64_t seed, uint32_t kappa, bool valid,
                                            uint64_t t0, RadCache& rc, uint32_t (&o)[16],
                                            uint64_t srht_s, uint32_t srht_walsh,
                                            uint32_t sign_mask, uint32_t one_pair) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  if (!valid) {
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = 0u;
    return;
  }
  if (kind >= PI_SRHT_BASE && (t0 & 31) == 0) {
    // 32 rows: D word (stream 6, κ-independent, cached per 128 rows) XOR the
    // Walsh pattern of s_κ's low 5 bits XOR parity(s_κ & t0) (t0 32-aligned)
    const uint32_t dw = rad_word(rc, t0 >> 5, 0u, k0, k1, TAG_SRHT_D);
    const uint32_t hb = (uint32_t)__popcll((unsigned long long)(srht_s & t0)) & 1u;
    const uint32_t w = dw ^ srht_walsh ^ (0u - hb);
#pragma unroll
    for (int p = 0; p < 16; ++p) o[p] = lop3_and_or(w * (1u << (15 - p)), sign_mask, one_pair);
  } else if (kind == PI_RADEMACHER && (t0 & 31) == 0) {
    const uint32_t w = rad_word(rc, t0 >> 5, kappa, k0, k1);
#pragma unroll
    for (int p = 0; p < 16; ++p)  // shift as a multiply: IMAD on the FMA pipe, one LOP3 on ALU
      o[p] = lop3_and_or(w * (1u << (15 - p)), sign_mask, one_pair);
  } else if (kind == PI_GAUSSIAN && (t0 & 3) == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint64_t tq = (t0 >> 2) + q;
      const u32x4 w = philox4x32_10((uint32_t)tq, kappa, (uint32_t)(tq >> 32), TAG_GAUSSIAN, k0, k1);
      uint16_t a, b, c, d;
      gauss_pair(w.x, w.y, a, b);
      gauss_pair(w.z, w.w, c, d);
      o[2 * q] = (uint32_t)a | ((uint32_t)b << 16);
      o[2 * q + 1] = (uint32_t)c | ((uint32_t)d << 16);
    }
  } else {
    // generic (unaligned block start, Hadamard test mode): element by element
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      uint32_t lohi[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint64_t t = t0 + 2 * p + e;
        if (kind == PI_RADEMACHER) {
          const uint32_t w = rad_word(rc, t >> 5, kappa, k0, k1);
          lohi[e] = ((w >> rad_pos((uint32_t)(t & 31))) & 1u) ? 0xBF80u : 0x3F80u;
        } else if (kind >= PI_SRHT_BASE) {
          const uint32_t w = rad_word(rc, t >> 5, 0u, k0, k1, TAG_SRHT_D);
          const uint32_t bit = ((w >> rad_pos((uint32_t)(t & 31))) & 1u) ^
                               ((uint32_t)__popcll((unsigned long long)(srht_s & t)) & 1u);
          lohi[e] = bit ? 0xBF80u : 0x3F80u;
        } else {
          lohi[e] = pi_bits(kind, seed, kappa, t);
        }
      }
      o[p] = lohi[0] | (lohi[1] << 16);
    }
  }
}

// SMP_K1_TRACE=<pair index> (tuning builds only): clock64 stamps of one CTA
// pair's pipeline events per K-block, read back with smp_debug_k1_trace
#ifdef SMP_K1_TRACE
__device__ unsigned long long g_k1_trace[2][8][512];
#define K1_TR(ev, it)                                                              \
  do {                                                                             \
    if ((blockIdx.x >> 1) == SMP_K1_TRACE && (it) < 512) g_k1_trace[rank][ev][it] = clock64(); \
  } while (0)
#else
#define K1_TR(ev, it)
#endif

template <bool PANEL, int GS>
__global__ void __launch_bounds__(tc_threads(GS), 1)
sketch_tc_kernel(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap tmap_pi,
                 SketchTCParams p) {
  static_assert(GS >= 2 && GS <= MAX_GEN_SETS, "generator sets");
  constexpr int PIS = 2 * GS;                        // Π TMEM ring stages (one pair per set)
  constexpr int NST = PANEL ? P_STAGES : X_STAGES;   // ring stages
  constexpr int STG = PANEL ? P_STAGE : X_STAGE;     // bytes per stage
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023u) & ~1023u) - raw_addr);
  uint8_t* x_s = smem;                                              // [NST][X 16 KB (| Π 16 KB)]
  double* red = reinterpret_cast<double*>(smem + NST * STG);        // [NORM_RG][128]
  uint64_t* xfull = reinterpret_cast<uint64_t*>(smem + NST * STG + NORM_RED);
  uint64_t* xempty = xfull + NST;
  uint64_t* ready = xempty + NST;         // leader only: X and Π of both CTAs ready
  uint64_t* pfull = ready + NST;
  uint64_t* pempty = pfull + PI_STAGES;
  uint64_t* tmem_full = pempty + PI_STAGES;
  uint32_t* tmem_base_s = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = cluster_ctarank();
  // pair decomposition: kt innermost so pairs sharing an X tile run together
  int bid = blockIdx.x >> 1;
  const int kt = bid % p.k_tiles; bid /= p.k_tiles;
  const int nt = bid % p.n_tiles; bid /= p.n_tiles;
  const int split = bid;
  const int kb_begin = (int)(((int64_t)split * p.kb_total) / p.splits);
  const int kb_end = (int)(((int64_t)(split + 1) * p.kb_total) / p.splits);
  const int nkb = kb_end - kb_begin;
  const int n0 = nt * TC_BN + (int)rank * HALF_N;                // this SM's columns
  const int kappa0 = kt * TC_BM + (int)rank * 128;               // this SM's κ rows

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&xfull[s], 1);
      mbar_init(&xempty[s], 1 + NUM_NORM_WARPS);
      mbar_init(&ready[s], 2);
    }
    for (int s = 0; s < PI_STAGES; ++s) {
      mbar_init(&pfull[s], 4);   // one set of 4 warps writes a stage
      mbar_init(&pempty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmap);
    if (PANEL) tma_prefetch_desc(&tmap_pi);
  }
  if (warp == 1) tmem_alloc2(tmem_base_s, TMEM_COLS);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tmem_base_s;

  if (warp == 0) {
    // ---------------- TMA producer: this SM's half of the X tile
    if (lane == 0) {
      for (int it = 0; it < nkb; ++it) {
        const int s = it % NST;
        mbar_wait_backoff(&xempty[s], ((uint32_t)(it / NST) & 1u) ^ 1u, p.backoff_ns);
        K1_TR(0, it);
        mbar_arrive_expect_tx(&xfull[s], STG);
        const int row = (kb_begin + it) * TC_BK;
        tma_load_2d(x_s + s * STG, &tmap, &xfull[s], n0, row);
        tma_load_2d(x_s + s * STG + 8192, &tmap, &xfull[s], n0 + 64, row);
        if (PANEL) tma_load_2d(x_s + s * STG + X_STAGE, &tmap_pi, &xfull[s], row, kappa0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread)
    if (rank == 0 && lane == 0) {
      const uint32_t idesc = make_idesc_bf16(256, 256, 0, 1);
      const uint32_t x_addr = smem_u32(x_s);
      for (int it = 0; it < nkb; ++it) {
        const int s = it % NST, ps = it % PIS;
        mbar_wait(&ready[s], (uint32_t)(it / NST) & 1u);
        tc_fence_after();
        K1_TR(5, it);
        if (!(p.debug & 4)) {
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            const uint64_t bdesc = make_sdesc_sw128(x_addr + s * STG + kk * 2048, 8192, 1024);
            if (PANEL) {
              // A = Π tile, K-major SW128 (128 B rows = 64 t; 16 t = 32 B per MMA)
              const uint64_t adesc = make_sdesc_sw128(x_addr + s * STG + X_STAGE + kk * 32, 16, 1024);
              tc_mma2_ss(tbase, adesc, bdesc, idesc, (it | kk) != 0 ? 1u : 0u);
            } else {
              tc_mma2_ts(tbase, tbase + ACC_COLS + ps * PI_COLS + kk * 8, bdesc, idesc,
                         (it | kk) != 0 ? 1u : 0u);
            }
          }
        }
        tc_commit2(&xempty[s], 0x3);
        if (!PANEL) tc_commit2(&pempty[ps], 0x3);
        K1_TR(6, it);
      }
      tc_commit2(tmem_full, 0x3);
    }
  } else if (warp == 2) {
    // ---------------- relay: this CTA's X and Π of stage s are ready
    if (lane == 0) {
      const uint32_t leader_ready = mapa_shared(smem_u32(ready), 0);
      for (int it = 0; it < nkb; ++it) {
        const int s = it % NST, ps = it % PIS;
        mbar_wait(&xfull[s], (uint32_t)(it / NST) & 1u);
        K1_TR(1, it);
        if (!PANEL) mbar_wait(&pfull[ps], (uint32_t)(it / PIS) & 1u);
        K1_TR(4, it);
        mbar_arrive_cluster(leader_ready + 8u * (uint32_t)s);
      }
    }
  } else if ((warp >= 4 && warp < 8) || warp >= 16) {
    // ---------------- Π generators: thread owns TMEM lane 32*quad + lane (one
    // κ); set 0 (warps 4..7) and set 1 (warps 16..19) take alternate PAIRS of
    // K-blocks (2jp, 2jp+1), all 64 rows of each, so that one Philox call
    // (128 rows of one κ) serves the whole pair when the rows are 128-aligned;
    // the next pair's call is issued between the TMEM store and its wait, so
    // its latency overlaps the store (idle in PANEL mode: Π arrives by TMA)
    if (PANEL) goto role_done;
    const int quad = warp & 3;
    const int set = warp < 8 ? 0 : ((warp - 16) >> 2) + 1;
    const int kl = 32 * quad + lane;
    const int kappa = kappa0 + kl;
    const bool valid = kappa < p.k;
    const uint32_t k0 = (uint32_t)p.seed, k1 = (uint32_t)(p.seed >> 32);
    RadCache rc{~0ull, 0, 0, 0, 0};
    uint64_t srht_s = 0;
    uint32_t srht_walsh = 0;
    if (p.kind >= PI_SRHT_BASE && valid) {
      srht_s = srht_row(p.seed, p.kind - PI_SRHT_BASE, (uint32_t)kappa);
      srht_walsh = walsh32_interleaved((uint32_t)(srht_s & 31u));
    }
    const bool word_kind = p.kind == PI_RADEMACHER || p.kind >= PI_SRHT_BASE;
    const uint32_t sign_mask = opaque_u32(0x80008000u), one_pair = opaque_u32(0x3F803F80u);
    const uint32_t taddr = tbase + ((uint32_t)(32 * quad) << 16) + ACC_COLS;
    for (int jp = set; 2 * jp < nkb; jp += GS) {
      for (int h = 0; h < 2; ++h) {
        const int it = 2 * jp + h;
        if (it >= nkb) break;
        const int ps = it % PIS;
        const uint64_t t0 = (uint64_t)p.row0 + (uint64_t)(kb_begin + it) * TC_BK;
        uint32_t o[16], o2[16];
        if (quad == 0 && lane == 0) K1_TR(2, it);
        if (p.debug & 2) {
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] = o2[i] = 0x3F803F80u;
        } else {
          gen_pi_half(p.kind, p.seed, (uint32_t)kappa, valid, t0, rc, o, srht_s, srht_walsh, sign_mask, one_pair);
          gen_pi_half(p.kind, p.seed, (uint32_t)kappa, valid, t0 + 32, rc, o2, srht_s, srht_walsh, sign_mask,
                      one_pair);
        }
        if (quad == 0 && lane == 0) K1_TR(3, it);
        mbar_wait_backoff(&pempty[ps], ((uint32_t)(it / PIS) & 1u) ^ 1u, p.backoff_ns);
        tc_fence_after();
        if (quad == 0 && lane == 0) K1_TR(7, it);
        tmem_st_32x32b_x16(taddr + ps * PI_COLS, o);
        tmem_st_32x32b_x16(taddr + ps * PI_COLS + 16, o2);
        if (h == 1 || it + 1 == nkb) {
          // prefetch the Philox words of this set's next pair
          const int itn = 2 * (jp + GS);
          if (word_kind && valid && itn < nkb && !(p.debug & 2)) {
            const uint64_t tn = (uint64_t)p.row0 + (uint64_t)(kb_begin + itn) * TC_BK;
            if ((tn & 31) == 0) {
              if (p.kind == PI_RADEMACHER) (void)rad_word(rc, tn >> 5, (uint32_t)kappa, k0, k1);
              else (void)rad_word(rc, tn >> 5, 0u, k0, k1, TAG_SRHT_D);
            }
          }
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&pfull[ps]);
      }
    }
  } else if (warp >= 8) {
    // ---------------- norm warps (fp64 Σx²), then TMEM epilogue
    // thread (rg, q): 16-byte chunk q (box q>>3, chunk q&7) of rows r ≡ rg (mod 16)
    const int g = tid - 256;
    const int q = g & 15, rg = g >> 4;
    const int box = q >> 3, chunk = q & 7;
    // (fp32 double-float column sums, as K1F uses, were measured here too:
    // cfg1 0.545 vs 0.550 ms, cfg2 30.3 vs 29.5 ms per launch — the 56 extra
    // FADDs per K-block cost the power-capped cfg2 more than the fp64 adds)
    double acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
    // norm duty is split over the κ tiles that share this X tile: K-block kb
    // belongs to κ tile kb % k_tiles (counter kept incrementally)
    const bool norms_on = p.do_norms && !(p.debug & 1);
    int duty_ctr = kb_begin % p.k_tiles;
    for (int it = 0; it < nkb; ++it) {
      const int s = it % NST;
      mbar_wait_backoff(&xfull[s], (uint32_t)(it / NST) & 1u, p.backoff_ns);
      const bool duty = norms_on && duty_ctr == kt;
      if (++duty_ctr == p.k_tiles) duty_ctr = 0;
      if (duty) {
        const uint8_t* base = x_s + s * STG + box * 8192;
        uint4 v[NORM_ROWS];
#pragma unroll
        for (int rr = 0; rr < NORM_ROWS; ++rr) {
          const int r = rg + NORM_RG * rr;
          if (p.debug & 16)
            v[rr] = make_uint4(it * 3u + rr, it ^ rr, it + 7u, it * 5u);
          else
            v[rr] = *reinterpret_cast<const uint4*>(base + r * 128 + ((chunk ^ (r & 7)) << 4));
        }
        // exact fp32 squares (bf16 has 8 significant bits), summed over the
        // thread's NORM_ROWS rows in fp32, then one fp64 add per column
        // (R4: relative error <= 3·2^-24 worst case per chunk);
        // one FHFMA.BF16 per element (no unpack)
        float sq[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) sq[e] = 0.f;
#pragma unroll
        for (int rr = 0; rr < NORM_ROWS; ++rr) {
          const uint32_t w[4] = {v[rr].x, v[rr].y, v[rr].z, v[rr].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) fma_bf16x2_f32(w[e], w[e], sq[2 * e], sq[2 * e + 1]);
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] += (double)sq[e];
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&xempty[s]);
    }
    // norm partials: reduce the row groups in a fixed order
#pragma unroll
    for (int e = 0; e < 8; ++e) red[rg * HALF_N + box * 64 + chunk * 8 + e] = acc[e];
    named_bar_sync(1, 32 * NUM_NORM_WARPS);
    const int slot = split * p.k_tiles + kt;
    if (g < HALF_N) {
      double v = red[g];
#pragma unroll
      for (int w = 1; w < NORM_RG; ++w) v += red[w * HALF_N + g];
      if (n0 + g < p.n) p.pnorm[(int64_t)slot * p.n + n0 + g] = v;
    }
    // TMEM -> partial slot: warp quad owns lanes 32*quad..; the two warps of
    // a quad split the 256 accumulator columns
    const int quad = warp & 3;
    const int chalf = (warp - 8) >> 2;
    if (nkb > 0) {
      mbar_wait_backoff(tmem_full, 0, p.backoff_ns ? 4 * p.backoff_ns : 0);
      tc_fence_after();
    }
    const int kappa = kappa0 + 32 * quad + lane;
    const int ncol0 = nt * TC_BN;
    for (int cc = chalf * 4; cc < chalf * 4 + 4; ++cc) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tbase + ((uint32_t)(32 * quad) << 16) + cc * 32, r);
      tc_wait_ld();
      if (nkb == 0) {
#pragma unroll
        for (int j = 0; j < 32; ++j) r[j] = 0u;
      }
      if (kappa < p.k) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int col = ncol0 + cc * 32 + j;
          if (col < p.n) p.part[((int64_t)split * p.n + col) * p.k + kappa] = __uint_as_float(r[j]);
        }
      }
    }
  }
role_done:
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tbase, TMEM_COLS);
  }
}

// ---------------------------------------------------------------- Π panel
// panel[κ * ld + (t - t0)] = Π(κ, t) (bf16 bits) for κ < k, t in [t0, t0 + rows);
// thread per (κ, 4-row group): one Philox call for the Gaussian stream
// (DESIGN.md §3.2-3.3), 8 contiguous bytes written.
__global__ void pi_panel_kmajor_kernel(int kind, uint64_t seed, int k, int kpad, int64_t t0,
                                       int64_t rows, int64_t ld, uint16_t* __restrict__ panel) {
  // Rademacher: thread per (κ, 32-row word), one Philox call per 128 rows
  // (the word of DESIGN.md §3.3), 64 bytes written; otherwise thread per
  // (κ, 4-row group), one Philox call for the Gaussian stream, 8 bytes.
  // Gaussian, 8-aligned rows and pitch: thread per (κ, 8-row group), two
  // independent Philox calls in flight and one 16-byte store
  const int grp = (kind == PI_RADEMACHER && (t0 & 31) == 0) ? 32
                  : (kind == PI_GAUSSIAN && (t0 & 7) == 0 && (ld & 7) == 0) ? 8 : 4;
  const int64_t ng = (rows + grp - 1) / grp;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  // (e < 2^32 for any panel K1 uses: kpad <= 4096 and rows / grp < 2^20)
  const uint32_t ngu = (uint32_t)ng;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ng * kpad;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int kappa = (int)((uint32_t)e / ngu);
    const int64_t g = (int64_t)((uint32_t)e - (uint32_t)kappa * ngu);
    const int64_t t = t0 + grp * g;
    uint16_t* dst = panel + (int64_t)kappa * ld + grp * g;
    if (grp == 32) {
      uint32_t w32 = 0;
      if (kappa < k) {
        const uint64_t tg = (uint64_t)t >> 7;
        const u32x4 w = philox4x32_10((uint32_t)tg, (uint32_t)kappa, (uint32_t)(tg >> 32), TAG_RADEMACHER, k0, k1);
        const uint32_t wi = (uint32_t)((t >> 5) & 3);
        w32 = wi == 0 ? w.x : wi == 1 ? w.y : wi == 2 ? w.z : w.w;
      }
      uint32_t o[16];
#pragma unroll
      for (int q = 0; q < 16; ++q)  // rows 2q (bit q), 2q+1 (bit 16+q)
        o[q] = kappa < k ? (0x3F803F80u | ((w32 << (15 - q)) & 0x8000u) | ((w32 >> (16 + q)) << 31)) : 0u;
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int q = 0; q < 4; ++q) d4[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
      continue;
    }
    if (grp == 8) {
      uint4 v = make_uint4(0u, 0u, 0u, 0u);
      if (kappa < k) {
        const uint64_t tq = (uint64_t)t >> 2, tq1 = tq + 1;
        const u32x4 w0 = philox4x32_10((uint32_t)tq, (uint32_t)kappa, (uint32_t)(tq >> 32), TAG_GAUSSIAN, k0, k1);
        const u32x4 w1 = philox4x32_10((uint32_t)tq1, (uint32_t)kappa, (uint32_t)(tq1 >> 32), TAG_GAUSSIAN, k0, k1);
        v.x = gauss_pair_bits(w0.x, w0.y);
        v.y = gauss_pair_bits(w0.z, w0.w);
        v.z = gauss_pair_bits(w1.x, w1.y);
        v.w = gauss_pair_bits(w1.z, w1.w);
      }
      *reinterpret_cast<uint4*>(dst) = v;
      continue;
    }
    uint16_t z[4];
    if (kappa >= k) {
      z[0] = z[1] = z[2] = z[3] = 0;
    } else if (kind == PI_GAUSSIAN && (t & 3) == 0) {
      const uint64_t tq = (uint64_t)t >> 2;
      const u32x4 w = philox4x32_10((uint32_t)tq, (uint32_t)kappa, (uint32_t)(tq >> 32), TAG_GAUSSIAN, k0, k1);
      gauss_pair(w.x, w.y, z[0], z[1]);
      gauss_pair(w.z, w.w, z[2], z[3]);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) z[j] = pi_bits(kind, seed, (uint32_t)kappa, (uint64_t)(t + j));
    }
    if ((ld & 3) == 0) {
      uint2 v;
      v.x = (uint32_t)z[0] | ((uint32_t)z[1] << 16);
      v.y = (uint32_t)z[2] | ((uint32_t)z[3] << 16);
      *reinterpret_cast<uint2*>(dst) = v;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) dst[j] = z[j];
    }
  }
}

cudaError_t launch_pi_panel_kmajor(int kind, uint64_t seed, int k, int kpad, int64_t t0, int64_t rows,
                                   int64_t ld, uint16_t* panel, cudaStream_t st, int blocks_per_sm) {
  // blocks_per_sm = 1: a background launch that leaves every SM room for a
  // K1F CTA beside it (256 threads x 40 registers next to K1F's 768 x 72)
  const int64_t tot = ((rows + 3) / 4) * kpad;  // upper bound on threads needed (grid-stride loop)
  const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * (blocks_per_sm > 0 ? blocks_per_sm : 16));
  pi_panel_kmajor_kernel<<<blocks, 256, 0, st>>>(kind, seed, k, kpad, t0, rows, ld, panel);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

#ifdef SMP_K1_TRACE
extern "C" __attribute__((visibility("default"))) int smp_debug_k1_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_k1_trace, sizeof(g_k1_trace));
}
#endif

int sketch_tc_smem_bytes() { return TC_SMEM; }
int sketch_tc_ctas_per_tile() { return 2; }

cudaError_t launch_sketch_tc(const void* X, int64_t ldx, SketchTCParams p, cudaStream_t st) {
  auto enc = get_encode_fn();
  if (!enc) return cudaErrorNotSupported;
  CUtensorMap tmap, tmap_pi;
  {
    cuuint64_t dims[2] = {(cuuint64_t)p.n, (cuuint64_t)p.rows};
    cuuint64_t strides[1] = {(cuuint64_t)ldx * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(X), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  }
  const bool panel = p.pi_panel != nullptr;
  if (panel) {
    // κ-major panel [k_tiles * 256][pi_ld]: box = 64 t (128 B, swizzled) x 128 κ
    cuuint64_t dims[2] = {(cuuint64_t)p.pi_ld, (cuuint64_t)p.k_tiles * 256};
    cuuint64_t strides[1] = {(cuuint64_t)p.pi_ld * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmap_pi, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<uint16_t*>(p.pi_panel),
                     dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  } else {
    tmap_pi = tmap;
  }
  // generator sets: 3 when several κ tiles share each X tile (see GS above);
  // SMP_K1_GEN_SETS = 2..4 overrides (tuning only)
  int gs = (!panel && p.k_tiles >= 2) ? 3 : 2;
  if (const char* e = getenv("SMP_K1_GEN_SETS")) {
    const int v = atoi(e);
    if (v >= 2 && v <= MAX_GEN_SETS) gs = v;
  }
  if (panel) gs = 2;  // Π arrives by TMA: the generator warps idle
  static PerDeviceOnce attr_set[4];
  const int smem = panel ? P_SMEM : TC_SMEM;
  const void* fn = panel ? (const void*)sketch_tc_kernel<true, 2>
                   : gs == 2 ? (const void*)sketch_tc_kernel<false, 2>
                   : gs == 3 ? (const void*)sketch_tc_kernel<false, 3>
                             : (const void*)sketch_tc_kernel<false, 4>;
  if (attr_set[panel ? 0 : gs - 1].need()) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2u * (unsigned)(p.n_tiles * p.k_tiles * p.splits));
  cfg.blockDim = dim3((unsigned)tc_threads(gs));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {(void*)&tmap, (void*)&tmap_pi, (void*)&p};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

}  // namespace smp
