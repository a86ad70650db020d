// Device-side building blocks for the SMP-PCA sm_100a kernels:
//   * Philox4x32-10 counter hash and the Π generators of
//     Alg. 1 line 2 — Rademacher, Gaussian (DESIGN.md
//     §3.2 fp32 Box–Muller), Hadamard test mode;
//   * thin inline-PTX wrappers for mbarrier, TMA (cp.async.bulk.tensor),
//     tcgen05 (alloc / mma / commit / ld) used by the dense sketch kernel.
// Nothing here is shared with the CPU oracle (oracle/smp_oracle.c), which
// re-implements the same written definitions independently.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace smp {

// cudaFuncSetAttribute is a per-device setting: remember, per call site, the
// devices it has been applied to (a process may drive several GPUs).
struct PerDeviceOnce {
  unsigned long long mask = 0;
  bool need() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return true;
    const unsigned long long bit = 1ull << dev;
    if (mask & bit) return false;
    mask |= bit;
    return true;
  }
};


// ---------------------------------------------------------------- hash
struct u32x4 { uint32_t x, y, z, w; };

__device__ __forceinline__ u32x4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2,
                                               uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return {c0, c1, c2, c3};
}

enum : int { PI_RADEMACHER = 0, PI_GAUSSIAN = 1, PI_HADAMARD = 2, PI_SRHT_BASE = 16 };

// Stream tags (c3 of the Philox counter), DESIGN.md §3.1.
enum : uint32_t { TAG_RADEMACHER = 1, TAG_GAUSSIAN = 2, TAG_OMEGA = 3, TAG_PART = 4, TAG_INIT = 5, TAG_SRHT_D = 6,
                  TAG_SRHT_S = 7 };

// ---------------------------------------------------------------- SRHT
// Π(κ, t) = D_t (−1)^popcount(s_κ & t) (R26; kind code 16 + L):
// s_κ = F_L(κ), a 4-round unbalanced Feistel bijection of [0, 2^L) whose
// round function is word 0 of Philox(ctr = (v, round, L, 7)); D_t from
// stream 6 in the Rademacher bit layout.
__device__ __forceinline__ uint64_t srht_row(uint64_t seed, int L, uint32_t kappa);
__device__ __forceinline__ uint32_t walsh32_interleaved(uint32_t s5) {
  // bit at (j >> 1) | ((j & 1) << 4) = parity(s5 & j), j = 0..31
  uint32_t w = 0;
#pragma unroll
  for (int j = 0; j < 32; ++j)
    w |= (uint32_t)(__popc(s5 & (uint32_t)j) & 1) << ((j >> 1) | ((j & 1) << 4));
  return w;
}

// ---------------------------------------------------------------- Gaussian G
// fp32 Box–Muller with stated polynomials.  Every operation
// is an explicitly rounded intrinsic so that nvcc cannot contract or
// reassociate: the bits must equal the oracle's.
__device__ __forceinline__ uint16_t bf16_rne_bits(float x) {
  uint32_t u = __float_as_uint(x);
  uint32_t lsb = (u >> 16) & 1u;
  return (uint16_t)((u + 0x7FFFu + lsb) >> 16);
}

// (z1 << 16) | z0 of G(wa, wb); z = bf16_rne(ρ·c), bf16_rne(ρ·s)
// by one cvt.rn.bf16x2.f32 (round to nearest even, as bf16_rne_bits: the
// products are finite)
__device__ __forceinline__ uint32_t gauss_pair_bits(uint32_t wa, uint32_t wb) {
  const float L0 = 0x1.000000p+0f, L1 = -0x1.000000p-1f, L2 = 0x1.5555c6p-2f,
              L3 = -0x1.00003ep-2f, L4 = 0x1.996178p-3f, L5 = -0x1.54e596p-3f,
              L6 = 0x1.28ce66p-3f, L7 = -0x1.0e2b8ep-3f, L8 = 0x1.ac49bap-4f,
              L9 = -0x1.6e4bbap-5f;
  const float LN2 = 0x1.62e430p-1f;
  const float S1 = 0x1.921fb6p+0f, S3 = -0x1.4abbcep-1f, S5 = 0x1.466bc6p-4f,
              S7 = -0x1.32d2ccp-8f, S9 = 0x1.507834p-13f;
  const float C2 = -0x1.3bd3ccp+0f, C4 = 0x1.03c1f0p-2f, C6 = -0x1.55d3c8p-6f,
              C8 = 0x1.e1f506p-11f, C10 = -0x1.a6d1f2p-16f;
  // u1 = ((wa>>8)+1) 2^-24 in (0,1]: exponent/mantissa split, f in [0.75,1.5)
  uint32_t v1 = (wa >> 8) + 1u;
  float u1 = __fmul_rn(__uint2float_rn(v1), 0x1p-24f);
  uint32_t bits = __float_as_uint(u1);
  int e = (int)(bits >> 23) - 127;
  uint32_t mant = bits & 0x7FFFFFu;
  float f;
  if (mant >= 0x400000u) { f = __uint_as_float(mant | 0x3F000000u); e += 1; }
  else { f = __uint_as_float(mant | 0x3F800000u); }
  float y = __fsub_rn(f, 1.0f);
  float p = L9;
  p = __fmaf_rn(p, y, L8); p = __fmaf_rn(p, y, L7); p = __fmaf_rn(p, y, L6);
  p = __fmaf_rn(p, y, L5); p = __fmaf_rn(p, y, L4); p = __fmaf_rn(p, y, L3);
  p = __fmaf_rn(p, y, L2); p = __fmaf_rn(p, y, L1); p = __fmaf_rn(p, y, L0);
  float lnf = __fmul_rn(y, p);
  float lnu = __fmaf_rn(__int2float_rn(e), LN2, lnf);
  float r2 = __fmul_rn(-2.0f, lnu);
  float rho = __fsqrt_rn(r2);
  uint32_t v2 = wb >> 8;
  uint32_t qn = (v2 + 0x200000u) >> 22;
  int32_t xi = (int32_t)v2 - (int32_t)(qn << 22);
  float x = __fmul_rn(__int2float_rn(xi), 0x1p-22f);
  float x2 = __fmul_rn(x, x);
  float sp = __fmaf_rn(__fmaf_rn(__fmaf_rn(__fmaf_rn(S9, x2, S7), x2, S5), x2, S3), x2, S1);
  float sn = __fmul_rn(x, sp);
  float cs = __fmaf_rn(__fmaf_rn(__fmaf_rn(__fmaf_rn(__fmaf_rn(C10, x2, C8), x2, C6), x2, C4), x2, C2), x2, 1.0f);
  // rotate by the quadrant (branch-free; negation is exact, so the values
  // equal the case analysis (cs, sn), (−sn, cs), (−cs, −sn), (sn, −cs))
  const uint32_t qq = qn & 3u;
  const float a = (qq & 1u) ? sn : cs;
  const float b = (qq & 1u) ? cs : sn;
  const float c = ((qq + 1u) & 2u) ? -a : a;
  const float s = (qq & 2u) ? -b : b;
  const float p0 = __fmul_rn(rho, c), p1 = __fmul_rn(rho, s);
  uint32_t z;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(z) : "f"(p1), "f"(p0));
  return z;
}

__device__ __forceinline__ void gauss_pair(uint32_t wa, uint32_t wb, uint16_t& z0, uint16_t& z1) {
  const uint32_t z = gauss_pair_bits(wa, wb);
  z0 = (uint16_t)(z & 0xFFFFu);
  z1 = (uint16_t)(z >> 16);
}

__device__ __forceinline__ uint64_t srht_row(uint64_t seed, int L, uint32_t kappa) {
  const int a = L / 2, b = L - a;
  const uint64_t mb = (1ull << b) - 1ull, ma = (1ull << a) - 1ull;
  uint64_t lo = (uint64_t)kappa & mb, hi = ((uint64_t)kappa >> b) & ma;
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    if ((r & 1) == 0) hi ^= (uint64_t)philox4x32_10((uint32_t)lo, (uint32_t)r, (uint32_t)L, TAG_SRHT_S, k0, k1).x & ma;
    else lo ^= (uint64_t)philox4x32_10((uint32_t)hi, (uint32_t)r, (uint32_t)L, TAG_SRHT_S, k0, k1).x & mb;
  }
  return (hi << b) | lo;
}

// Unscaled Π(κ, t) as bf16 bits (used by the SIMT/CSR paths and tests).
__device__ __forceinline__ uint16_t pi_bits(int kind, uint64_t seed, uint32_t kappa, uint64_t t) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  if (kind == PI_RADEMACHER) {
    u32x4 w = philox4x32_10((uint32_t)(t >> 7), kappa, (uint32_t)(t >> 39), TAG_RADEMACHER, k0, k1);
    uint32_t b = (uint32_t)(t & 127), e = b & 31;
    uint32_t word = (b >> 5) == 0 ? w.x : (b >> 5) == 1 ? w.y : (b >> 5) == 2 ? w.z : w.w;
    uint32_t pos = (e >> 1) | ((e & 1u) << 4);
    return ((word >> pos) & 1u) ? (uint16_t)0xBF80 : (uint16_t)0x3F80;
  } else if (kind == PI_GAUSSIAN) {
    u32x4 w = philox4x32_10((uint32_t)(t >> 2), kappa, (uint32_t)(t >> 34), TAG_GAUSSIAN, k0, k1);
    uint16_t z0, z1;
    if ((t & 3) < 2) gauss_pair(w.x, w.y, z0, z1); else gauss_pair(w.z, w.w, z0, z1);
    return (t & 1) ? z1 : z0;
  } else if (kind >= PI_SRHT_BASE) {
    const uint64_t sk = srht_row(seed, kind - PI_SRHT_BASE, kappa);
    const u32x4 w = philox4x32_10((uint32_t)(t >> 7), 0u, (uint32_t)(t >> 39), TAG_SRHT_D, k0, k1);
    const uint32_t b = (uint32_t)(t & 127), e = b & 31;
    const uint32_t word = (b >> 5) == 0 ? w.x : (b >> 5) == 1 ? w.y : (b >> 5) == 2 ? w.z : w.w;
    const uint32_t dbit = (word >> ((e >> 1) | ((e & 1u) << 4))) & 1u;
    const uint32_t hbit = (uint32_t)__popcll((unsigned long long)(sk & t)) & 1u;
    return (dbit ^ hbit) ? (uint16_t)0xBF80 : (uint16_t)0x3F80;
  } else {
    return (__popcll((unsigned long long)kappa & t) & 1) ? (uint16_t)0xBF80 : (uint16_t)0x3F80;
  }
}

__device__ __forceinline__ float bf16_bits_to_float(uint32_t b) { return __uint_as_float(b << 16); }

// ---------------------------------------------------------------- mixed-precision FMA
// acc + lo(x)·lo(y) and acc + hi(x)·hi(y) for packed bf16 pairs, accumulated
// in fp32 with one rounding (fma.rn.f32.bf16 -> FHFMA.BF16 with .H0/.H1
// operand selection: no unpack instructions).  A bf16 × bf16 product has at
// most 16 significant bits, so it is exact and each step equals
// fmaf(float(a), float(b), acc) bit for bit.
__device__ __forceinline__ void fma_bf16x2_f32(uint32_t x, uint32_t y, float& acc_lo, float& acc_hi) {
  asm("{\n\t.reg .b16 xl, xh, yl, yh;\n\t"
      "mov.b32 {xl, xh}, %2;\n\tmov.b32 {yl, yh}, %3;\n\t"
      "fma.rn.f32.bf16 %0, xl, yl, %0;\n\tfma.rn.f32.bf16 %1, xh, yh, %1;\n\t}"
      : "+f"(acc_lo), "+f"(acc_hi)
      : "r"(x), "r"(y));
}
// acc + v·lo(y), acc + v·hi(y) for a bf16 scalar v (in the low half of vb)
__device__ __forceinline__ void fma_bf16s_x2_f32(uint32_t vb, uint32_t y, float& acc_lo, float& acc_hi) {
  asm("{\n\t.reg .b16 vl, vh, yl, yh;\n\t"
      "mov.b32 {vl, vh}, %2;\n\tmov.b32 {yl, yh}, %3;\n\t"
      "fma.rn.f32.bf16 %0, vl, yl, %0;\n\tfma.rn.f32.bf16 %1, vl, yh, %1;\n\t}"
      : "+f"(acc_lo), "+f"(acc_hi)
      : "r"(vb), "r"(y));
}

// ---------------------------------------------------------------- PTX: misc
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

// ---------------------------------------------------------------- mbarrier
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: the warp is parked by the hardware
// until the phase completes (or the hint expires) instead of re-issuing the
// test in a loop — a spinning warp costs issue slots and power that the
// generator, norm and MMA warps sharing the SM need.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
#ifdef SMP_MBAR_NOSUSPEND
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
      "r"(parity), "r"(0x989680u)
      : "memory");
#endif
}

// Warp-wide wait with ONE polling lane: lane 0 tests the barrier (predicated
// inside the asm, so the warp never diverges), the result is broadcast with a
// shuffle, and once the phase has completed every lane observes it itself
// with a single test (the acquire each reader of TMA-written data needs).
// 32 lanes polling one mbarrier are 32 requests to the SM's barrier unit per
// test; the TMA's complete_tx updates and tcgen05.commit arrivals queue behind
// them.  All 32 lanes of the warp must call it.
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred P1, P2;\n\t"
        "setp.eq.u32 P2, %3, 0;\n\t"
        "mov.u32 %0, 0;\n\t"
        "@P2 mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %4;\n\t"
        "@P2 selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(lane), "r"(0x989680u)
        : "memory");
    ok = __shfl_sync(0xffffffffu, ok, 0);
  } while (!ok);
  mbar_wait(bar, parity);
}

// Wait with a back-off for warps whose wait is off the critical path (they
// sit ahead of a deep ring): one non-suspending test, then __nanosleep(ns)
// between tests, so that a parked warp stops taking issue slots from the
// warps that feed the tensor core (measured: spinning waiters were ~28% of
// K1's issued instructions on cfg2).  ns = 0 is mbar_wait.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, uint32_t ns) {
  if (ns == 0) { mbar_wait(bar, parity); return; }
  while (!mbar_test(bar, parity)) __nanosleep(ns);
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// ---------------------------------------------------------------- tcgen05
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 in, fp32 accumulate)
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns -> 32 registers per thread
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// ---------------------------------------------------------------- clusters / CTA pairs
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
// Arrive on an mbarrier of another CTA of the cluster.  Default (.cta-scope)
// release, as CUTLASS's ClusterBarrier::arrive(cta_id): the data it
// publishes was already made visible through the async proxy (TMA
// complete_tx, tcgen05.wait::st + fence), and a .cluster-scope release costs
// a full memory barrier (ERRBAR) per arrival.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// Remote arrive with cluster-scope release: publishes this CTA's generic-
// proxy SMEM writes (fenced to the async proxy) to the peer's MMA.
__device__ __forceinline__ void mbar_arrive_cluster_release(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
// D[tmem] (+)= A[tmem] * B[smem] across the CTA pair (M = 256), kind::f16
__device__ __forceinline__ void tc_mma2_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// D[tmem] (+)= A[smem] * B[smem] across the CTA pair (M = 256; each CTA
// supplies its 128 rows of A and half of B's N columns), kind::f16
__device__ __forceinline__ void tc_mma2_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// commit all prior MMAs of this thread; arrive on the barrier at the same
// offset in every CTA of cta_mask
__device__ __forceinline__ void tc_commit2(uint64_t* bar, uint16_t cta_mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(cta_mask)
      : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive 32-bit columns <- 32 registers per thread
__device__ __forceinline__ void tmem_st_32x32b_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_32x32b_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

// Shared-memory matrix descriptor (tcgen05 "version 1"), SWIZZLE_128B.
//   start>>4 in [0,14), LBO>>4 in [16,30), SBO>>4 in [32,46), version=1 at 46,
//   layout type 2 (SWIZZLE_128B) in [61,64).
__device__ __forceinline__ uint64_t make_sdesc_sw128(uint32_t saddr, uint32_t lbo_bytes,
                                                     uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor, kind::f16: D fp32, A/B bf16, A K-major, B MN-major.
__host__ __device__ constexpr uint32_t make_idesc_bf16(uint32_t M, uint32_t N, uint32_t a_mn,
                                                       uint32_t b_mn) {
  return (1u << 4)            // D format F32
         | (1u << 7)          // A format BF16
         | (1u << 10)         // B format BF16
         | (a_mn << 15)       // A major
         | (b_mn << 16)       // B major
         | ((N >> 3) << 17)   // N
         | ((M >> 4) << 24);  // M
}

}  // namespace smp
