// WAltMin persistent kernel (Alg. 2), templated on the
// rank r; instantiated in waltmin_r*.cu (split for parallel compilation) and
// driven by run_waltmin() in waltmin.cu.
#pragma once
#include <cstdlib>
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

#ifndef SMP_TRY
#define SMP_TRY(x)                          \
  do {                                      \
    cudaError_t e_ = (x);                   \
    if (e_ != cudaSuccess) return e_;       \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// The whole of Alg. 2 after the CSR/CSC setup runs as ONE cooperative
// persistent kernel (one CTA per SM, grid-wide barriers between phases):
// at n <= 10^4, r <= 16 every phase is latency-bound, so launch count and
// the number of grid-wide synchronisations are what the time is made of.
//
// Row ownership: warp gw (global) owns output rows o = gw, gw + W, ... of
// every phase, W = total warps — deterministic, so every reduction below
// has a fixed order and the result is bit-reproducible run to run.
//
// Orthonormalisation is CholeskyQR2 with the Gram partials reduced by EVERY
// CTA redundantly in the same fixed order (identical R^{-1} everywhere, no
// second barrier); the second triangular factor is folded into the next
// SpMM's output (Σ c (x T) = (Σ c x) T), so each half-iteration of the
// subspace iteration costs two grid barriers.
constexpr int WM_THREADS = 256;
constexpr int WM_HEAVY = 1024;  // minimum samples for a row to be split over a CTA
constexpr int WM_WARPS = WM_THREADS / 32;

struct WMParams {
  int64_t n1, n2;
  int T, init_iters;
  double trim_c, lam;
  uint64_t seed;
  const int64_t* rptr;   // CSR (Ω in (i,j) order): row pointers
  const int32_t* J;      //   column of each sample
  const double* w;       //   w = 1/q̂
  const double* wv;      //   w · M̃
  const int64_t* cptr;   // CSC copy (stable by j): column pointers
  const int32_t* cI;     //   row of each sample
  const double* cw;
  const double* cwv;
  const double* a2;
  const double* FA;
  double* Y;
  double* Z;
  double* U;
  double* V;
  double* gpart;  // [2][gridDim.x][NG]
  unsigned* bar;  // [2]: arrival count, generation
  uint64_t* trace;  // optional [4 * barriers] (SMP_WM_TRACE)
  uint64_t* trace2; // optional [64] phase stamps of CTA 0 (SMP_WM_TRACE)
  int stage_x;      // gathered factor rows staged into SMEM per phase (fits: n·r·8 B small)
  // heavy rows (> WM_HEAVY samples): compacted lists, counts, per-row flags
  int x_l1;         // gathers of non-staged factor rows through L1 (else L2-only)
  const int32_t* heavy_r;
  const int32_t* nheavy_r;
  const uint8_t* hflag_r;
  const int32_t* heavy_c;
  const int32_t* nheavy_c;
  const uint8_t* hflag_c;
  int64_t count;        // |Ω|
  int64_t cache_bytes;  // dynamic SMEM reserved for the two WMCache copies (0: off)
  // FRESH_2T1 (Alg. 2 line 3): phase ph (0 = init, 2t+1 = V-solve t,
  // 2t+2 = U-solve t) reads rptr + ph·rstride / cptr + ph·cstride (positions
  // into the subset-major sample arrays); 0 = REUSE_ALL (every phase, all of Ω)
  int64_t rstride, cstride;
  // tuning switches, read per call by the host (SMP_WM_STAGE / _CACHE / _CTAS)
  int env_stage, env_cache, env_ctas;
  float* Uout;
  float* Vout;
};

__device__ __forceinline__ uint64_t wm_globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Grid barrier on one monotonically increasing arrival counter (all CTAs are
// co-resident: cooperative launch; the counter is zeroed before the launch).
// Barrier nb completes when the counter reaches (nb + 1)·grid: thread 0
// arrives with a release reduction (orders the CTA's writes, published to it
// by the bar.sync before) and polls with acquire loads (orders the CTA's
// later reads after the other CTAs' writes).  No generation word, no reset,
// one L2 round trip from the last arrival to the release.
// trace (diagnostics, SMP_WM_TRACE): per barrier, CTA 0's arrival, the last
// arrival, CTA 0's release (globaltimer ns) and the last arriving CTA.
__device__ __forceinline__ void grid_sync(unsigned* bar, uint64_t* trace, int& nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned target = (unsigned)(nb + 1) * gridDim.x;
    if (trace) {
      if (blockIdx.x == 0) trace[4 * nb] = wm_globaltimer();
      unsigned old;
      asm volatile("atom.release.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(bar) : "memory");
      if (old == target - 1) {
        trace[4 * nb + 1] = wm_globaltimer();
        trace[4 * nb + 3] = blockIdx.x;
      }
    } else {
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
    }
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
    } while (v < target);
    if (trace && blockIdx.x == 0) trace[4 * nb + 2] = wm_globaltimer();
  }
  ++nb;
  __syncthreads();
}

// SMEM copy of one side of Ω restricted to the light rows this CTA owns
// (row o belongs to warp (o mod W) mod 8 of CTA (o mod W) / 8, W = 8·grid):
// the sample structure is the same in every phase, so after one copy the
// phases read their indices and weights from SMEM instead of L2 (the
// per-row latency that dominates small instances such as cfg1).
struct WMCache {
  int on;
  int soff[WM_WARPS];  // warp's first sample
  int roff[WM_WARPS];  // warp's first row-length entry (-1: heavy row, skipped)
  const int32_t* other;
  const double* w;
  const double* wv;
  const int32_t* len;
};

template <int R>
struct WMShared {
  static constexpr int NG = R * (R + 1) / 2;
  double T[R * R];            // current right factor (upper triangular), applied to outputs
  double Rinv[R * R];         // result of the last Cholesky
  double G[R * R];
  double red[WM_THREADS];     // reduction scratch
  double wg[WM_WARPS][NG];    // per-warp Gram partials
  double ys[WM_WARPS][R];     // per-warp row broadcast
  double hred[WM_WARPS][R * (R + 1) / 2 + R];  // heavy-row partials (SpMM: first R)
  int ea[NG], eb[NG];
  WMCache cache[2];           // [0]: rows of U/Z (CSR side), [1]: rows of V/Y (CSC side)
  int scan[2][WM_WARPS];
  int nh[2];                  // heavy-row counts (constant during the kernel)
};

template <int R>
__device__ __forceinline__ void set_identity(double* T) {
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) T[e] = (e / R == e % R) ? 1.0 : 0.0;
}

// y = acc · T (T upper triangular; T == nullptr: identity); rows whose norm
// exceeds trim_thr (if >= 0) are zeroed; y -> out row o; Gram partial += y yᵀ
template <int R>
__device__ __forceinline__ void emit_row(WMShared<R>& sm, int64_t o, const double (&acc)[R],
                                         const double* T, double* out, double trim_thr,
                                         double (&gl)[(WMShared<R>::NG + 31) / 32]) {
  constexpr int NG = WMShared<R>::NG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double y[R];
#pragma unroll
  for (int c = 0; c < R; ++c) {
    if (T) {
      double t = 0.0;
#pragma unroll
      for (int m = 0; m <= c; ++m) t = fma(acc[m], T[m * R + c], t);
      y[c] = t;
    } else {
      y[c] = acc[c];
    }
  }
  if (trim_thr >= 0.0) {
    double rn = 0.0;
#pragma unroll
    for (int c = 0; c < R; ++c) rn += y[c] * y[c];
    if (sqrt(rn) > trim_thr) {
#pragma unroll
      for (int c = 0; c < R; ++c) y[c] = 0.0;
    }
  }
  __syncwarp();
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < R; ++c) {
      out[o * R + c] = y[c];
      sm.ys[warp][c] = y[c];
    }
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < (NG + 31) / 32; ++q) {
    const int e = lane + 32 * q;
    if (e < NG) gl[q] = fma(sm.ys[warp][sm.ea[e]], sm.ys[warp][sm.eb[e]], gl[q]);
  }
  __syncwarp();
}

// per-warp Gram partials -> gpart[buf][cta] (fixed warp order)
template <int R>
__device__ __forceinline__ void flush_gram(WMShared<R>& sm, const double (&gl)[(WMShared<R>::NG + 31) / 32],
                                           double* gpart_buf) {
  constexpr int NG = WMShared<R>::NG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int q = 0; q < (NG + 31) / 32; ++q) {
    const int e = lane + 32 * q;
    if (e < NG) sm.wg[warp][e] = gl[q];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < NG; e += blockDim.x) {
    double s = 0.0;
    for (int w = 0; w < WM_WARPS; ++w) s += sm.wg[w][e];
    gpart_buf[(int64_t)blockIdx.x * NG + e] = s;
  }
}

// upper Cholesky of the reduced Gram sm.G = RᵀR and out = R^{-1} (one thread)
template <int R>
__device__ __noinline__ void chol_rinv(const WMShared<R>& sm, double* out) {
  // upper Cholesky G = RᵀR (L = Rᵀ), then Rinv = (Lᵀ)^{-1}; dead pivots
  // (rank deficiency) give zero columns.  Fully unrolled: registers only.
  double L[R][R], Ri[R][R], inv[R];
  bool dead[R];
  double tr = 0.0;
  {
    int e = 0;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = a; b < R; ++b) {
        L[b][a] = sm.G[e];  // lower triangle holds G
        if (a == b) tr += sm.G[e];
        ++e;
      }
  }
  const double tol = 1e-28 * (tr > 0.0 ? tr : 1.0);
#pragma unroll
  for (int j = 0; j < R; ++j) {
    double s = L[j][j];
#pragma unroll
    for (int q = 0; q < j; ++q) s -= L[j][q] * L[j][q];
    dead[j] = !(s > tol);
    const double d = dead[j] ? 0.0 : sqrt(s);
    inv[j] = dead[j] ? 0.0 : 1.0 / d;
    L[j][j] = d;
#pragma unroll
    for (int i = j + 1; i < R; ++i) {
      double t = L[i][j];
#pragma unroll
      for (int q = 0; q < j; ++q) t -= L[i][q] * L[j][q];
      L[i][j] = t * inv[j];
    }
  }
  // Ri = (Lᵀ)^{-1} (upper): back substitution per column c
#pragma unroll
  for (int c = 0; c < R; ++c)
#pragma unroll
    for (int i = R - 1; i >= 0; --i) {
      double t = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int q = i + 1; q < R; ++q) t -= L[q][i] * Ri[q][c];
      Ri[i][c] = (dead[i] || dead[c]) ? 0.0 : t * inv[i];
    }
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int c = 0; c < R; ++c) out[i * R + c] = Ri[i][c];
}

// G = Σ_cta gpart[buf][cta] (identical fixed order in every CTA), then
// R^{-1} of the upper Cholesky factor into sm.Rinv (dead pivots -> zero columns)
// Optionally also stages X[0 .. sn) into xs (see stage_rows): its first
// chunk of loads is issued together with the Gram loads (one L2 round trip
// for both on small instances).
template <int R>
__device__ void reduce_chol(WMShared<R>& sm, const double* gpart_buf, const double* SX = nullptr,
                            int64_t sn = 0, double* xs = nullptr, bool do_chol = true) {
  constexpr int NG = WMShared<R>::NG;
  constexpr int MAXK = 16;  // independent loads in flight per thread (one L2 round trip at r <= 6)
  constexpr int SU = 8;     // stage loads (16 B) per thread in the first chunk
  const int G = gridDim.x;
  const int groups = blockDim.x / NG;  // >= 1 for NG <= 136 < 256
  const int tid = threadIdx.x;
  const int64_t tot2 = SX ? (sn * R) / 2 : 0;
  const double2* src2 = reinterpret_cast<const double2*>(SX);
  double2 sv[SU];
#pragma unroll
  for (int u = 0; u < SU; ++u) {
    const int64_t e = tid + (int64_t)u * blockDim.x;
    sv[u] = e < tot2 ? __ldcg(src2 + e) : make_double2(0.0, 0.0);
  }
  if (tid < groups * NG) {
    // thread (g, e) sums CTAs b = g, g + groups, ... in increasing order
    const int e = tid % NG, g = tid / NG;
    double s = 0.0;
    for (int base = g; base < G; base += groups * MAXK) {
      double v[MAXK];
#pragma unroll
      for (int q = 0; q < MAXK; ++q) {
        const int b = base + groups * q;
        v[q] = b < G ? __ldcg(gpart_buf + (int64_t)b * NG + e) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < MAXK; ++q) s += v[q];
    }
    sm.red[tid] = s;
  }
  if (SX) {
    double2* dst = reinterpret_cast<double2*>(xs);
#pragma unroll
    for (int u = 0; u < SU; ++u) {
      const int64_t e = tid + (int64_t)u * blockDim.x;
      if (e < tot2) dst[e] = sv[u];
    }
    // the rest (large stages) in batches of SU loads in flight, as stage_rows
    for (int64_t b = tid + (int64_t)SU * blockDim.x; b < tot2; b += (int64_t)SU * blockDim.x) {
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int64_t e = b + (int64_t)u * blockDim.x;
        sv[u] = e < tot2 ? __ldcg(src2 + e) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < SU; ++u) {
        const int64_t e = b + (int64_t)u * blockDim.x;
        if (e < tot2) dst[e] = sv[u];
      }
    }
    if (((sn * R) & 1) && tid == 0) xs[sn * R - 1] = __ldcg(SX + sn * R - 1);
  }
  __syncthreads();
  if (tid < NG) {
    double s = 0.0;
    for (int g = 0; g < groups; ++g) s += sm.red[g * NG + tid];
    sm.G[tid] = s;  // packed upper triangle, row-major (ea/eb order)
  }
  __syncthreads();
  if (!do_chol) return;  // caller overlaps chol_rinv with other work
  if (tid == 0) chol_rinv<R>(sm, sm.Rinv);
  __syncthreads();
}

// Loops are fully unrolled (register-resident arrays) for r <= 10 — the
// ranks of the configured workloads — and left rolled above that to bound
// code size and compile time.
// loads in flight per lane in the sample loops (memory-level parallelism
// against the L2 latency of the gathered X rows; fewer for large r to bound
// registers)
template <int R>
struct WMUnroll { static constexpr int U = R <= 6 ? 4 : (R <= 10 ? 2 : 1); };

// Fill sm.cache[sd] for this CTA's light rows of one side, if they fit in
// the remaining region [*region, end); all threads of the CTA call this.
static __device__ void build_cache(WMCache& c, int (&scan)[2][WM_WARPS], const int64_t* __restrict__ ptr,
                            const int32_t* __restrict__ other, const double* __restrict__ w,
                            const double* __restrict__ wv, int64_t nout, const uint8_t* hflag,
                            uint8_t*& region, const uint8_t* end) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * WM_WARPS;
  const int64_t o0 = (int64_t)blockIdx.x * WM_WARPS + warp;
  const int nrows = o0 < nout ? (int)((nout - 1 - o0) / W + 1) : 0;
  int64_t ns = 0;
  for (int k = lane; k < nrows; k += 32) {
    const int64_t o = o0 + (int64_t)k * W;
    if (!(hflag && hflag[o])) ns += ptr[o + 1] - ptr[o];
  }
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, sh);
  if (lane == 0) { scan[0][warp] = (int)(ns < (1 << 30) ? ns : (1 << 30)); scan[1][warp] = nrows; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t S = 0, Rr = 0;
    for (int q = 0; q < WM_WARPS; ++q) {
      c.soff[q] = (int)S; c.roff[q] = (int)Rr;
      S += scan[0][q]; Rr += scan[1][q];
    }
    const int64_t bytes = S * 16 + ((S * 4 + Rr * 4 + 15) & ~(int64_t)15);
    c.on = (region + bytes <= end) ? 1 : 0;
    if (c.on) {
      double* d = reinterpret_cast<double*>(region);
      c.w = d;
      c.wv = d + S;
      int32_t* i = reinterpret_cast<int32_t*>(d + 2 * S);
      c.other = i;
      c.len = i + S;
      region += bytes;
    }
  }
  __syncthreads();
  if (!c.on) return;
  double* cw = const_cast<double*>(c.w);
  double* cwv = const_cast<double*>(c.wv);
  int32_t* co = const_cast<int32_t*>(c.other);
  int32_t* cl = const_cast<int32_t*>(c.len);
  int64_t q = c.soff[warp];
  for (int k = 0; k < nrows; ++k) {
    const int64_t o = o0 + (int64_t)k * W;
    const bool hv = hflag && hflag[o];
    const int64_t p0 = ptr[o], p1 = ptr[o + 1];
    if (lane == 0) cl[c.roff[warp] + k] = hv ? -1 : (int)(p1 - p0);
    if (hv) continue;
    for (int64_t e = p0 + lane; e < p1; e += 32) {
      const int64_t t = q + (e - p0);
      co[t] = other[e];
      cw[t] = w[e];
      cwv[t] = wv[e];
    }
    q += p1 - p0;
  }
  __syncthreads();
}

// Copy the factor rows X[0 .. n) (n·R doubles, written by other CTAs before
// the last grid barrier) into this CTA's SMEM, so that the phase's gathers —
// one per sample, the latency-critical part — are SMEM reads, not L2 trips.
template <int R>
__device__ __forceinline__ const double* stage_rows(const double* X, int64_t n, double* xs, bool on) {
  if (!on) return nullptr;
  // 16-byte loads, 8 in flight per thread (one L2 round trip for ~32 KB)
  const int64_t tot2 = (n * R) / 2;
  const double2* src = reinterpret_cast<const double2*>(X);
  double2* dst = reinterpret_cast<double2*>(xs);
  for (int64_t b = threadIdx.x; b < tot2; b += 8 * (int64_t)blockDim.x) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = b + (int64_t)u * blockDim.x;
      v[u] = e < tot2 ? __ldcg(src + e) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t e = b + (int64_t)u * blockDim.x;
      if (e < tot2) dst[e] = v[u];
    }
  }
  if (((n * R) & 1) && threadIdx.x == 0) xs[n * R - 1] = __ldcg(X + n * R - 1);
  __syncthreads();
  return xs;
}

// one gathered factor row x = X[oi, 0:R]: from the SMEM stage when present,
// else from global memory — L1-cached (l1: the grid barrier's fences order it
// after the producing phase) in 16-byte pieces for even R, or L2-only scalars
template <int R>
__device__ __forceinline__ void gather_row(const double* X, const double* Xs, int32_t oi, bool l1,
                                           double (&x)[R]) {
  if (Xs) {
#pragma unroll
    for (int l = 0; l < R; ++l) x[l] = Xs[(int64_t)oi * R + l];
  } else if (l1) {
    if constexpr ((R & 1) == 0) {
      const double2* s2 = reinterpret_cast<const double2*>(X + (int64_t)oi * R);
#pragma unroll
      for (int l = 0; l < R / 2; ++l) {
        const double2 v = s2[l];
        x[2 * l] = v.x;
        x[2 * l + 1] = v.y;
      }
    } else {
#pragma unroll
      for (int l = 0; l < R; ++l) x[l] = X[(int64_t)oi * R + l];
    }
  } else {
#pragma unroll
    for (int l = 0; l < R; ++l) x[l] = __ldcg(X + (int64_t)oi * R + l);
  }
}

// lane-strided partial sum over the samples [q0, q1): acc += Σ coef X[other]
template <int R>
__device__ __forceinline__ void spmm_accum(int64_t q0, int64_t q1, const int32_t* __restrict__ other,
                                           const double* __restrict__ coef, const double* X,
                                           const double* Xs, bool l1, double (&acc)[R]) {
  constexpr int U = WMUnroll<R>::U;
  const int lane = threadIdx.x & 31;
  // software-pipelined: the next group's (coef, index) loads are issued before
  // this group's factor-row gathers, so a group costs one L2 round trip, not two
  double cn[U];
  int32_t on[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t q = q0 + lane + 32 * u;
    const bool ok = q < q1;
    cn[u] = ok ? coef[q] : 0.0;
    on[u] = ok ? other[q] : 0;
  }
  for (int64_t base = q0 + lane; base < q1; base += 32 * U) {
    double c[U];
    int32_t oi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      c[u] = cn[u];
      oi[u] = on[u];
      const int64_t q = base + 32 * (U + u);
      const bool ok = q < q1;
      cn[u] = ok ? coef[q] : 0.0;
      on[u] = ok ? other[q] : 0;
    }
    double x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) gather_row<R>(X, Xs, oi[u], l1, x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int l = 0; l < R; ++l) acc[l] = fma(c[u], x[u][l], acc[l]);
  }
#pragma unroll
  for (int l = 0; l < R; ++l)
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) acc[l] += __shfl_xor_sync(0xffffffffu, acc[l], sh);
}

// out[o] = (Σ_{p in [ptr[o], ptr[o+1])} coef[p] X[other[p]]) · T (samples of
// row o stored contiguously: CSR order, or the pre-permuted CSC copy).
// Rows with more than WM_HEAVY samples (listed in heavy[0 .. *n_heavy)) are
// split over the 8 warps of one CTA and combined in SMEM in warp order; the
// others take one warp each.  Deterministic either way.
template <int R>
__device__ void spmm_phase(WMShared<R>& sm, const int64_t* __restrict__ ptr,
                           const int32_t* __restrict__ other, const double* __restrict__ coef,
                           const double* X, int64_t nout, double* out, double* gpart_buf,
                           const double* Xs, const int32_t* heavy, int n_heavy,
                           const uint8_t* hflag, bool l1, const WMCache& cc, bool chol_pending = false) {
  constexpr int NG = WMShared<R>::NG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * WM_WARPS;
  double gl[(NG + 31) / 32];
#pragma unroll
  for (int q = 0; q < (NG + 31) / 32; ++q) gl[q] = 0.0;
  const int nh = heavy ? n_heavy : 0;
  // chol_pending: sm.T (= R^{-1} of the reduced Gram in sm.G) is not computed
  // yet.  Thread 0 computes it while the other warps accumulate their first
  // row (the sums do not need T); every warp meets once at named barrier 1
  // before its first emit.  With heavy rows (CTA-wide, need T at once) it is
  // computed up front.
  bool wait_t = chol_pending;
  if (chol_pending && nh > 0) {
    if (threadIdx.x == 0) chol_rinv<R>(sm, sm.T);
    __syncthreads();
    wait_t = false;
  } else if (chol_pending && warp == 0) {
    if (lane == 0) chol_rinv<R>(sm, sm.T);
    __syncwarp();
  }
  for (int hi = blockIdx.x; hi < nh; hi += gridDim.x) {
    const int64_t o = heavy[hi];
    const int64_t p0 = ptr[o], p1 = ptr[o + 1];
    const int64_t len = p1 - p0;
    double acc[R];
#pragma unroll
    for (int l = 0; l < R; ++l) acc[l] = 0.0;
    spmm_accum<R>(p0 + (len * warp) / WM_WARPS, p0 + (len * (warp + 1)) / WM_WARPS, other, coef, X, Xs, l1, acc);
    if (lane == 0)
#pragma unroll
      for (int l = 0; l < R; ++l) sm.hred[warp][l] = acc[l];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int l = 0; l < R; ++l) {
        double t = sm.hred[0][l];
        for (int w2 = 1; w2 < WM_WARPS; ++w2) t += sm.hred[w2][l];
        acc[l] = t;
      }
      emit_row<R>(sm, o, acc, sm.T, out, -1.0, gl);
    }
    __syncthreads();
  }
  const bool cached = cc.on != 0;
  int64_t cq = cached ? cc.soff[warp] : 0;
  const int32_t* clen = cached ? cc.len + cc.roff[warp] : nullptr;
  const int32_t* src_o = cached ? cc.other : other;
  const double* src_c = cached ? cc.wv : coef;
  int k = 0;
  for (int64_t o = (int64_t)blockIdx.x * WM_WARPS + warp; o < nout; o += W, ++k) {
    int64_t q0, q1;
    if (cached) {
      const int len = clen[k];
      if (len < 0) continue;
      q0 = cq; q1 = cq + len; cq = q1;
    } else {
      if (hflag && hflag[o]) continue;
      q0 = ptr[o]; q1 = ptr[o + 1];
    }
    double acc[R];
#pragma unroll
    for (int l = 0; l < R; ++l) acc[l] = 0.0;
    spmm_accum<R>(q0, q1, src_o, src_c, X, Xs, l1, acc);
    if (wait_t) {
      asm volatile("bar.sync 1, %0;" ::"r"(WM_THREADS) : "memory");
      wait_t = false;
    }
    emit_row<R>(sm, o, acc, sm.T, out, -1.0, gl);
  }
  if (wait_t) asm volatile("bar.sync 1, %0;" ::"r"(WM_THREADS) : "memory");
  flush_gram<R>(sm, gl, gpart_buf);
}

// rows owned by this warp: out[o] <- X[o] · Tm, optionally trimmed (line 6,
// R13: zero rows with ||U0_i|| > c sqrt(r) ||A_i|| / ||A||_F); Gram partial
template <int R>
__device__ void transform_phase(WMShared<R>& sm, const double* X, int64_t n, const double* Tm,
                                double* out, double* gpart_buf, bool trim, const WMParams& p) {
  constexpr int NG = WMShared<R>::NG;
  const int64_t W = (int64_t)gridDim.x * WM_WARPS;
  double gl[(NG + 31) / 32];
#pragma unroll
  for (int q = 0; q < (NG + 31) / 32; ++q) gl[q] = 0.0;
  const double frob = trim ? sqrt(*p.FA) : 0.0;
  for (int64_t o = (int64_t)blockIdx.x * WM_WARPS + (threadIdx.x >> 5); o < n; o += W) {
    double acc[R];
#pragma unroll
    for (int l = 0; l < R; ++l) acc[l] = __ldcg(X + o * R + l);
    const double thr = (trim && frob > 0.0) ? p.trim_c * sqrt((double)R) * sqrt(p.a2[o]) / frob : -1.0;
    emit_row<R>(sm, o, acc, Tm, out, thr, gl);
  }
  if (gpart_buf) flush_gram<R>(sm, gl, gpart_buf);
}

// lane-strided partial normal equations over the samples [q0, q1):
// g += Σ w x xᵀ (upper triangle), h += Σ w M̃ x, then a fixed xor-butterfly
template <int R>
__device__ __forceinline__ void als_accum(int64_t q0, int64_t q1, const int32_t* __restrict__ other,
                                          const double* __restrict__ w, const double* __restrict__ wv,
                                          const double* X, const double* Xs, bool l1,
                                          double (&g)[R * (R + 1) / 2],
                                          double (&h)[R]) {
  constexpr int NG = R * (R + 1) / 2;
  constexpr int U = WMUnroll<R>::U;
  const int lane = threadIdx.x & 31;
  // software-pipelined as spmm_accum: next group's (w, w·M̃, index) loads first
  double wn[U], vn[U];
  int32_t on[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int64_t q = q0 + lane + 32 * u;
    const bool ok = q < q1;
    wn[u] = ok ? w[q] : 0.0;
    vn[u] = ok ? wv[q] : 0.0;
    on[u] = ok ? other[q] : 0;
  }
  for (int64_t base = q0 + lane; base < q1; base += 32 * U) {
    double ws[U], vs[U];
    int32_t oi[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ws[u] = wn[u];
      vs[u] = vn[u];
      oi[u] = on[u];
      const int64_t q = base + 32 * (U + u);
      const bool ok = q < q1;
      wn[u] = ok ? w[q] : 0.0;
      vn[u] = ok ? wv[q] : 0.0;
      on[u] = ok ? other[q] : 0;
    }
    double x[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u) gather_row<R>(X, Xs, oi[u], l1, x[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int e = 0;
#pragma unroll
      for (int a = 0; a < R; ++a) {
        const double wa = ws[u] * x[u][a];
        h[a] = fma(vs[u], x[u][a], h[a]);
#pragma unroll
        for (int b = a; b < R; ++b) { g[e] = fma(wa, x[u][b], g[e]); ++e; }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < NG; ++e)
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) g[e] += __shfl_xor_sync(0xffffffffu, g[e], sh);
#pragma unroll
  for (int a = 0; a < R; ++a)
#pragma unroll
    for (int sh = 16; sh > 0; sh >>= 1) h[a] += __shfl_xor_sync(0xffffffffu, h[a], sh);
}

// ridge Cholesky solve of one output row from its normal equations gh =
// [G upper triangle | h] in SMEM (called by one lane).  Not inlined: one copy
// serves the light- and heavy-row paths (two inlined copies spill at R >= 4).
template <int R>
__device__ __noinline__ void als_solve(const double* gh, double lam, double* out, int64_t o) {
  constexpr int NG = R * (R + 1) / 2;
  const double* g = gh;
  const double* h = gh + NG;
  // ridge Cholesky solve (G + lam tr(G)/r I) x = h; empty/singular -> 0
  // (R14).  Fully unrolled: registers only.
  double L[R][R], xs[R], y[R], inv[R];
  double tr = 0.0;
  {
    int e = 0;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = a; b < R; ++b) {
        L[b][a] = g[e];
        if (a == b) tr += g[e];
        ++e;
      }
  }
  bool ok = tr > 0.0;
  const double shift = lam * tr / (double)R;
#pragma unroll
  for (int a = 0; a < R; ++a) L[a][a] += shift;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    double s = L[j][j];
#pragma unroll
    for (int q = 0; q < j; ++q) s -= L[j][q] * L[j][q];
    ok = ok && (s > 0.0);
    const double d = sqrt(s > 0.0 ? s : 1.0);
    inv[j] = 1.0 / d;
    L[j][j] = d;
#pragma unroll
    for (int i = j + 1; i < R; ++i) {
      double t = L[i][j];
#pragma unroll
      for (int q = 0; q < j; ++q) t -= L[i][q] * L[j][q];
      L[i][j] = t * inv[j];
    }
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    double t = h[i];
#pragma unroll
    for (int q = 0; q < i; ++q) t -= L[i][q] * y[q];
    y[i] = t * inv[i];
  }
#pragma unroll
  for (int i = R - 1; i >= 0; --i) {
    double t = y[i];
#pragma unroll
    for (int q = i + 1; q < R; ++q) t -= L[q][i] * xs[q];
    xs[i] = t * inv[i];
  }
#pragma unroll
  for (int a = 0; a < R; ++a) out[o * R + a] = ok ? xs[a] : 0.0;
}

// one weighted least-squares half step (lines 8/9; R14):
// out[o] = (G_o + lam tr(G_o)/r I)^{-1} h_o over the samples of output row o,
// G_o = Σ w x xᵀ, h_o = Σ w M̃ x.  Heavy rows (> WM_HEAVY samples) are split
// over a CTA's 8 warps and combined in SMEM in warp order.
template <int R>
__device__ void als_phase(WMShared<R>& sm, const int64_t* __restrict__ ptr,
                          const int32_t* __restrict__ other, const double* __restrict__ w,
                          const double* __restrict__ wv, const double* X, int64_t nout, double lam,
                          double* out, const double* Xs, const int32_t* heavy, int n_heavy,
                          const uint8_t* hflag, bool l1, const WMCache& cc) {
  constexpr int NG = WMShared<R>::NG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t W = (int64_t)gridDim.x * WM_WARPS;
  const int nh = heavy ? n_heavy : 0;
  for (int hi = blockIdx.x; hi < nh; hi += gridDim.x) {
    const int64_t o = heavy[hi];
    const int64_t p0 = ptr[o], p1 = ptr[o + 1];
    const int64_t len = p1 - p0;
    double g[NG], h[R];
#pragma unroll
    for (int e = 0; e < NG; ++e) g[e] = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) h[a] = 0.0;
    als_accum<R>(p0 + (len * warp) / WM_WARPS, p0 + (len * (warp + 1)) / WM_WARPS, other, w, wv, X, Xs, l1, g, h);
    if (lane == 0) {
#pragma unroll
      for (int e = 0; e < NG; ++e) sm.hred[warp][e] = g[e];
#pragma unroll
      for (int a = 0; a < R; ++a) sm.hred[warp][NG + a] = h[a];
    }
    __syncthreads();
    // entry e summed over the warps in warp order by thread e (fixed order)
    double t = 0.0;
    if (threadIdx.x < NG + R) {
      t = sm.hred[0][threadIdx.x];
#pragma unroll
      for (int w2 = 1; w2 < WM_WARPS; ++w2) t += sm.hred[w2][threadIdx.x];
    }
    __syncthreads();
    if (threadIdx.x < NG + R) sm.hred[0][threadIdx.x] = t;
    __syncthreads();
    if (threadIdx.x == 0) als_solve<R>(sm.hred[0], lam, out, o);
    __syncthreads();
  }
  const bool cached = cc.on != 0;
  int64_t cq = cached ? cc.soff[warp] : 0;
  const int32_t* clen = cached ? cc.len + cc.roff[warp] : nullptr;
  const int32_t* src_o = cached ? cc.other : other;
  const double* src_w = cached ? cc.w : w;
  const double* src_v = cached ? cc.wv : wv;
  int k = 0;
  for (int64_t o = (int64_t)blockIdx.x * WM_WARPS + warp; o < nout; o += W, ++k) {
    int64_t q0, q1;
    if (cached) {
      const int len = clen[k];
      if (len < 0) continue;
      q0 = cq; q1 = cq + len; cq = q1;
    } else {
      if (hflag && hflag[o]) continue;
      q0 = ptr[o]; q1 = ptr[o + 1];
    }
    double g[NG], h[R];
#pragma unroll
    for (int e = 0; e < NG; ++e) g[e] = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) h[a] = 0.0;
    als_accum<R>(q0, q1, src_o, src_w, src_v, X, Xs, l1, g, h);
    if (lane == 0) {
#pragma unroll
      for (int e = 0; e < NG; ++e) sm.hred[warp][e] = g[e];
#pragma unroll
      for (int a = 0; a < R; ++a) sm.hred[warp][NG + a] = h[a];
      als_solve<R>(sm.hred[warp], lam, out, o);
    }
    __syncwarp();
  }
}

template <int R>
__global__ void __launch_bounds__(WM_THREADS, 1) wm_persistent_kernel(WMParams p) {
  constexpr int NG = WMShared<R>::NG;
  extern __shared__ __align__(16) uint8_t wm_smem[];
  WMShared<R>& sm = *reinterpret_cast<WMShared<R>*>(wm_smem);
  double* xs = reinterpret_cast<double*>(wm_smem + ((sizeof(WMShared<R>) + 15) & ~(size_t)15));
  const bool stg = p.stage_x != 0;
  __shared__ double TZ[R * R];
  const int tid = threadIdx.x;
  if (tid == 0) {
    int e = 0;
    for (int a = 0; a < R; ++a)
      for (int b = a; b < R; ++b) { sm.ea[e] = a; sm.eb[e] = b; ++e; }
  }
  set_identity<R>(sm.T);
  sm.cache[0].on = 0;
  sm.cache[1].on = 0;
  if (tid == 0) {
    sm.nh[0] = p.heavy_r ? *p.nheavy_r : 0;
    sm.nh[1] = p.heavy_c ? *p.nheavy_c : 0;
  }
  __syncthreads();
  if (p.cache_bytes > 0) {
    uint8_t* region = reinterpret_cast<uint8_t*>(xs) + (stg ? ((size_t)(p.n1 > p.n2 ? p.n1 : p.n2) * R * 8) : 0);
    const uint8_t* end = region + p.cache_bytes;
    build_cache(sm.cache[0], sm.scan, p.rptr, p.J, p.w, p.wv, p.n1, p.hflag_r, region, end);
    build_cache(sm.cache[1], sm.scan, p.cptr, p.cI, p.cw, p.cwv, p.n2, p.hflag_c, region, end);
  }
  const int64_t G = gridDim.x;
  int buf = 0;
  int nbar = 0;
  auto gp = [&](int b) { return p.gpart + (int64_t)b * G * NG; };
  // CholeskyQR2 of the rows just written to X (Gram already in gp(buf)):
  // leaves X · T orthonormal with T = R2^{-1} in sm.T
  auto cqr2 = [&](double* X, int64_t n) {
    grid_sync(p.bar, p.trace, nbar);
    reduce_chol<R>(sm, gp(buf));
    buf ^= 1;
    transform_phase<R>(sm, X, n, sm.Rinv, X, gp(buf), false, p);
    grid_sync(p.bar, p.trace, nbar);
    reduce_chol<R>(sm, gp(buf));
    buf ^= 1;
    for (int e = tid; e < R * R; e += blockDim.x) sm.T[e] = sm.Rinv[e];
    __syncthreads();
  };

  // line 5: Y0 Rademacher
  for (int64_t e = (int64_t)blockIdx.x * WM_THREADS + tid; e < p.n2 * R; e += G * WM_THREADS) {
    const int64_t j = e / R;
    const int l = (int)(e - j * R);
    const u32x4 wd = philox4x32_10((uint32_t)j, (uint32_t)l, 0u, TAG_INIT, (uint32_t)p.seed,
                                   (uint32_t)(p.seed >> 32));
    p.Y[e] = (wd.x & 1u) ? -1.0 : 1.0;
  }
  grid_sync(p.bar, p.trace, nbar);
  // subspace iteration (R12): Z = R Y, Y = Rᵀ Z, each orthonormalised by
  // one CholeskyQR whose triangular factor is folded into the next SpMM
  // (stored rows · T is the orthonormal basis); the final Z gets CholeskyQR2
  // defer: leave the Cholesky to the next spmm_phase (chol_pending), which
  // overlaps it with the first row's accumulation
  auto cqr1_defer = [&](const double* SX, int64_t sn) {
    grid_sync(p.bar, p.trace, nbar);
    reduce_chol<R>(sm, gp(buf), stg ? SX : nullptr, sn, xs, false);
    buf ^= 1;
  };
  const int iters = p.init_iters > 0 ? p.init_iters : 1;
  // diagnostics (SMP_WM_TRACE): CTA 0's time in the first Z-side SpMM phases
  auto stamp = [&](int slot) {
    if (p.trace2 && blockIdx.x == 0 && tid == 0 && slot < 64) p.trace2[slot] = wm_globaltimer();
  };
  for (int it = 0; it < iters; ++it) {
    stamp(4 * it);
    // Y rows: staged with the previous reduction, except before the first half
    const double* xsY = it == 0 ? stage_rows<R>(p.Y, p.n2, xs, stg) : (stg ? xs : nullptr);
    stamp(4 * it + 1);
    spmm_phase<R>(sm, p.rptr, p.J, p.wv, p.Y, p.n1, p.Z, gp(buf), xsY, p.heavy_r, sm.nh[0], p.hflag_r, p.x_l1,
                  sm.cache[0], it > 0);
    stamp(4 * it + 2);
    if (it == iters - 1) {  // the last Y half does not reach U0
      cqr2(p.Z, p.n1);
      break;
    }
    cqr1_defer(p.Z, p.n1);
    stamp(4 * it + 3);
    spmm_phase<R>(sm, p.cptr, p.cI, p.cwv, p.Z, p.n2, p.Y, gp(buf), stg ? xs : nullptr,
                  p.heavy_c, sm.nh[1], p.hflag_c, p.x_l1, sm.cache[1], true);
    cqr1_defer(p.Y, p.n2);  // it + 1 < iters here; its Cholesky runs in the next row SpMM
  }
  for (int e = tid; e < R * R; e += blockDim.x) TZ[e] = sm.T[e];
  __syncthreads();
  if (p.trim_c > 0.0) {
    // line 6: U0 = Z T, trim, re-orthonormalise (CholeskyQR2), U = U0 T'
    transform_phase<R>(sm, p.Z, p.n1, TZ, p.Z, gp(buf), true, p);
    cqr2(p.Z, p.n1);
    transform_phase<R>(sm, p.Z, p.n1, sm.T, p.U, nullptr, false, p);
  } else {
    transform_phase<R>(sm, p.Z, p.n1, TZ, p.U, nullptr, false, p);
  }
  grid_sync(p.bar, p.trace, nbar);
  // lines 7-10: T alternating weighted least-squares half steps
  if (p.T == 0)
    for (int64_t e = (int64_t)blockIdx.x * WM_THREADS + tid; e < p.n2 * R; e += G * WM_THREADS) p.V[e] = 0.0;
  for (int t = 0; t < p.T; ++t) {
    als_phase<R>(sm, p.cptr + (2 * t + 1) * p.cstride, p.cI, p.cw, p.cwv, p.U, p.n2, p.lam, p.V,
                 stage_rows<R>(p.U, p.n1, xs, stg), p.heavy_c, sm.nh[1], p.hflag_c, p.x_l1, sm.cache[1]);
    grid_sync(p.bar, p.trace, nbar);
    als_phase<R>(sm, p.rptr + (2 * t + 2) * p.rstride, p.J, p.w, p.wv, p.V, p.n1, p.lam, p.U,
                 stage_rows<R>(p.V, p.n2, xs, stg), p.heavy_r, sm.nh[0], p.hflag_r, p.x_l1, sm.cache[0]);
    grid_sync(p.bar, p.trace, nbar);
  }
  // output (Û(T), V̂(T)) in fp32
  for (int64_t e = (int64_t)blockIdx.x * WM_THREADS + tid; e < p.n1 * R; e += G * WM_THREADS)
    p.Uout[e] = (float)__ldcg(p.U + e);
  for (int64_t e = (int64_t)blockIdx.x * WM_THREADS + tid; e < p.n2 * R; e += G * WM_THREADS)
    p.Vout[e] = (float)__ldcg(p.V + e);
}

template <int R>
cudaError_t launch_wm(WMParams& p, cudaStream_t st) {
  constexpr size_t XS_MAX = 160 * 1024;  // staged factor rows (n_max · r doubles)
  const size_t base = (sizeof(WMShared<R>) + 15) & ~(size_t)15;
  const size_t xs_bytes = (size_t)(p.n1 > p.n2 ? p.n1 : p.n2) * R * 8;
  p.stage_x = (p.env_stage && xs_bytes <= XS_MAX) ? 1 : 0;  // SMP_WM_STAGE=0: never stage
  int dev = 0, sms = 0, per_sm = 0, optin = 0;
  SMP_TRY(cudaGetDevice(&dev));
  SMP_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  SMP_TRY(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  SMP_TRY(cudaFuncGetAttributes(&fa, wm_persistent_kernel<R>));
  optin -= (int)fa.sharedSizeBytes;  // dynamic limit = opt-in total - static
  size_t smem = base + (p.stage_x ? xs_bytes : 0);
  // sample cache (WMCache): reserve twice the average per-CTA need of both
  // sides (20 B per sample and side + row lengths) when that fits beside the
  // stage — otherwise leave the SMEM to L1, which the unstaged gathers use.
  // SMP_WM_CACHE=0 disables it (tuning); FRESH_2T1 phases read different
  // subsets, so the (whole-Ω) cache is off there.
  const int env_cache = p.env_cache && p.rstride == 0;
  // one CTA per SM at most (co-resident: cooperative launch), and no more CTAs
  // than needed for the per-warp row count a full grid would give: the same
  // critical path with fewer barrier participants and Gram partials (cfg1:
  // 1024 rows -> 128 CTAs of one row per warp; cfg4 2.85 -> 2.60 ms).
  // SMP_WM_CTAS overrides (tuning).
  const int env_ctas = p.env_ctas;
  int grid = sms;
  {
    const int64_t nmax = p.n1 > p.n2 ? p.n1 : p.n2;
    const int64_t per_warp = (nmax + (int64_t)sms * WM_WARPS - 1) / ((int64_t)sms * WM_WARPS);
    if (per_warp > 0) {
      const int64_t need = (nmax + per_warp * WM_WARPS - 1) / (per_warp * WM_WARPS);
      grid = (int)(need < 1 ? 1 : (need < sms ? need : sms));
    }
  }
  if (env_ctas > 0 && env_ctas <= sms) grid = env_ctas;
  p.cache_bytes = 0;
  if (env_cache && grid > 0) {
    const int64_t avg = (2 * 20 * p.count + 4 * (p.n1 + p.n2)) / grid;
    const int64_t want = 2 * avg + 4096;
    if ((int64_t)smem + want <= (int64_t)optin) {
      p.cache_bytes = want;
      smem += (size_t)want;
    }
  }
  // per device (cheap; a process may drive several GPUs)
  SMP_TRY(cudaFuncSetAttribute(wm_persistent_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, optin));
  SMP_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wm_persistent_kernel<R>, WM_THREADS, smem));
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel((const void*)wm_persistent_kernel<R>, dim3(grid), dim3(WM_THREADS),
                                     args, smem, st);
}

}  // namespace smp
