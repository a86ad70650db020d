// K7-K9: WAltMin (Alg. 2; Step 3, Eq. 3) with
// the REUSE_ALL or FRESH_2T1 partition of line 3 (R11):
//   w = 1/q̂ (line 2); R = w .* P_Ω(M̃) (line 4);
//   U0 = top-r left subspace of R by subspace iteration from a Rademacher
//        start (line 5; R12), CholeskyQR2 orthonormalisation;
//   trim rows with ||U0_i|| > c sqrt(r) ||A_i||/||A||_F (line 6; R13), re-QR;
//   T x { V = argmin_V ||R^½(M̃ - U Vᵀ)|| (line 8); U = argmin_U (line 9) }
//   via per-row r×r weighted normal equations + ridge Cholesky (R14).
// Ω arrives sorted by (i,j) → CSR by slicing; CSC by a stable radix sort on j.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include "waltmin_impl.cuh"

namespace smp {



__global__ void wm_weights_kernel(const double* __restrict__ qhat, const float* __restrict__ val,
                                  int64_t cnt, double* __restrict__ w, double* __restrict__ wv) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cnt;
       s += (int64_t)gridDim.x * blockDim.x) {
    const double q = qhat[s];
    const double ww = q > 0.0 ? __ddiv_rn(1.0, q) : 0.0;
    w[s] = ww;
    wv[s] = __dmul_rn(ww, (double)val[s]);
  }
}

// ptr[g·(nout+1) + o] = lower_bound(keys, g·nout + o) for o in [0, nout],
// g in [0, groups): row pointers of every subset of a (subset, row)-sorted key
// sequence (groups = 1: plain CSR pointers)
template <class K>
__global__ void wm_ptr_kernel(const K* __restrict__ keys, int64_t cnt, int64_t nout, int groups,
                              int64_t* __restrict__ ptr) {
  const int64_t tot = (int64_t)groups * (nout + 1);
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = e / (nout + 1), o = e - g * (nout + 1);
    const int64_t target = g * nout + o;
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    ptr[e] = lo;
  }
}

// CSC copy of the per-sample arrays in column order (perm from the stable sort)
__global__ void wm_gather_csc_kernel(const int32_t* __restrict__ perm, const int32_t* __restrict__ I,
                                     const double* __restrict__ w, const double* __restrict__ wv,
                                     int64_t cnt, int32_t* __restrict__ cI, double* __restrict__ cw,
                                     double* __restrict__ cwv) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cnt;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = perm[q];
    cI[q] = I[s];
    cw[q] = w[s];
    cwv[q] = wv[s];
  }
}

__global__ void wm_iota_kernel(int32_t* __restrict__ p, int64_t cnt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cnt;
       s += (int64_t)gridDim.x * blockDim.x)
    p[s] = (int32_t)s;
}

// heavy[o] = 1 iff output row o has more than thr samples; idx[o] = o
__global__ void wm_heavy_flags_kernel(const int64_t* __restrict__ ptr, int64_t nout, int64_t thr,
                                      uint8_t* __restrict__ flag, int32_t* __restrict__ idx) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < nout;
       o += (int64_t)gridDim.x * blockDim.x) {
    flag[o] = (ptr[o + 1] - ptr[o]) > thr ? 1 : 0;
    idx[o] = (int32_t)o;
  }
}

// ---- FRESH_2T1 partition (Alg. 2 line 3; R11):
// key_s = (w1 << 32) | w0 of Philox(ctr = (i, j, 0, 4), key = seed); the
// sample of rank p in (key, s) order goes to subset p mod nsub.
__global__ void wm_part_key_kernel(const int32_t* __restrict__ I, const int32_t* __restrict__ J, int64_t cnt,
                                   uint64_t seed, uint64_t* __restrict__ key) {
  const uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cnt;
       s += (int64_t)gridDim.x * blockDim.x) {
    const u32x4 w = philox4x32_10((uint32_t)I[s], (uint32_t)J[s], 0u, TAG_PART, k0, k1);
    key[s] = ((uint64_t)w.y << 32) | (uint64_t)w.x;
  }
}

__global__ void wm_sub_kernel(const int32_t* __restrict__ rank_to_s, int64_t cnt, int nsub,
                              int32_t* __restrict__ sub) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < cnt;
       p += (int64_t)gridDim.x * blockDim.x)
    sub[rank_to_s[p]] = (int32_t)(p % nsub);
}

// subset-major copy: sample q of the new order is original sample ord[q];
// rk = sub·n1 + i (CSR key), ck = sub·n2 + j (CSC key)
__global__ void wm_fresh_gather_kernel(const int32_t* __restrict__ ord, const int32_t* __restrict__ sub,
                                       const int32_t* __restrict__ I, const int32_t* __restrict__ J,
                                       const float* __restrict__ val, const double* __restrict__ qhat,
                                       int64_t cnt, int64_t n1, int64_t n2, int32_t* __restrict__ I2,
                                       int32_t* __restrict__ J2, float* __restrict__ val2,
                                       double* __restrict__ q2, int64_t* __restrict__ rk,
                                       int64_t* __restrict__ ck) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < cnt;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = ord[q];
    const int64_t g = sub[s];
    I2[q] = I[s];
    J2[q] = J[s];
    val2[q] = val[s];
    q2[q] = qhat[s];
    rk[q] = g * n1 + I[s];
    ck[q] = g * n2 + J[s];
  }
}

// stream-ordered workspace, released on every return path
struct WmScratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit WmScratch(cudaStream_t s) : st(s) {}
  template <class T>
  cudaError_t alloc(T*& p, int64_t bytes) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, (size_t)(bytes > 0 ? bytes : 1), st);
    if (e == cudaSuccess) { ptrs.push_back(q); p = static_cast<T*>(q); }
    return e;
  }
  ~WmScratch() { for (void* q : ptrs) cudaFreeAsync(q, st); }
};

static int bits_for(int64_t v) {  // bits needed to represent values < v (at least 1)
  int b = 1;
  while (b < 63 && ((int64_t)1 << b) < v) ++b;
  return b;
}

template <int R>
cudaError_t launch_wm(WMParams& p, cudaStream_t st);  // waltmin_r*.cu

static cudaError_t launch_wm_r(int r, WMParams& p, cudaStream_t st) {
  switch (r) {
#define SMP_WM_CASE(RR) case RR: return launch_wm<RR>(p, st);
    SMP_WM_CASE(1) SMP_WM_CASE(2) SMP_WM_CASE(3) SMP_WM_CASE(4) SMP_WM_CASE(5) SMP_WM_CASE(6)
    SMP_WM_CASE(7) SMP_WM_CASE(8) SMP_WM_CASE(9) SMP_WM_CASE(10) SMP_WM_CASE(11) SMP_WM_CASE(12)
    SMP_WM_CASE(13) SMP_WM_CASE(14) SMP_WM_CASE(15) SMP_WM_CASE(16)
#undef SMP_WM_CASE
    default: return cudaErrorInvalidValue;
  }
}

int waltmin_grid_ctas() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return sms;
}

static int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)std::min<int64_t>(b, 148 * 16);
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

cudaError_t run_waltmin(const WaltminArgs& a, cudaStream_t st) {
  const int64_t cnt = a.count, n1 = a.n1, n2 = a.n2;
  const int r = a.r;
  if (r < 1 || r > 16) return cudaErrorInvalidValue;
  const bool fresh = a.partition == 1;
  const int nsub = fresh ? 2 * a.T + 1 : 1;
  WmScratch ws(st);
  double *w, *wv, *cw, *cwv, *Y, *Z, *U, *V, *gpart;
  unsigned* bar;
  int64_t *rptr, *cptr;
  int32_t *iota, *perm, *cI;
  const int64_t c1 = cnt > 0 ? cnt : 1;
  const int gctas = waltmin_grid_ctas();
  if (gctas < 1) return cudaErrorNoDevice;
  SMP_TRY(ws.alloc(w, c1 * 8));
  SMP_TRY(ws.alloc(wv, c1 * 8));
  SMP_TRY(ws.alloc(cw, c1 * 8));
  SMP_TRY(ws.alloc(cwv, c1 * 8));
  SMP_TRY(ws.alloc(cI, c1 * 4));
  SMP_TRY(ws.alloc(Y, n2 * r * 8));
  SMP_TRY(ws.alloc(Z, n1 * r * 8));
  SMP_TRY(ws.alloc(U, n1 * r * 8));
  SMP_TRY(ws.alloc(V, n2 * r * 8));
  SMP_TRY(ws.alloc(gpart, (int64_t)2 * gctas * r * (r + 1) / 2 * 8));
  SMP_TRY(ws.alloc(bar, 64));
  SMP_TRY(ws.alloc(rptr, (int64_t)nsub * (n1 + 1) * 8));
  SMP_TRY(ws.alloc(cptr, (int64_t)nsub * (n2 + 1) * 8));
  SMP_TRY(ws.alloc(iota, c1 * 4));
  SMP_TRY(ws.alloc(perm, c1 * 4));
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  auto cub_scratch = [&](size_t need) -> cudaError_t {
    if (need <= cub_bytes && cub_tmp) return cudaSuccess;
    void* q = nullptr;
    SMP_TRY(ws.alloc(q, (int64_t)need));
    cub_tmp = q;
    cub_bytes = need;
    return cudaSuccess;
  };
  const int gc = grid_for(cnt, 256);

  // the sample arrays the phases read: Ω as given (REUSE_ALL) or its
  // subset-major copy (FRESH_2T1)
  const int32_t* sI = a.I;
  const int32_t* sJ = a.J;
  const float* sval = a.val;
  const double* sq = a.qhat;
  int64_t *rk = nullptr, *ck = nullptr;
  wm_iota_kernel<<<gc, 256, 0, st>>>(iota, cnt);
  if (fresh && cnt > 0) {
    uint64_t *key, *key_s;
    int32_t *sub, *sub_s, *ord, *I2, *J2;
    float* val2;
    double* q2;
    SMP_TRY(ws.alloc(key, c1 * 8));
    SMP_TRY(ws.alloc(key_s, c1 * 8));
    SMP_TRY(ws.alloc(sub, c1 * 4));
    SMP_TRY(ws.alloc(sub_s, c1 * 4));
    SMP_TRY(ws.alloc(ord, c1 * 4));
    SMP_TRY(ws.alloc(I2, c1 * 4));
    SMP_TRY(ws.alloc(J2, c1 * 4));
    SMP_TRY(ws.alloc(val2, c1 * 4));
    SMP_TRY(ws.alloc(q2, c1 * 8));
    SMP_TRY(ws.alloc(rk, c1 * 8));
    SMP_TRY(ws.alloc(ck, c1 * 8));
    wm_part_key_kernel<<<gc, 256, 0, st>>>(a.I, a.J, cnt, a.seed, key);
    size_t need = 0;
    SMP_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, key, key_s, iota, perm, (int)cnt, 0, 64, st));
    SMP_TRY(cub_scratch(need));
    SMP_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, need, key, key_s, iota, perm, (int)cnt, 0, 64, st));
    wm_sub_kernel<<<gc, 256, 0, st>>>(perm, cnt, nsub, sub);
    // stable by subset: within a subset the (i, j) order of Ω is kept
    SMP_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, sub, sub_s, iota, ord, (int)cnt, 0, bits_for(nsub), st));
    SMP_TRY(cub_scratch(need));
    SMP_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, need, sub, sub_s, iota, ord, (int)cnt, 0, bits_for(nsub), st));
    wm_fresh_gather_kernel<<<gc, 256, 0, st>>>(ord, sub, a.I, a.J, a.val, a.qhat, cnt, n1, n2, I2, J2, val2, q2,
                                                rk, ck);
    sI = I2; sJ = J2; sval = val2; sq = q2;
  }
  wm_weights_kernel<<<gc, 256, 0, st>>>(sq, sval, cnt, w, wv);
  // CSR pointers (per subset); CSC: stable radix sort of the column key
  if (fresh) {
    wm_ptr_kernel<int64_t><<<grid_for((int64_t)nsub * (n1 + 1), 256), 256, 0, st>>>(rk, cnt, n1, nsub, rptr);
    int64_t* ck_s;
    SMP_TRY(ws.alloc(ck_s, c1 * 8));
    const int eb = bits_for((int64_t)nsub * n2 + 1);
    size_t need = 0;
    SMP_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, ck, ck_s, iota, perm, (int)cnt, 0, eb, st));
    SMP_TRY(cub_scratch(need));
    SMP_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, need, ck, ck_s, iota, perm, (int)cnt, 0, eb, st));
    wm_ptr_kernel<int64_t><<<grid_for((int64_t)nsub * (n2 + 1), 256), 256, 0, st>>>(ck_s, cnt, n2, nsub, cptr);
  } else {
    wm_ptr_kernel<int32_t><<<grid_for(n1 + 1, 256), 256, 0, st>>>(sI, cnt, n1, 1, rptr);
    int32_t* jsorted;
    SMP_TRY(ws.alloc(jsorted, c1 * 4));
    const int end_bit = bits_for(n2 + 1);
    size_t need = 0;
    SMP_TRY(cub::DeviceRadixSort::SortPairs(nullptr, need, sJ, jsorted, iota, perm, (int)cnt, 0, end_bit, st));
    SMP_TRY(cub_scratch(need));
    SMP_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, need, sJ, jsorted, iota, perm, (int)cnt, 0, end_bit, st));
    wm_ptr_kernel<int32_t><<<grid_for(n2 + 1, 256), 256, 0, st>>>(jsorted, cnt, n2, 1, cptr);
  }
  wm_gather_csc_kernel<<<gc, 256, 0, st>>>(perm, sI, w, wv, cnt, cI, cw, cwv);

  // heavy rows / columns (REUSE_ALL only): stable compaction (fixed order ->
  // fixed CTA assignment -> deterministic Gram partials)
  const int64_t nmax = std::max<int64_t>(std::max<int64_t>(n1, n2), 1);
  // Split a row over a CTA when it has more than WM_HEAVY = 1024 samples: a
  // warp walks its rows one after another, latency-bound (~64 samples per
  // L2 round trip), so one long row sets the phase time however light the
  // warp's other rows are (cfg3: fully sampled rows of 8,000-10,000 samples
  // against 3,254 per warp on average; measured per WAltMin call: threshold
  // 1024 -> 8.2 ms, 2048 -> 9.3, 4096 -> 11.3, 4x the per-warp average
  // (13,018) -> 13.7; cfg1 (rows <= 564) splits none; cfg2 4.8 ms either way,
  // 512 no better).  SMP_WM_HEAVY overrides the threshold (0 = warp-per-row
  // only; tuning).
  const char* hv = getenv("SMP_WM_HEAVY");
  const int64_t heavy_thr = fresh ? 0 : (hv ? atoll(hv) : (int64_t)WM_HEAVY);
  uint8_t *hfr = nullptr, *hfc = nullptr;
  int32_t *hidx = nullptr, *hlr = nullptr, *hlc = nullptr, *nh = nullptr;
  if (heavy_thr > 0) {
    SMP_TRY(ws.alloc(hfr, n1 + 1));
    SMP_TRY(ws.alloc(hfc, n2 + 1));
    SMP_TRY(ws.alloc(hidx, nmax * 4));
    SMP_TRY(ws.alloc(hlr, (n1 + 1) * 4));
    SMP_TRY(ws.alloc(hlc, (n2 + 1) * 4));
    SMP_TRY(ws.alloc(nh, 2 * 4));
    size_t need = 0;
    SMP_TRY(cub::DeviceSelect::Flagged(nullptr, need, hidx, hfr, hlr, nh, (int)nmax, st));
    SMP_TRY(cub_scratch(need));
    SMP_TRY(cudaMemsetAsync(nh, 0, 2 * 4, st));
    if (n1 > 0) {
      wm_heavy_flags_kernel<<<grid_for(n1, 256), 256, 0, st>>>(rptr, n1, heavy_thr, hfr, hidx);
      size_t h1 = cub_bytes;
      SMP_TRY(cub::DeviceSelect::Flagged(cub_tmp, h1, hidx, hfr, hlr, nh, (int)n1, st));
    }
    if (n2 > 0) {
      wm_heavy_flags_kernel<<<grid_for(n2, 256), 256, 0, st>>>(cptr, n2, heavy_thr, hfc, hidx);
      size_t h2 = cub_bytes;
      SMP_TRY(cub::DeviceSelect::Flagged(cub_tmp, h2, hidx, hfc, hlc, nh + 1, (int)n2, st));
    }
  }

  // lines 5-10: one cooperative persistent kernel
  SMP_TRY(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st));
  WMParams p{};
  p.n1 = n1; p.n2 = n2; p.count = cnt; p.T = a.T; p.init_iters = a.init_iters;
  p.trim_c = a.trim_c; p.lam = a.lam; p.seed = a.seed;
  p.rptr = rptr; p.J = sJ; p.w = w; p.wv = wv;
  p.cptr = cptr; p.cI = cI; p.cw = cw; p.cwv = cwv;
  p.a2 = a.a_norm2; p.FA = a.FA;
  p.Y = Y; p.Z = Z; p.U = U; p.V = V; p.gpart = gpart; p.bar = bar;
  p.Uout = a.U; p.Vout = a.V;
  p.rstride = fresh ? n1 + 1 : 0;
  p.cstride = fresh ? n2 + 1 : 0;
  // tuning switches, read on every call
  p.x_l1 = env_int("SMP_WM_L1", 1) == 0 ? 0 : 1;  // 0: L2-only gathers (A/B switch)
  p.env_stage = env_int("SMP_WM_STAGE", 1);
  p.env_cache = env_int("SMP_WM_CACHE", 1);
  p.env_ctas = env_int("SMP_WM_CTAS", 0);
  if (heavy_thr > 0) {
    p.heavy_r = hlr; p.nheavy_r = nh; p.hflag_r = hfr;
    p.heavy_c = hlc; p.nheavy_c = nh + 1; p.hflag_c = hfc;
  }
  const char* tr = getenv("SMP_WM_TRACE");
  uint64_t* trace = nullptr;
  const int max_bar = 2 * (a.init_iters + 4) + 2 * a.T + 8;
  if (tr && atoi(tr)) {
    SMP_TRY(ws.alloc(trace, 4 * 8 * (int64_t)max_bar + 64 * 8));
    SMP_TRY(cudaMemsetAsync(trace, 0, 4 * 8 * (size_t)max_bar + 64 * 8, st));
  }
  p.trace = trace;
  p.trace2 = trace ? trace + 4 * max_bar : nullptr;
  SMP_TRY(launch_wm_r(r, p, st));
  if (trace) {
    std::vector<uint64_t> t(4 * (size_t)max_bar + 64);
    SMP_TRY(cudaMemcpyAsync(t.data(), trace, t.size() * 8, cudaMemcpyDeviceToHost, st));
    SMP_TRY(cudaStreamSynchronize(st));
    for (int b = 0; b < max_bar && t[4 * b]; ++b)
      fprintf(stderr, "wm barrier %3d: cta0 work %8.2f us, skew to last %8.2f us (cta %3d), release %6.2f us\n",
              b, b ? (t[4 * b] - t[4 * (b - 1) + 2]) * 1e-3 : 0.0,
              ((int64_t)t[4 * b + 1] - (int64_t)t[4 * b]) * 1e-3, (int)t[4 * b + 3],
              ((int64_t)t[4 * b + 2] - (int64_t)t[4 * b + 1]) * 1e-3);
    const uint64_t* t2 = t.data() + 4 * max_bar;
    for (int i = 0; i + 4 < 64 && t2[i + 4]; i += 4)
      fprintf(stderr, "wm iter %2d: stage %.2f us, Z-SpMM+flush %.2f us, barrier+chol %.2f us, Y half %.2f us\n",
              i / 4, (t2[i + 1] - t2[i]) * 1e-3, (t2[i + 2] - t2[i + 1]) * 1e-3, (t2[i + 3] - t2[i + 2]) * 1e-3,
              (t2[i + 4] - t2[i + 3]) * 1e-3);
  }
  return cudaGetLastError();
}

}  // namespace smp
