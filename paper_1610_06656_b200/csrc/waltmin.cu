// K7-K9: WAltMin (Alg. 2; Step 3, Eq. 3) with
// the REUSE_ALL partition (R11):
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

// ptr[o] = lower_bound(keys, o) for o in [0, nout]
__global__ void wm_ptr_kernel(const int32_t* __restrict__ keys, int64_t cnt, int64_t nout,
                              int64_t* __restrict__ ptr) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o <= nout;
       o += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = cnt;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < o) lo = mid + 1; else hi = mid;
    }
    ptr[o] = lo;
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

cudaError_t run_waltmin(const WaltminArgs& a, cudaStream_t st) {
  const int64_t cnt = a.count, n1 = a.n1, n2 = a.n2;
  const int r = a.r;
  if (r < 1 || r > 16) return cudaErrorInvalidValue;
  // workspace
  double *w, *wv, *cw, *cwv, *Y, *Z, *U, *V, *gpart;
  unsigned* bar;
  int64_t *rptr, *cptr;
  int32_t *iota, *perm, *jsorted, *cI;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  const int64_t c1 = cnt > 0 ? cnt : 1;
  const int gctas = waltmin_grid_ctas();
  if (gctas < 1) return cudaErrorNoDevice;
  SMP_TRY(cudaMallocAsync(&w, c1 * 8, st));
  SMP_TRY(cudaMallocAsync(&wv, c1 * 8, st));
  SMP_TRY(cudaMallocAsync(&cw, c1 * 8, st));
  SMP_TRY(cudaMallocAsync(&cwv, c1 * 8, st));
  SMP_TRY(cudaMallocAsync(&cI, c1 * 4, st));
  SMP_TRY(cudaMallocAsync(&Y, n2 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&Z, n1 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&U, n1 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&V, n2 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&gpart, (int64_t)2 * gctas * r * (r + 1) / 2 * 8, st));
  SMP_TRY(cudaMallocAsync(&bar, 64, st));
  SMP_TRY(cudaMallocAsync(&rptr, (n1 + 1) * 8, st));
  SMP_TRY(cudaMallocAsync(&cptr, (n2 + 1) * 8, st));
  SMP_TRY(cudaMallocAsync(&iota, c1 * 4, st));
  SMP_TRY(cudaMallocAsync(&perm, c1 * 4, st));
  SMP_TRY(cudaMallocAsync(&jsorted, c1 * 4, st));

  wm_weights_kernel<<<grid_for(cnt, 256), 256, 0, st>>>(a.qhat, a.val, cnt, w, wv);
  wm_ptr_kernel<<<grid_for(n1 + 1, 256), 256, 0, st>>>(a.I, cnt, n1, rptr);
  // CSC: stable radix sort of (J, s) -> perm; column pointers on sorted J
  wm_iota_kernel<<<grid_for(cnt, 256), 256, 0, st>>>(iota, cnt);
  int end_bit = 1;
  while (end_bit < 32 && ((int64_t)1 << end_bit) <= n2) ++end_bit;
  SMP_TRY(cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, a.J, jsorted, iota, perm, (int)cnt, 0,
                                          end_bit, st));
  SMP_TRY(cudaMallocAsync(&cub_tmp, cub_bytes > 0 ? cub_bytes : 1, st));
  SMP_TRY(cub::DeviceRadixSort::SortPairs(cub_tmp, cub_bytes, a.J, jsorted, iota, perm, (int)cnt, 0,
                                          end_bit, st));
  wm_ptr_kernel<<<grid_for(n2 + 1, 256), 256, 0, st>>>(jsorted, cnt, n2, cptr);
  wm_gather_csc_kernel<<<grid_for(cnt, 256), 256, 0, st>>>(perm, a.I, w, wv, cnt, cI, cw, cwv);

  // heavy rows / columns: stable compaction (fixed order -> fixed CTA
  // assignment -> deterministic Gram partials)
  const int64_t nmax = std::max<int64_t>(std::max<int64_t>(n1, n2), 1);
  // Split a row over a CTA only when it is long in absolute terms AND several
  // times a warp's average share: the CTA runs its heavy rows before its light
  // ones, so splitting rows near the average only serialises work (cfg1:
  // rows <= 564 samples, 119 per warp -> none split).  SMP_WM_HEAVY overrides
  // the threshold (0 = warp-per-row only; tuning).
  const char* hv = getenv("SMP_WM_HEAVY");
  const int64_t avg_warp = cnt / ((int64_t)gctas * WM_WARPS) + 1;
  const int64_t heavy_thr = hv ? atoll(hv) : std::max<int64_t>(WM_HEAVY, 4 * avg_warp);
  uint8_t *hfr, *hfc;
  int32_t *hidx, *hlr, *hlc, *nh;
  void* sel_tmp = nullptr;
  size_t sel_bytes = 0;
  SMP_TRY(cudaMallocAsync(&hfr, n1 + 1, st));
  SMP_TRY(cudaMallocAsync(&hfc, n2 + 1, st));
  SMP_TRY(cudaMallocAsync(&hidx, nmax * 4, st));
  SMP_TRY(cudaMallocAsync(&hlr, (n1 + 1) * 4, st));
  SMP_TRY(cudaMallocAsync(&hlc, (n2 + 1) * 4, st));
  SMP_TRY(cudaMallocAsync(&nh, 2 * 4, st));
  SMP_TRY(cub::DeviceSelect::Flagged(nullptr, sel_bytes, hidx, hfr, hlr, nh, (int)nmax, st));
  SMP_TRY(cudaMallocAsync(&sel_tmp, sel_bytes > 0 ? sel_bytes : 1, st));
  SMP_TRY(cudaMemsetAsync(nh, 0, 2 * 4, st));
  if (n1 > 0) {
    wm_heavy_flags_kernel<<<grid_for(n1, 256), 256, 0, st>>>(rptr, n1, heavy_thr, hfr, hidx);
    SMP_TRY(cub::DeviceSelect::Flagged(sel_tmp, sel_bytes, hidx, hfr, hlr, nh, (int)n1, st));
  }
  if (n2 > 0) {
    wm_heavy_flags_kernel<<<grid_for(n2, 256), 256, 0, st>>>(cptr, n2, heavy_thr, hfc, hidx);
    SMP_TRY(cub::DeviceSelect::Flagged(sel_tmp, sel_bytes, hidx, hfc, hlc, nh + 1, (int)n2, st));
  }

  // lines 5-10: one cooperative persistent kernel
  SMP_TRY(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st));
  WMParams p{};
  p.n1 = n1; p.n2 = n2; p.count = cnt; p.T = a.T; p.init_iters = a.init_iters;
  p.trim_c = a.trim_c; p.lam = a.lam; p.seed = a.seed;
  p.rptr = rptr; p.J = a.J; p.w = w; p.wv = wv;
  p.cptr = cptr; p.cI = cI; p.cw = cw; p.cwv = cwv;
  p.a2 = a.a_norm2; p.FA = a.FA;
  p.Y = Y; p.Z = Z; p.U = U; p.V = V; p.gpart = gpart; p.bar = bar;
  p.Uout = a.U; p.Vout = a.V;
  const char* xl = getenv("SMP_WM_L1");  // 0: L2-only gathers (A/B switch)
  p.x_l1 = (xl && atoi(xl) == 0) ? 0 : 1;
  if (heavy_thr > 0) {
    p.heavy_r = hlr; p.nheavy_r = nh; p.hflag_r = hfr;
    p.heavy_c = hlc; p.nheavy_c = nh + 1; p.hflag_c = hfc;
  }
  const char* tr = getenv("SMP_WM_TRACE");
  uint64_t* trace = nullptr;
  const int max_bar = 2 * (a.init_iters + 4) + 2 * a.T + 8;
  if (tr && atoi(tr)) {
    SMP_TRY(cudaMalloc(&trace, 4 * 8 * (size_t)max_bar + 64 * 8));
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
    cudaFree(trace);
  }
  SMP_TRY(cudaGetLastError());
  cudaFreeAsync(w, st); cudaFreeAsync(wv, st); cudaFreeAsync(cw, st); cudaFreeAsync(cwv, st);
  cudaFreeAsync(cI, st); cudaFreeAsync(Y, st); cudaFreeAsync(Z, st);
  cudaFreeAsync(U, st); cudaFreeAsync(V, st); cudaFreeAsync(gpart, st); cudaFreeAsync(bar, st);
  cudaFreeAsync(rptr, st); cudaFreeAsync(cptr, st); cudaFreeAsync(iota, st);
  cudaFreeAsync(perm, st); cudaFreeAsync(jsorted, st); cudaFreeAsync(cub_tmp, st);
  cudaFreeAsync(hfr, st); cudaFreeAsync(hfc, st); cudaFreeAsync(hidx, st); cudaFreeAsync(hlr, st);
  cudaFreeAsync(hlc, st); cudaFreeAsync(nh, st); cudaFreeAsync(sel_tmp, st);
  return cudaGetLastError();
}

}  // namespace smp
