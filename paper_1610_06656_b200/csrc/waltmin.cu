// K7-K9: WAltMin (Alg. 2; Step 3, Eq. 3) with
// the REUSE_ALL partition (R11):
//   w = 1/q̂ (line 2); R = w .* P_Ω(M̃) (line 4);
//   U0 = top-r left subspace of R by subspace iteration from a Rademacher
//        start (line 5; R12), CholeskyQR2 orthonormalisation;
//   trim rows with ||U0_i|| > c sqrt(r) ||A_i||/||A||_F (line 6; R13), re-QR;
//   T x { V = argmin_V ||R^½(M̃ - U Vᵀ)|| (line 8); U = argmin_U (line 9) }
//   via per-row r×r weighted normal equations + ridge Cholesky (R14).
// Ω arrives sorted by (i,j) → CSR by slicing; CSC by a stable radix sort on j.
#include <cub/device/device_radix_sort.cuh>
#include "smp_device.cuh"
#include "smp_kernels.h"

namespace smp {

constexpr int RMAX = 16;

#define SMP_TRY(x)                          \
  do {                                      \
    cudaError_t e_ = (x);                   \
    if (e_ != cudaSuccess) return e_;       \
  } while (0)

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

__global__ void wm_iota_kernel(int32_t* __restrict__ p, int64_t cnt) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < cnt;
       s += (int64_t)gridDim.x * blockDim.x)
    p[s] = (int32_t)s;
}

__global__ void wm_init_y_kernel(double* __restrict__ Y, int64_t n2, int r, uint64_t seed) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n2 * r;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / r;
    const int l = (int)(e - j * r);
    const u32x4 w = philox4x32_10((uint32_t)j, (uint32_t)l, 0u, TAG_INIT, (uint32_t)seed,
                                  (uint32_t)(seed >> 32));
    Y[e] = (w.x & 1u) ? -1.0 : 1.0;
  }
}

// out[o] = Σ_{p in [ptr[o], ptr[o+1])} coef[s] X[other[s]],  s = perm ? perm[p] : p
__global__ void wm_spmm_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ perm,
                               const int32_t* __restrict__ other, const double* __restrict__ coef,
                               const double* __restrict__ X, int64_t nout, int r,
                               double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t o = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); o < nout; o += nw) {
    double acc[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) acc[l] = 0.0;
    const int64_t p0 = ptr[o], p1 = ptr[o + 1];
    for (int64_t q = p0 + lane; q < p1; q += 32) {
      const int64_t s = perm ? perm[q] : q;
      const double c = coef[s];
      const double* x = X + (int64_t)other[s] * r;
#pragma unroll
      for (int l = 0; l < RMAX; ++l)
        if (l < r) acc[l] = fma(c, x[l], acc[l]);
    }
#pragma unroll
    for (int l = 0; l < RMAX; ++l) {
      if (l < r) {
        double v = acc[l];
#pragma unroll
        for (int sh = 16; sh > 0; sh >>= 1) v += __shfl_xor_sync(0xffffffffu, v, sh);
        if (lane == 0) out[o * r + l] = v;
      }
    }
  }
}

// ---- CholeskyQR: G = ZᵀZ (partials per block, fixed-order sum), R = chol(G),
// Z <- Z R^{-1}.  Dead pivots (rank deficiency) give zero columns.
constexpr int GRAM_ROWS = 256;

__global__ void wm_gram_partial_kernel(const double* __restrict__ Z, int64_t n, int r,
                                       double* __restrict__ gpart) {
  __shared__ double zs[GRAM_ROWS * RMAX];
  const int64_t r0 = blockIdx.x * (int64_t)GRAM_ROWS;
  const int64_t rows = min((int64_t)GRAM_ROWS, n - r0);
  for (int e = threadIdx.x; e < rows * r; e += blockDim.x) zs[e] = Z[r0 * r + e];
  __syncthreads();
  const int npair = r * r;
  for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
    const int a = pr / r, b = pr - a * r;
    double s = 0.0;
    if (a <= b)
      for (int64_t i = 0; i < rows; ++i) s = fma(zs[i * r + a], zs[i * r + b], s);
    gpart[(int64_t)blockIdx.x * npair + pr] = s;
  }
}

__global__ void wm_gram_chol_kernel(const double* __restrict__ gpart, int nblk, int r,
                                    double* __restrict__ Rinv) {
  __shared__ double G[RMAX * RMAX];
  __shared__ double L[RMAX * RMAX];
  const int npair = r * r;
  for (int pr = threadIdx.x; pr < npair; pr += blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblk; ++b) s += gpart[(int64_t)b * npair + pr];
    G[pr] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tr = 0.0;
    for (int a = 0; a < r; ++a) tr += G[a * r + a];
    const double tol = 1e-28 * (tr > 0.0 ? tr : 1.0);
    // upper Cholesky G = RᵀR, stored as L = Rᵀ (lower)
    int dead[RMAX];
    for (int j = 0; j < r; ++j) {
      double s = G[j * r + j];
      for (int p = 0; p < j; ++p) s -= L[j * r + p] * L[j * r + p];
      dead[j] = !(s > tol);
      const double d = dead[j] ? 0.0 : sqrt(s);
      L[j * r + j] = d;
      for (int i = j + 1; i < r; ++i) {
        double t = G[j * r + i];  // G symmetric, upper stored at (j,i)
        for (int p = 0; p < j; ++p) t -= L[i * r + p] * L[j * r + p];
        L[i * r + j] = dead[j] ? 0.0 : t / d;
      }
    }
    // Rinv = (Lᵀ)^{-1}, upper triangular; dead columns -> 0
    for (int c = 0; c < r; ++c) {
      for (int i = r - 1; i >= 0; --i) {
        double t = (i == c) ? 1.0 : 0.0;
        for (int p = i + 1; p < r; ++p) t -= L[p * r + i] * Rinv[p * r + c];
        Rinv[i * r + c] = dead[i] ? 0.0 : t / L[i * r + i];
      }
    }
    for (int c = 0; c < r; ++c)
      if (dead[c])
        for (int i = 0; i < r; ++i) Rinv[i * r + c] = 0.0;
  }
}

__global__ void wm_apply_rinv_kernel(double* __restrict__ Z, int64_t n, int r,
                                     const double* __restrict__ Rinv) {
  __shared__ double Rs[RMAX * RMAX];
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) Rs[e] = Rinv[e];
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double z[RMAX], o[RMAX];
#pragma unroll
    for (int l = 0; l < RMAX; ++l) z[l] = l < r ? Z[i * r + l] : 0.0;
#pragma unroll
    for (int c = 0; c < RMAX; ++c) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < RMAX; ++l)
        if (l <= c && c < r) s = fma(z[l], Rs[l * r + c], s);
      o[c] = s;
    }
#pragma unroll
    for (int c = 0; c < RMAX; ++c)
      if (c < r) Z[i * r + c] = o[c];
  }
}

static cudaError_t orthonormalize(double* Z, int64_t n, int r, double* gpart, double* Rinv,
                                  cudaStream_t st) {
  const int nblk = (int)((n + GRAM_ROWS - 1) / GRAM_ROWS);
  for (int pass = 0; pass < 2; ++pass) {  // CholeskyQR2
    wm_gram_partial_kernel<<<nblk, 128, 0, st>>>(Z, n, r, gpart);
    wm_gram_chol_kernel<<<1, 256, 0, st>>>(gpart, nblk, r, Rinv);
    wm_apply_rinv_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(Z, n, r, Rinv);
  }
  return cudaGetLastError();
}

__global__ void wm_trim_kernel(double* __restrict__ Z, int64_t n1, int r, double trim_c,
                               const double* __restrict__ a2, const double* __restrict__ FA) {
  const double frob = sqrt(*FA);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1;
       i += (int64_t)gridDim.x * blockDim.x) {
    double rn = 0.0;
    for (int l = 0; l < r; ++l) rn += Z[i * r + l] * Z[i * r + l];
    rn = sqrt(rn);
    const double thr = trim_c * sqrt((double)r) * sqrt(a2[i]) / frob;
    if (rn > thr)
      for (int l = 0; l < r; ++l) Z[i * r + l] = 0.0;
  }
}

// ---- K9: one weighted least-squares half step.  Warp per output row o;
// lanes own entries of (G upper triangle, h); samples in CSR/CSC order.
constexpr int ALS_WARPS = 4;

__global__ void __launch_bounds__(ALS_WARPS * 32)
wm_als_kernel(const int64_t* __restrict__ ptr, const int32_t* __restrict__ perm,
              const int32_t* __restrict__ other, const double* __restrict__ w,
              const float* __restrict__ val, const double* __restrict__ X, int64_t nout, int r,
              double lam, double* __restrict__ out) {
  __shared__ double xs_all[ALS_WARPS][32][RMAX];
  __shared__ double ws_all[ALS_WARPS][32];
  __shared__ double vs_all[ALS_WARPS][32];
  __shared__ double gh_all[ALS_WARPS][RMAX * RMAX + RMAX];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double(*xs)[RMAX] = xs_all[wid];
  double* ws = ws_all[wid];
  double* vs = vs_all[wid];
  double* gh = gh_all[wid];
  const int ng = r * (r + 1) / 2, ne = ng + r;
  const int64_t nw = (int64_t)gridDim.x * ALS_WARPS;
  for (int64_t o = blockIdx.x * (int64_t)ALS_WARPS + wid; o < nout; o += nw) {
    double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // ne <= 152 -> <= 5 slots per lane
    int ea[5], eb[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int e = lane + 32 * q;
      int a = 0, b = 0;
      if (e < ng) {  // row-major upper triangle enumeration
        int rem = e;
        a = 0;
        while (rem >= r - a) { rem -= r - a; ++a; }
        b = a + rem;
      } else if (e < ne) {
        a = e - ng; b = -1;
      } else {
        a = -1; b = -1;
      }
      ea[q] = a; eb[q] = b;
    }
    const int64_t p0 = ptr[o], p1 = ptr[o + 1];
    for (int64_t base = p0; base < p1; base += 32) {
      const int nb = (int)min((int64_t)32, p1 - base);
      if (lane < nb) {
        const int64_t s = perm ? perm[base + lane] : base + lane;
        ws[lane] = w[s];
        vs[lane] = (double)val[s];
        const double* x = X + (int64_t)other[s] * r;
        for (int l = 0; l < r; ++l) xs[lane][l] = x[l];
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int a = ea[q], b = eb[q];
        if (a < 0) continue;
        double s = acc[q];
        if (b >= 0) {
          for (int m = 0; m < nb; ++m) s = __dadd_rn(s, __dmul_rn(__dmul_rn(ws[m], xs[m][a]), xs[m][b]));
        } else {
          for (int m = 0; m < nb; ++m) s = __dadd_rn(s, __dmul_rn(__dmul_rn(ws[m], vs[m]), xs[m][a]));
        }
        acc[q] = s;
      }
      __syncwarp();
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int a = ea[q], b = eb[q];
      if (a < 0) continue;
      if (b >= 0) { gh[a * r + b] = acc[q]; gh[b * r + a] = acc[q]; }
      else gh[r * r + a] = acc[q];
    }
    __syncwarp();
    if (lane == 0) {
      // ridge Cholesky solve (G + lam tr(G)/r I) x = h; empty -> 0 (R14)
      double* G = gh;
      const double* h = gh + r * r;
      double x[RMAX], y[RMAX], L[RMAX * RMAX];
      double tr = 0.0;
      for (int a = 0; a < r; ++a) tr += G[a * r + a];
      bool ok = tr > 0.0;
      for (int a = 0; a < r; ++a) x[a] = 0.0;
      if (ok) {
        const double shift = lam * tr / (double)r;
        for (int a = 0; a < r; ++a)
          for (int b = 0; b < r; ++b) L[a * r + b] = G[a * r + b] + (a == b ? shift : 0.0);
        for (int j = 0; j < r && ok; ++j) {
          double s = L[j * r + j];
          for (int q = 0; q < j; ++q) s -= L[j * r + q] * L[j * r + q];
          if (!(s > 0.0)) { ok = false; break; }
          const double d = sqrt(s);
          L[j * r + j] = d;
          for (int i = j + 1; i < r; ++i) {
            double t = L[i * r + j];
            for (int q = 0; q < j; ++q) t -= L[i * r + q] * L[j * r + q];
            L[i * r + j] = t / d;
          }
        }
        if (ok) {
          for (int i = 0; i < r; ++i) {
            double t = h[i];
            for (int q = 0; q < i; ++q) t -= L[i * r + q] * y[q];
            y[i] = t / L[i * r + i];
          }
          for (int i = r - 1; i >= 0; --i) {
            double t = y[i];
            for (int q = i + 1; q < r; ++q) t -= L[q * r + i] * x[q];
            x[i] = t / L[i * r + i];
          }
        } else {
          for (int a = 0; a < r; ++a) x[a] = 0.0;
        }
      }
      for (int a = 0; a < r; ++a) out[o * r + a] = x[a];
    }
    __syncwarp();
  }
}

__global__ void wm_to_float_kernel(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    y[e] = (float)x[e];
}

static int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  return (int)std::min<int64_t>(b, 148 * 16);
}

cudaError_t run_waltmin(const WaltminArgs& a, cudaStream_t st) {
  const int64_t cnt = a.count, n1 = a.n1, n2 = a.n2;
  const int r = a.r;
  if (r < 1 || r > RMAX) return cudaErrorInvalidValue;
  // workspace
  double *w, *wv, *Y, *Z, *U, *V, *gpart, *Rinv;
  int64_t *rptr, *cptr;
  int32_t *iota, *perm, *jsorted;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
  const int64_t c1 = cnt > 0 ? cnt : 1;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  const int gblk = (int)((nmax + GRAM_ROWS - 1) / GRAM_ROWS);
  SMP_TRY(cudaMallocAsync(&w, c1 * 8, st));
  SMP_TRY(cudaMallocAsync(&wv, c1 * 8, st));
  SMP_TRY(cudaMallocAsync(&Y, n2 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&Z, n1 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&U, n1 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&V, n2 * r * 8, st));
  SMP_TRY(cudaMallocAsync(&gpart, (int64_t)gblk * r * r * 8, st));
  SMP_TRY(cudaMallocAsync(&Rinv, RMAX * RMAX * 8, st));
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

  // line 5: subspace iteration on R = w .* P_Ω(M̃)
  wm_init_y_kernel<<<grid_for(n2 * r, 256), 256, 0, st>>>(Y, n2, r, a.seed);
  const int spmm_blocks1 = grid_for(n1 * 32, 256), spmm_blocks2 = grid_for(n2 * 32, 256);
  for (int it = 0; it < a.init_iters; ++it) {
    wm_spmm_kernel<<<spmm_blocks1, 256, 0, st>>>(rptr, nullptr, a.J, wv, Y, n1, r, Z);
    SMP_TRY(orthonormalize(Z, n1, r, gpart, Rinv, st));
    wm_spmm_kernel<<<spmm_blocks2, 256, 0, st>>>(cptr, perm, a.I, wv, Z, n2, r, Y);
    SMP_TRY(orthonormalize(Y, n2, r, gpart, Rinv, st));
  }
  if (a.init_iters == 0) {
    // no iteration: U0 = orth(R Y0)
    wm_spmm_kernel<<<spmm_blocks1, 256, 0, st>>>(rptr, nullptr, a.J, wv, Y, n1, r, Z);
    SMP_TRY(orthonormalize(Z, n1, r, gpart, Rinv, st));
  }
  // line 6: trim, then re-orthonormalise
  if (a.trim_c > 0.0) {
    wm_trim_kernel<<<grid_for(n1, 256), 256, 0, st>>>(Z, n1, r, a.trim_c, a.a_norm2, a.FA);
    SMP_TRY(orthonormalize(Z, n1, r, gpart, Rinv, st));
  }
  SMP_TRY(cudaMemcpyAsync(U, Z, n1 * r * 8, cudaMemcpyDeviceToDevice, st));
  // lines 7-10
  const int als1 = grid_for(n1 * 32, ALS_WARPS * 32), als2 = grid_for(n2 * 32, ALS_WARPS * 32);
  if (a.T == 0) SMP_TRY(cudaMemsetAsync(V, 0, n2 * r * 8, st));
  for (int t = 0; t < a.T; ++t) {
    wm_als_kernel<<<als2, ALS_WARPS * 32, 0, st>>>(cptr, perm, a.I, w, a.val, U, n2, r, a.lam, V);
    wm_als_kernel<<<als1, ALS_WARPS * 32, 0, st>>>(rptr, nullptr, a.J, w, a.val, V, n1, r, a.lam, U);
  }
  wm_to_float_kernel<<<grid_for(n1 * r, 256), 256, 0, st>>>(U, n1 * r, a.U);
  wm_to_float_kernel<<<grid_for(n2 * r, 256), 256, 0, st>>>(V, n2 * r, a.V);
  SMP_TRY(cudaGetLastError());
  cudaFreeAsync(w, st); cudaFreeAsync(wv, st); cudaFreeAsync(Y, st); cudaFreeAsync(Z, st);
  cudaFreeAsync(U, st); cudaFreeAsync(V, st); cudaFreeAsync(gpart, st); cudaFreeAsync(Rinv, st);
  cudaFreeAsync(rptr, st); cudaFreeAsync(cptr, st); cudaFreeAsync(iota, st);
  cudaFreeAsync(perm, st); cudaFreeAsync(jsorted, st); cudaFreeAsync(cub_tmp, st);
  return cudaGetLastError();
}

}  // namespace smp
