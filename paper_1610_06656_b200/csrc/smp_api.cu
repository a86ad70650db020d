// libsmp.so: C-ABI implementation (include/smp.h).  Owns the handle, the
// workspace and the launch sequence of the SMP-PCA hot path:
//   sketch_block -> K1 (tcgen05 sketch + fused norms) -> K2 (split-K reduce)
//   finalize     -> K4 + R5 pairwise Frobenius tree
//   sample_est.  -> alpha/beta, K5 count, scan, K5 write, K6 SDDMM
//   waltmin      -> K7-K9
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/smp.h"
#include "smp_device.cuh"
#include "smp_kernels.h"

cudaError_t smp_convert_f64_f32(const double* x, int64_t n, float* y, cudaStream_t st);

struct smp_handle {
  smp_sketch_desc d;
  cudaStream_t st = nullptr;
  int dev = 0;
  int64_t n1 = 0, n2 = 0, ntot = 0;
  int k = 0;
  float* acc_sk = nullptr;     // [ntot][k] unscaled sums
  double* acc_nrm = nullptr;   // [ntot]
  float* part = nullptr;
  int64_t part_cap = 0;
  double* pnorm = nullptr;
  int64_t pnorm_cap = 0;
  double* xchg = nullptr;      // combine exchange buffer [ntot*k | ntot] (fp64)
  int64_t xchg_cap = 0;
  uint16_t* planes = nullptr;
  int64_t planes_cap = 0;
  // pipelined plane split (sketch_dense_split): double buffers, aux stream
  uint16_t* planes2[2] = {nullptr, nullptr};
  int64_t planes2_cap[2] = {0, 0};
  double* pnorm2[2] = {nullptr, nullptr};
  int64_t pnorm2_cap[2] = {0, 0};
  uint16_t* panel2[2] = {nullptr, nullptr};
  int64_t panel2_cap[2] = {0, 0};
  cudaEvent_t ev_prep[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr}, ev_sync = nullptr;
  cudaStream_t aux_st = nullptr;
  // row-multinomial sampler scratch
  smp::MnWorkspace mn;
  uint16_t* pi_panel = nullptr;  // K1 Gaussian Π panel (κ-major)
  int64_t pi_panel_cap = 0;
  int64_t panel_row0 = -1, panel_ld = 0, panel_kpad = 0;  // rows the panel holds
  // LELA pass 2 transposed chunks
  float* lela_at = nullptr;
  float* lela_bt = nullptr;
  int64_t lela_at_cap = 0, lela_bt_cap = 0;
  double* lela_pn = nullptr;
  int64_t lela_pn_cap = 0;
  // finalized state
  float* fin_sk = nullptr;     // [ntot][k]
  double* fin_sknorm = nullptr;
  double* fin_D = nullptr;
  double* FAFB = nullptr;      // [2]
  int* status = nullptr;
  double* pw_scratch = nullptr;
  int64_t pw_cap = 0;
  bool finalized = false;
  // sampling scratch
  double* alpha = nullptr;     // [n1 + n2] (alpha then beta)
  int64_t* blk = nullptr;
  int64_t blk_cap = 0;
  int64_t* d_total = nullptr;
  int64_t* h_total = nullptr;  // pinned
  int* h_status = nullptr;     // pinned
  double* h_fafb = nullptr;    // pinned
  // host staging
  void* stage[2] = {nullptr, nullptr};
  int64_t stage_bytes = 0;
  cudaStream_t copy_st = nullptr;
  cudaEvent_t ev_copied[2] = {nullptr, nullptr};
  cudaEvent_t ev_used[2] = {nullptr, nullptr};
  int64_t launches = 0;
  smp::CsrWorkspace csr;
  // K1 timing instrumentation
  bool timing = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used_n = 0;
  std::string err;
};

namespace {

// NVTX range over one ABI call (visible in nsys / ncu --nvtx timelines)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

smp_status fail(smp_handle* h, smp_status s, const char* fmt, ...) {
  if (h) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    h->err = buf;
  }
  return s;
}

smp_status cuda_fail(smp_handle* h, cudaError_t e, const char* where) {
  return fail(h, SMP_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

#define CK(h, x, where)                                 \
  do {                                                  \
    cudaError_t e_ = (x);                               \
    if (e_ != cudaSuccess) return cuda_fail(h, e_, where); \
  } while (0)

template <class T>
cudaError_t ensure(T*& p, int64_t& cap, int64_t need) {
  if (need <= cap) return cudaSuccess;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  cudaError_t e = cudaMalloc(&p, (size_t)need * sizeof(T));
  if (e == cudaSuccess) cap = need;
  return e;
}

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

int srht_L(int64_t d) {
  int L = 1;
  while (L < 62 && ((int64_t)1 << L) < d) ++L;
  return L;
}

// Π kind code passed to the kernels (SRHT carries its Hadamard order: 16 + L)
int pi_code(const smp_handle* h) {
  return h->d.pi_kind == SMP_PI_SRHT ? 16 + srht_L(h->d.d_total) : h->d.pi_kind;
}

// split-K factor for the tcgen05 sketch.  Two constraints:
//  * accuracy: a CTA's fp32 TMEM accumulation chain is at most
//    K1_MAX_KB K-blocks (64 rows each); measured: 41.7K MMA updates per
//    chain (cfg4 with 3 splits) gave 1.6e-5 relative column error, above
//    the 1e-5 tolerance, 3.6K updates (cfg1) gave < 4e-6 (R21);
//  * occupancy: fill the 148 SMs with >= 95% of the last wave, fewest
//    splits first (searched up to 2x the accuracy minimum).
//    With a Gaussian Π the (plane-split) products carry 12 significant bits
//    and the chain is capped at 16,384 rows: 14.5K-row chains measured
//    1.5e-6, 58K-row chains 4.3e-5 (cfg4, full size).
constexpr int K1_MAX_KB = 1024;        // 65,536 rows per accumulation chain (±1 Π)
constexpr int K1_MAX_KB_GAUSS = 256;   // 16,384 rows (Gaussian Π)

// K1's off-critical-path barrier waiters (TMA producer, Π generators, norm
// warps, epilogue) sleep this long between tests instead of spinning
// (SMP_K1_BACKOFF_NS overrides; 0 = spin).
constexpr uint32_t K1_BACKOFF_NS = 0;

int choose_splits(int tiles, int kb_total, int max_kb) {
  const int sms = 148;
  const int smin = std::max(1, (kb_total + max_kb - 1) / max_kb);
  int best_s = smin;
  double best_eff = -1.0;
  const int smax = std::max(smin, std::min(kb_total, std::max(64, 2 * smin)));
  for (int s = smin; s <= smax; ++s) {
    const int64_t ctas = (int64_t)tiles * s;
    const int64_t waves = (ctas + sms - 1) / sms;
    const double eff = (double)ctas / (double)(waves * sms);
    if (eff >= 0.95) return s;
    if (eff > best_eff + 1e-9) { best_eff = eff; best_s = s; }
  }
  return best_s;
}

// One matrix, one dense bf16 block through K1 + K2.
smp_status sketch_dense_bf16(smp_handle* h, int64_t row0, int64_t rows, const void* X, int64_t ldx,
                             int64_t ncols, int planes, int64_t col_off, bool do_norms,
                             const uint16_t* ext_panel = nullptr, const int32_t* col_map = nullptr) {
  using namespace smp;
  const int k = h->k;
  SketchTCParams p{};
  p.rows = rows;
  p.row0 = row0;
  p.n = (int32_t)ncols;
  p.k = k;
  p.n_tiles = (int32_t)((ncols + 255) / 256);
  p.k_tiles = (k + 255) / 256;
  p.kb_total = (int32_t)((rows + 63) / 64);
  p.splits = choose_splits(2 * p.n_tiles * p.k_tiles, p.kb_total,
                           h->d.pi_kind == SMP_PI_GAUSSIAN ? K1_MAX_KB_GAUSS : K1_MAX_KB);
  p.kind = pi_code(h);
  p.do_norms = do_norms ? 1 : 0;
  { const char* dbg = getenv("SMP_K1_DEBUG"); p.debug = dbg ? atoi(dbg) : 0; }
  { const char* bo = getenv("SMP_K1_BACKOFF_NS"); p.backoff_ns = bo ? (uint32_t)atoi(bo) : K1_BACKOFF_NS; }
  p.seed = h->d.seed;
  CK(h, ensure(h->part, h->part_cap, (int64_t)p.splits * ncols * k), "alloc partials");
  CK(h, ensure(h->pnorm, h->pnorm_cap, (int64_t)p.splits * p.k_tiles * ncols), "alloc pnorm");
  p.part = h->part;
  p.pnorm = h->pnorm;
  p.pi_panel = nullptr;
  p.pi_ld = 0;
  static const int panel_mode = [] {
    const char* e = getenv("SMP_K1_PANEL");  // tuning switch: 1 = panel for every Π kind
    return e ? atoi(e) : 0;
  }();
  const bool panel_fits = (int64_t)p.k_tiles * 256 * (int64_t)p.kb_total * 64 <= (1ll << 30);
  if (ext_panel) {  // generated by the caller (pipelined split path)
    p.pi_panel = ext_panel;
    p.pi_ld = (int64_t)p.kb_total * 64;
  } else if ((p.kind == SMP_PI_GAUSSIAN || panel_mode == 1) && panel_fits) {
    // Π once per block into a κ-major panel that K1 streams by TMA (Gaussian:
    // ~33 ALU ops per entry would otherwise be repeated for every column
    // tile).  A and B blocks over the same rows reuse the panel.
    const int64_t ld = (int64_t)p.kb_total * 64;
    const int64_t kpad = (int64_t)p.k_tiles * 256;
    const bool cached = h->pi_panel && h->panel_row0 == row0 && h->panel_ld == ld &&
                        h->panel_kpad == kpad;
    if (!cached) {
      CK(h, ensure(h->pi_panel, h->pi_panel_cap, kpad * ld), "alloc pi panel");
      CK(h, launch_pi_panel_kmajor(p.kind, p.seed, k, (int)kpad, row0, ld, ld, h->pi_panel, h->st),
         "pi panel");
      h->launches += 1;
      h->panel_row0 = row0;
      h->panel_ld = ld;
      h->panel_kpad = kpad;
    }
    p.pi_panel = h->pi_panel;
    p.pi_ld = ld;
  }
  const bool time_k1 = h->timing && h->d.input != SMP_IN_CSR_F32;  // CSR handles time K3d
  if (time_k1) {
    while (h->ev_pool.size() < h->ev_used_n + 2) {
      cudaEvent_t e;
      CK(h, cudaEventCreate(&e), "event");
      h->ev_pool.push_back(e);
    }
    CK(h, cudaEventRecord(h->ev_pool[h->ev_used_n], h->st), "event");
  }
  CK(h, launch_sketch_tc(X, ldx, p, h->st), "sketch_tc");
  if (time_k1) {
    CK(h, cudaEventRecord(h->ev_pool[h->ev_used_n + 1], h->st), "event");
    h->ev_used_n += 2;
  }
  const int64_t n = ncols / planes;
  CK(h, launch_reduce_sketch(h->part, p.splits, planes, n, k,
                             col_map ? h->acc_sk : h->acc_sk + col_off * k, h->st, col_map),
     "reduce_sketch");
  h->launches += 2;
  if (do_norms) {
    CK(h, launch_reduce_norms(h->pnorm, p.splits * p.k_tiles, n,
                              col_map ? h->acc_nrm : h->acc_nrm + col_off, h->st, col_map),
       "reduce_norms");
    h->launches += 1;
  }
  return SMP_OK;
}

// One matrix, one block split into exact bf16 planes per row chunk (fp32
// inputs always; bf16 inputs with a Gaussian Π, R21), norms from
// the input values in fp64, then K1 over the (planes · n)-wide plane matrix.
smp_status sketch_dense_split(smp_handle* h, int64_t row0, int64_t rows, const void* X, int x_bf16,
                              int64_t ldx, int64_t n, int64_t col_off) {
  using namespace smp;
  const bool gauss = h->d.pi_kind == SMP_PI_GAUSSIAN;
  const int mode = x_bf16 ? 2 : (gauss ? 4 : 3);
  const int np = x_bf16 ? 2 : 3;
  const int64_t ldp = ((np * n + 7) / 8) * 8;
  const int64_t kpad = ((h->k + 255) / 256) * 256;
  int64_t chunk = std::max<int64_t>(64, std::min<int64_t>(rows, (int64_t)(2048ll << 20) / (ldp * 2)));
  if (gauss)  // K1's Π panel for a chunk: at most 512 MB (kpad x chunk bf16)
    chunk = std::max<int64_t>(64, std::min<int64_t>(chunk, (512ll << 20) / (kpad * 2)));
  const int seg_rows = 512;  // rows per split thread (and per fp64 norm partial)
  const int64_t chunk_pad = ((chunk + 63) / 64) * 64;
  const int64_t segs_max = (chunk + seg_rows - 1) / seg_rows;
  // Row chunks, double-buffered: split into planes (HBM-bound) and the
  // Gaussian Π panel (ALU-bound), then K1 (tensor-bound).
  for (int b = 0; b < 2; ++b) {
    CK(h, ensure(h->planes2[b], h->planes2_cap[b], chunk_pad * ldp), "alloc planes");
    CK(h, ensure(h->pnorm2[b], h->pnorm2_cap[b], segs_max * n), "alloc pnorm");
    if (gauss) CK(h, ensure(h->panel2[b], h->panel2_cap[b], kpad * chunk_pad), "alloc pi panel");
    if (!h->ev_prep[b]) CK(h, cudaEventCreateWithFlags(&h->ev_prep[b], cudaEventDisableTiming), "event");
    if (!h->ev_free[b]) CK(h, cudaEventCreateWithFlags(&h->ev_free[b], cudaEventDisableTiming), "event");
  }
  // SMP_SPLIT_OVERLAP=1 runs the split on a second stream, overlapped with K1
  // (measured no faster on cfg4: the kernels share the SMs); default: one stream
  static const bool overlap = [] {
    const char* e = getenv("SMP_SPLIT_OVERLAP");
    return e && atoi(e) == 1;
  }();
  if (overlap && !h->aux_st) CK(h, cudaStreamCreateWithFlags(&h->aux_st, cudaStreamNonBlocking), "stream");
  cudaStream_t aux = overlap ? h->aux_st : h->st;
  if (!h->ev_sync) CK(h, cudaEventCreateWithFlags(&h->ev_sync, cudaEventDisableTiming), "event");
  // aux starts after everything already on the main stream (reset, earlier blocks)
  CK(h, cudaEventRecord(h->ev_sync, h->st), "event");
  CK(h, cudaStreamWaitEvent(aux, h->ev_sync, 0), "wait");
  const int64_t es = x_bf16 ? 2 : 4;
  int i = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += chunk, ++i) {
    const int b = i & 1;
    const int64_t rc = std::min(chunk, rows - r0);
    const int64_t segs = (rc + seg_rows - 1) / seg_rows;
    if (i >= 2) CK(h, cudaStreamWaitEvent(aux, h->ev_free[b], 0), "wait");
    CK(h, launch_split_planes(static_cast<const uint8_t*>(X) + r0 * ldx * es, x_bf16, ldx, rc, n, mode,
                              h->planes2[b], ldp, h->pnorm2[b], seg_rows, aux),
       "split_planes");
    CK(h, launch_reduce_norms(h->pnorm2[b], (int)segs, n, h->acc_nrm + col_off, aux), "reduce_norms");
    h->launches += 2;
    if (gauss) {
      const int64_t ld = ((rc + 63) / 64) * 64;
      CK(h, launch_pi_panel_kmajor(pi_code(h), h->d.seed, h->k, (int)kpad, row0 + r0, ld, ld,
                                   h->panel2[b], aux),
         "pi panel");
      h->launches += 1;
    }
    CK(h, cudaEventRecord(h->ev_prep[b], aux), "event");
    CK(h, cudaStreamWaitEvent(h->st, h->ev_prep[b], 0), "wait");
    smp_status s = sketch_dense_bf16(h, row0 + r0, rc, h->planes2[b], ldp, np * n, np, col_off, false,
                                     gauss ? h->panel2[b] : nullptr);
    if (s != SMP_OK) return s;
    CK(h, cudaEventRecord(h->ev_free[b], h->st), "event");
  }
  // the norms (reduced on aux) are complete before anything later on main
  CK(h, cudaEventRecord(h->ev_sync, aux), "event");
  CK(h, cudaStreamWaitEvent(h->st, h->ev_sync, 0), "wait");
  return SMP_OK;
}

// fp32 block through K1F (split fused into the sketch kernel): Π panel per
// row chunk (κ-major, <= 512 MB), K1F, K2 over the 3 planes, norms.
smp_status sketch_dense_f32_fused(smp_handle* h, int64_t row0, int64_t rows, const float* X, int64_t ldx,
                                  int64_t n, int64_t col_off) {
  using namespace smp;
  const bool gauss = h->d.pi_kind == SMP_PI_GAUSSIAN;
  const int k = h->k;
  const int k_tiles = (k + 255) / 256;
  const int64_t kpad = (int64_t)k_tiles * 256;
  int64_t chunk = std::min<int64_t>(rows, (512ll << 20) / (kpad * 2));
  chunk = std::max<int64_t>(64, (chunk / 64) * 64);
  // Several row chunks: the Π panel of chunk c + 1 is generated on a second
  // stream (two panel buffers), released as soon as K1F of chunk c - 1 is done,
  // so it runs under the K2 / norm reduce of chunk c - 1 and the ramp of K1F(c)
  // instead of after them.  Measured on cfg4 (0.58 ms of panel per 3.1 ms of
  // K1F): stage 15.6 vs 15.9-16.2 ms serial.  A true side-by-side run does not
  // pay: only ONE 256-thread panel block fits beside a K1F CTA (registers), and
  // at 1-2 blocks per SM the latency-bound panel kernel takes longer than K1F
  // (SMP_F32_PANEL_BLOCKS=1: 19.3 ms, 2: 18.4 ms).  SMP_F32_PANEL_OVERLAP=0: serial.
  const int64_t nchunks = (rows + chunk - 1) / chunk;
  const bool pipe = nchunks >= 2 && [] {
    const char* e = getenv("SMP_F32_PANEL_OVERLAP");
    return e ? atoi(e) != 0 : true;
  }();
  const int64_t ld_max = ((std::min(chunk, rows) + 63) / 64) * 64;
  uint16_t* pan[2] = {nullptr, nullptr};
  const int bg_blocks = [] {   // blocks per SM of the background panel launches (tuning)
    const char* e = getenv("SMP_F32_PANEL_BLOCKS");
    return e ? atoi(e) : 16;
  }();
  auto gen_panel = [&](int64_t c, cudaStream_t st) -> cudaError_t {
    const int64_t r0c = c * chunk, rcc = std::min(chunk, rows - r0c);
    const int64_t ldc = ((rcc + 63) / 64) * 64;
    return launch_pi_panel_kmajor(pi_code(h), h->d.seed, k, (int)kpad, row0 + r0c, ldc, ldc, pan[c & 1], st,
                                  c == 0 ? 16 : bg_blocks);
  };
  if (pipe) {
    CK(h, ensure(h->pi_panel, h->pi_panel_cap, kpad * ld_max), "alloc pi panel");
    CK(h, ensure(h->panel2[0], h->panel2_cap[0], kpad * ld_max), "alloc pi panel");
    pan[0] = h->pi_panel;
    pan[1] = h->panel2[0];
    if (!h->aux_st) CK(h, cudaStreamCreateWithFlags(&h->aux_st, cudaStreamNonBlocking), "stream");
    for (int b = 0; b < 2; ++b) {
      if (!h->ev_prep[b]) CK(h, cudaEventCreateWithFlags(&h->ev_prep[b], cudaEventDisableTiming), "event");
      if (!h->ev_free[b]) CK(h, cudaEventCreateWithFlags(&h->ev_free[b], cudaEventDisableTiming), "event");
    }
    if (!h->ev_sync) CK(h, cudaEventCreateWithFlags(&h->ev_sync, cudaEventDisableTiming), "event");
    // the second stream starts after everything already queued on the main one
    CK(h, cudaEventRecord(h->ev_sync, h->st), "event");
    CK(h, cudaStreamWaitEvent(h->aux_st, h->ev_sync, 0), "wait");
    CK(h, gen_panel(0, h->aux_st), "pi panel");
    CK(h, cudaEventRecord(h->ev_prep[0], h->aux_st), "event");
    h->launches += 1;
    h->panel_row0 = -1;   // the cached single-chunk panel is overwritten
  }
  int64_t ci = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += chunk, ++ci) {
    const int64_t rc = std::min(chunk, rows - r0);
    SketchTCParams p{};
    p.rows = rc;
    p.row0 = row0 + r0;
    p.n = (int32_t)n;
    p.k = k;
    p.n_tiles = (int32_t)((n + 127) / 128);
    p.k_tiles = k_tiles;
    p.kb_total = (int32_t)((rc + 63) / 64);
    p.splits = choose_splits(2 * p.n_tiles * p.k_tiles, p.kb_total, gauss ? K1_MAX_KB_GAUSS : K1_MAX_KB);
    p.kind = pi_code(h);
    p.do_norms = 1;
    p.seed = h->d.seed;
    const int64_t ld = (int64_t)p.kb_total * 64;
    CK(h, ensure(h->part, h->part_cap, (int64_t)p.splits * 3 * n * k), "alloc partials");
    CK(h, ensure(h->pnorm, h->pnorm_cap, (int64_t)p.splits * p.k_tiles * n), "alloc pnorm");
    if (pipe) {
      if (ci + 1 < nchunks) {
        // buffer (ci + 1) & 1 was last read by K1F of chunk ci - 1
        if (ci >= 1) CK(h, cudaStreamWaitEvent(h->aux_st, h->ev_free[(ci + 1) & 1], 0), "wait");
        CK(h, gen_panel(ci + 1, h->aux_st), "pi panel");
        CK(h, cudaEventRecord(h->ev_prep[(ci + 1) & 1], h->aux_st), "event");
        h->launches += 1;
      }
      CK(h, cudaStreamWaitEvent(h->st, h->ev_prep[ci & 1], 0), "wait");
    } else {
      CK(h, ensure(h->pi_panel, h->pi_panel_cap, kpad * ld), "alloc pi panel");
      const bool cached = h->panel_row0 == p.row0 && h->panel_ld == ld && h->panel_kpad == kpad;
      if (!cached) {
        CK(h, launch_pi_panel_kmajor(p.kind, p.seed, k, (int)kpad, p.row0, ld, ld, h->pi_panel, h->st), "pi panel");
        h->launches += 1;
        h->panel_row0 = p.row0;
        h->panel_ld = ld;
        h->panel_kpad = kpad;
      }
    }
    p.part = h->part;
    p.pnorm = h->pnorm;
    p.pi_panel = pipe ? pan[ci & 1] : h->pi_panel;
    p.pi_ld = ld;
    { const char* dbg = getenv("SMP_K1F_DEBUG"); p.debug = dbg ? atoi(dbg) : 0; }  // ablation only
    if (h->timing) {
      while (h->ev_pool.size() < h->ev_used_n + 2) {
        cudaEvent_t e;
        CK(h, cudaEventCreate(&e), "event");
        h->ev_pool.push_back(e);
      }
      CK(h, cudaEventRecord(h->ev_pool[h->ev_used_n], h->st), "event");
    }
    CK(h, launch_sketch_tc_f32(X + r0 * ldx, ldx, p, gauss ? 4 : 3, h->st), "sketch_tc_f32");
    if (h->timing) {
      CK(h, cudaEventRecord(h->ev_pool[h->ev_used_n + 1], h->st), "event");
      h->ev_used_n += 2;
    }
    if (pipe) CK(h, cudaEventRecord(h->ev_free[ci & 1], h->st), "event");
    CK(h, launch_reduce_sketch(h->part, p.splits, 3, n, k, h->acc_sk + col_off * k, h->st), "reduce_sketch");
    CK(h, launch_reduce_norms(h->pnorm, p.splits * p.k_tiles, n, h->acc_nrm + col_off, h->st), "reduce_norms");
    h->launches += 3;
  }
  return SMP_OK;
}

// TMA needs a 16-byte aligned base and row pitch: repack unaligned bf16
// blocks through the handle's staging buffer (device to device, chunked).
smp_status sketch_dense_bf16_repack(smp_handle* h, int64_t row0, int64_t rows, const void* X,
                                    int64_t ldx, int64_t n, int64_t col_off) {
  const int64_t ldp = ((n + 7) / 8) * 8;
  const int64_t chunk = std::max<int64_t>(64, std::min<int64_t>(rows, (int64_t)(256ll << 20) / (ldp * 2)));
  CK(h, ensure(h->planes, h->planes_cap, chunk * ldp), "alloc repack");
  for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
    const int64_t rc = std::min(chunk, rows - r0);
    CK(h, cudaMemcpy2DAsync(h->planes, ldp * 2, static_cast<const uint16_t*>(X) + r0 * ldx, ldx * 2,
                            n * 2, rc, cudaMemcpyDeviceToDevice, h->st), "repack");
    smp_status s = sketch_dense_bf16(h, row0 + r0, rc, h->planes, ldp, n, 1, col_off, true);
    if (s != SMP_OK) return s;
  }
  return SMP_OK;
}

smp_status check_rows(smp_handle* h, int64_t row0, int64_t rows) {
  if (rows < 0 || row0 < h->d.row_begin || row0 + rows > h->d.row_end)
    return fail(h, SMP_EINVAL, "rows [%lld, %lld) outside the handle's range [%lld, %lld)",
                (long long)row0, (long long)(row0 + rows), (long long)h->d.row_begin,
                (long long)h->d.row_end);
  return SMP_OK;
}

}  // namespace

extern "C" {

const char* smp_status_str(smp_status s) {
  switch (s) {
    case SMP_OK: return "SMP_OK";
    case SMP_EIO: return "SMP_EIO";
    case SMP_EINVAL: return "SMP_EINVAL";
    case SMP_ENUMERIC: return "SMP_ENUMERIC";
    case SMP_ECUDA: return "SMP_ECUDA";
    case SMP_ECAPACITY: return "SMP_ECAPACITY";
    case SMP_ENOMEM: return "SMP_ENOMEM";
  }
  return "SMP_UNKNOWN";
}

const char* smp_last_error(const smp_handle* h) { return h ? h->err.c_str() : "null handle"; }

int64_t smp_kernel_launches(const smp_handle* h) { return h ? h->launches : 0; }

smp_status smp_sketch_init(smp_handle** out, const smp_sketch_desc* d, void* stream) {
  NvtxRange nvtx_("smp_sketch_init");
  if (!out || !d) return SMP_EINVAL;
  *out = nullptr;
  if (d->k < 1 || d->k > 4096 || d->n1 < 1 || (!d->a_is_b && d->n2 < 1) || d->d_total < 1 ||
      d->row_begin < 0 || d->row_end > d->d_total || d->row_begin > d->row_end)
    return SMP_EINVAL;
  if (d->pi_kind < 0 || d->pi_kind > 3 || d->input < 0 || d->input > 2) return SMP_EINVAL;
  if (d->pi_kind == SMP_PI_SRHT && (int64_t)d->k > ((int64_t)1 << srht_L(d->d_total))) return SMP_EINVAL;
  if (d->pi_kind == SMP_PI_HADAMARD_TEST && (d->k != d->d_total || !is_pow2(d->d_total)))
    return SMP_EINVAL;
  if (d->n1 > (1ll << 31) - 1 || d->n2 > (1ll << 31) - 1) return SMP_EINVAL;
  smp_handle* h = new smp_handle();
  h->d = *d;
  h->st = reinterpret_cast<cudaStream_t>(stream);
  cudaGetDevice(&h->dev);
  {
    // WAltMin workspace comes from the device's default stream-ordered pool;
    // keep freed blocks cached instead of returning them at every sync
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, h->dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  h->n1 = d->n1;
  h->n2 = d->a_is_b ? d->n1 : d->n2;
  h->ntot = d->a_is_b ? d->n1 : d->n1 + d->n2;
  h->k = d->k;
  const int64_t nk = h->ntot * (int64_t)h->k;
  cudaError_t e = cudaSuccess;
  e = cudaMalloc(&h->acc_sk, nk * 4);
  if (e == cudaSuccess) e = cudaMalloc(&h->acc_nrm, h->ntot * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->fin_sk, nk * 4);
  if (e == cudaSuccess) e = cudaMalloc(&h->fin_sknorm, h->ntot * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->fin_D, h->ntot * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->FAFB, 2 * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->status, sizeof(int));
  if (e == cudaSuccess) e = cudaMalloc(&h->alpha, (h->n1 + h->n2) * 8);
  if (e == cudaSuccess) e = cudaMalloc(&h->d_total, 8);
  if (e == cudaSuccess) e = cudaMallocHost(&h->h_total, 8);
  if (e == cudaSuccess) e = cudaMallocHost(&h->h_status, sizeof(int));
  if (e == cudaSuccess) e = cudaMallocHost(&h->h_fafb, 16);
  if (e != cudaSuccess) {
    smp_destroy(h);
    return e == cudaErrorMemoryAllocation ? SMP_ENOMEM : SMP_ECUDA;
  }
  *out = h;
  return smp_sketch_reset(h);
}

smp_status smp_sketch_reset(smp_handle* h) {
  NvtxRange nvtx_("smp_sketch_reset");
  if (!h) return SMP_EINVAL;
  CK(h, cudaMemsetAsync(h->acc_sk, 0, h->ntot * (int64_t)h->k * 4, h->st), "memset");
  CK(h, cudaMemsetAsync(h->acc_nrm, 0, h->ntot * 8, h->st), "memset");
  CK(h, cudaMemsetAsync(h->status, 0, sizeof(int), h->st), "memset");
  h->finalized = false;
  return SMP_OK;
}

void smp_destroy(smp_handle* h) {
  if (!h) return;
  if (h->st) cudaStreamSynchronize(h->st);
  cudaFree(h->acc_sk); cudaFree(h->acc_nrm); cudaFree(h->part); cudaFree(h->pnorm); cudaFree(h->xchg);
  smp::mn_workspace_free(h->mn);
  cudaFree(h->lela_at); cudaFree(h->lela_bt); cudaFree(h->lela_pn);
  cudaFree(h->planes); cudaFree(h->pi_panel); cudaFree(h->fin_sk); cudaFree(h->fin_sknorm); cudaFree(h->fin_D);
  cudaFree(h->FAFB); cudaFree(h->status); cudaFree(h->pw_scratch); cudaFree(h->alpha);
  cudaFree(h->blk); cudaFree(h->d_total);
  smp::csr_workspace_free(h->csr);
  if (h->h_total) cudaFreeHost(h->h_total);
  if (h->h_status) cudaFreeHost(h->h_status);
  if (h->h_fafb) cudaFreeHost(h->h_fafb);
  for (int i = 0; i < 2; ++i) {
    if (h->stage[i]) cudaFree(h->stage[i]);
    if (h->ev_copied[i]) cudaEventDestroy(h->ev_copied[i]);
    if (h->ev_used[i]) cudaEventDestroy(h->ev_used[i]);
  }
  if (h->copy_st) cudaStreamDestroy(h->copy_st);
  if (h->aux_st) { cudaStreamSynchronize(h->aux_st); cudaStreamDestroy(h->aux_st); }
  for (int b = 0; b < 2; ++b) {
    cudaFree(h->planes2[b]); cudaFree(h->pnorm2[b]); cudaFree(h->panel2[b]);
    if (h->ev_prep[b]) cudaEventDestroy(h->ev_prep[b]);
    if (h->ev_free[b]) cudaEventDestroy(h->ev_free[b]);
  }
  if (h->ev_sync) cudaEventDestroy(h->ev_sync);
  for (auto e : h->ev_pool) cudaEventDestroy(e);
  delete h;
}

smp_status smp_sketch_block(smp_handle* h, int64_t row0, int64_t rows, const void* A, int64_t lda,
                            const void* B, int64_t ldb) {
  NvtxRange nvtx_("smp_sketch_block");
  if (!h) return SMP_EINVAL;
  smp_status s = check_rows(h, row0, rows);
  if (s != SMP_OK) return s;
  if (h->d.input == SMP_IN_CSR_F32)
    return fail(h, SMP_EINVAL, "CSR handle: use smp_sketch_block_csr");
  if (rows == 0) return SMP_OK;
  const bool two = !h->d.a_is_b;
  if (!A || lda < h->n1 || (two && (!B || ldb < h->n2)))
    return fail(h, SMP_EINVAL, "null pointer or leading dimension smaller than n");
  if (rows >= (1ll << 31)) return fail(h, SMP_EINVAL, "block of >= 2^31 rows");
  h->finalized = false;
  if (h->d.input == SMP_IN_DENSE_BF16) {
    auto aligned = [](const void* p, int64_t ld) {
      return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 8 == 0);
    };
    if ((reinterpret_cast<uintptr_t>(A) & 1) || (two && (reinterpret_cast<uintptr_t>(B) & 1)))
      return fail(h, SMP_EINVAL, "bf16 input must be 2-byte aligned");
    if (h->d.pi_kind == SMP_PI_GAUSSIAN) {
      s = sketch_dense_split(h, row0, rows, A, 1, lda, h->n1, 0);
      if (s != SMP_OK || !two) return s;
      return sketch_dense_split(h, row0, rows, B, 1, ldb, h->n2, h->n1);
    }
    s = aligned(A, lda) ? sketch_dense_bf16(h, row0, rows, A, lda, h->n1, 1, 0, true)
                        : sketch_dense_bf16_repack(h, row0, rows, A, lda, h->n1, 0);
    if (s != SMP_OK || !two) return s;
    return aligned(B, ldb) ? sketch_dense_bf16(h, row0, rows, B, ldb, h->n2, 1, h->n1, true)
                           : sketch_dense_bf16_repack(h, row0, rows, B, ldb, h->n2, h->n1);
  }
  // fp32
  if (reinterpret_cast<uintptr_t>(A) % 4 != 0 || (two && reinterpret_cast<uintptr_t>(B) % 4 != 0))
    return fail(h, SMP_EINVAL, "fp32 input must be 4-byte aligned");
  static const bool fused = [] {  // SMP_F32_FUSED=0: materialised planes (reference path)
    const char* e = getenv("SMP_F32_FUSED");
    return !(e && atoi(e) == 0);
  }();
  auto ok16 = [](const void* q, int64_t ld) { return reinterpret_cast<uintptr_t>(q) % 16 == 0 && ld % 4 == 0; };
  if (fused && ok16(A, lda) && (!two || ok16(B, ldb))) {
    s = sketch_dense_f32_fused(h, row0, rows, static_cast<const float*>(A), lda, h->n1, 0);
    if (s != SMP_OK || !two) return s;
    return sketch_dense_f32_fused(h, row0, rows, static_cast<const float*>(B), ldb, h->n2, h->n1);
  }
  s = sketch_dense_split(h, row0, rows, A, 0, lda, h->n1, 0);
  if (s != SMP_OK || !two) return s;
  return sketch_dense_split(h, row0, rows, B, 0, ldb, h->n2, h->n1);
}

smp_status smp_sketch_block_host(smp_handle* h, int64_t row0, int64_t rows, const void* A,
                                 int64_t lda, const void* B, int64_t ldb, int64_t chunk_rows) {
  NvtxRange nvtx_("smp_sketch_block_host");
  if (!h) return SMP_EINVAL;
  smp_status s = check_rows(h, row0, rows);
  if (s != SMP_OK) return s;
  if (h->d.input == SMP_IN_CSR_F32) return fail(h, SMP_EINVAL, "CSR handle: host path is dense only");
  const bool two = !h->d.a_is_b;
  if (!A || lda < h->n1 || (two && (!B || ldb < h->n2)))
    return fail(h, SMP_EINVAL, "null pointer or leading dimension smaller than n");
  const int64_t es = h->d.input == SMP_IN_DENSE_BF16 ? 2 : 4;
  // device copies are packed with ld rounded up to a multiple of 8 elements
  const int64_t lda_d = ((h->n1 + 7) / 8) * 8, ldb_d = two ? ((h->n2 + 7) / 8) * 8 : 0;
  const int64_t row_bytes = (lda_d + ldb_d) * es;
  if (chunk_rows <= 0) chunk_rows = std::max<int64_t>(64, ((256ll << 20) / row_bytes) / 64 * 64);
  const int64_t need = chunk_rows * row_bytes;
  if (need > h->stage_bytes) {
    for (int i = 0; i < 2; ++i) {
      if (h->stage[i]) cudaFree(h->stage[i]);
      h->stage[i] = nullptr;
      CK(h, cudaMalloc(&h->stage[i], need), "alloc staging");
    }
    h->stage_bytes = need;
  }
  if (!h->copy_st) {
    CK(h, cudaStreamCreateWithFlags(&h->copy_st, cudaStreamNonBlocking), "stream");
    for (int i = 0; i < 2; ++i) {
      CK(h, cudaEventCreateWithFlags(&h->ev_copied[i], cudaEventDisableTiming), "event");
      CK(h, cudaEventCreateWithFlags(&h->ev_used[i], cudaEventDisableTiming), "event");
      CK(h, cudaEventRecord(h->ev_used[i], h->st), "event");
    }
  }
  int buf = 0;
  for (int64_t r0 = 0; r0 < rows; r0 += chunk_rows, buf ^= 1) {
    const int64_t rc = std::min(chunk_rows, rows - r0);
    uint8_t* dA = static_cast<uint8_t*>(h->stage[buf]);
    uint8_t* dB = dA + rc * lda_d * es;
    CK(h, cudaStreamWaitEvent(h->copy_st, h->ev_used[buf], 0), "wait");
    CK(h, cudaMemcpy2DAsync(dA, lda_d * es, static_cast<const uint8_t*>(A) + r0 * lda * es, lda * es,
                            h->n1 * es, rc, cudaMemcpyHostToDevice, h->copy_st), "H2D A");
    if (two)
      CK(h, cudaMemcpy2DAsync(dB, ldb_d * es, static_cast<const uint8_t*>(B) + r0 * ldb * es,
                              ldb * es, h->n2 * es, rc, cudaMemcpyHostToDevice, h->copy_st), "H2D B");
    CK(h, cudaEventRecord(h->ev_copied[buf], h->copy_st), "event");
    CK(h, cudaStreamWaitEvent(h->st, h->ev_copied[buf], 0), "wait");
    s = smp_sketch_block(h, row0 + r0, rc, dA, lda_d, two ? dB : nullptr, ldb_d);
    if (s != SMP_OK) return s;
    CK(h, cudaEventRecord(h->ev_used[buf], h->st), "event");
  }
  CK(h, cudaStreamSynchronize(h->st), "sync");
  return SMP_OK;
}

smp_status smp_sketch_block_csr(smp_handle* h, int64_t row0, int64_t rows, const int64_t* a_rowptr,
                                const int32_t* a_col, const float* a_val, int64_t a_nnz,
                                const int64_t* b_rowptr, const int32_t* b_col, const float* b_val,
                                int64_t b_nnz) {
  NvtxRange nvtx_("smp_sketch_block_csr");
  if (!h) return SMP_EINVAL;
  smp_status s = check_rows(h, row0, rows);
  if (s != SMP_OK) return s;
  if (h->d.input != SMP_IN_CSR_F32) return fail(h, SMP_EINVAL, "handle is not a CSR handle");
  if (rows == 0) return SMP_OK;
  const bool two = !h->d.a_is_b;
  if (!a_rowptr || (a_nnz > 0 && (!a_col || !a_val)) ||
      (two && (!b_rowptr || (b_nnz > 0 && (!b_col || !b_val)))))
    return fail(h, SMP_EINVAL, "null CSR array");
  (void)a_nnz; (void)b_nnz;
  h->finalized = false;
  const int64_t l0 = h->csr.launches;
  h->csr.bounds_pre = false;
  h->csr.ev_pool = nullptr;
  h->csr.ev_used = &h->ev_used_n;
  // tensor-core head (K3): columns with density >= δ whose
  // nonzeros are small integers go through K1 as a dense bf16 matrix
  const double head_density = [] {  // read per call (tests switch it)
    const char* e = getenv("SMP_CSR_HEAD_DENSITY");
    return e ? atof(e) : 0.02;
  }();
  const int64_t a_n = h->n1, b_n = two ? h->n2 : 0;
  const uint16_t* lut = nullptr;
  if (head_density > 0.0) {
    int n_head = 0;
    CK(h, smp::csr_select_head(h->csr, a_rowptr, a_col, a_n, two ? b_rowptr : nullptr,
                               two ? b_col : nullptr, b_n, rows, head_density, &n_head, h->st),
       "csr head");
    if (n_head > 0) {
      // per head chunk: the tail K3 over the chunk's rows (which generates
      // each Π panel once and also transposes it into the κ-major head panel),
      // then K1 (PANEL) on the head chunk that the same pass densified
      lut = h->csr.head_lut;
      const int64_t ldh = ((n_head + 63) / 64) * 64;
      const int64_t kpad = ((h->k + 255) / 256) * 256;
      const int64_t rp = smp::csr_panel_rows(a_n + b_n);
      int64_t chunk = std::min<int64_t>(rows, (1ll << 30) / (ldh * 2));            // 1 GB dense chunk
      chunk = std::min<int64_t>(chunk, (512ll << 20) / (kpad * 2));                // 512 MB Π panel
      if (const char* e = getenv("SMP_CSR_HEAD_CHUNK")) chunk = std::min<int64_t>(chunk, atoll(e));  // tests
      chunk = std::max<int64_t>(rp, (chunk / rp) * rp);
      const int64_t cpad = ((std::min(chunk, rows) + 63) / 64) * 64;
      // SMP_CSR_HEAD_OVERLAP=1: the head K1 of a chunk on a side stream,
      // overlapped with the next chunk's tail (tensor cores + TMA vs L2
      // gathers + SIMT), double-buffered; default: serial on the main stream
      const bool ovl = [] {
        const char* e = getenv("SMP_CSR_HEAD_OVERLAP");
        return e ? atoi(e) != 0 : false;  // measured: no gain (K1 and the sort passes contend for SMs)
      }() && rows > chunk;
      uint16_t* xhb[2] = {nullptr, nullptr};
      uint16_t* kmb[2] = {nullptr, nullptr};
      CK(h, ensure(h->csr.xhead, h->csr.xhead_cap, cpad * ldh), "alloc head");
      CK(h, ensure(h->csr.kmaj, h->csr.kmaj_cap, kpad * cpad), "alloc head panel");
      xhb[0] = xhb[1] = h->csr.xhead;
      kmb[0] = kmb[1] = h->csr.kmaj;
      cudaStream_t side = h->st;
      if (ovl) {
        CK(h, ensure(h->csr.xhead1, h->csr.xhead1_cap, cpad * ldh), "alloc head");
        CK(h, ensure(h->csr.kmaj1, h->csr.kmaj1_cap, kpad * cpad), "alloc head panel");
        xhb[1] = h->csr.xhead1;
        kmb[1] = h->csr.kmaj1;
        if (!h->aux_st) CK(h, cudaStreamCreateWithFlags(&h->aux_st, cudaStreamNonBlocking), "stream");
        side = h->aux_st;
        for (int b = 0; b < 2; ++b) {
          if (!h->csr.ev_tail[b]) CK(h, cudaEventCreateWithFlags(&h->csr.ev_tail[b], cudaEventDisableTiming), "event");
          if (!h->csr.ev_head[b]) CK(h, cudaEventCreateWithFlags(&h->csr.ev_head[b], cudaEventDisableTiming), "event");
        }
        // the side stream starts after everything already queued on the main one
        CK(h, cudaEventRecord(h->csr.ev_tail[0], h->st), "event");
        CK(h, cudaStreamWaitEvent(side, h->csr.ev_tail[0], 0), "wait");
      }
      h->csr.ev_pool = h->timing ? &h->ev_pool : nullptr;
      CK(h, smp::csr_bounds(h->csr, a_rowptr, two ? b_rowptr : nullptr, a_n + b_n, rows, h->st), "bounds");
      // SMP_CSR_PROFILE=1: device time of the head's K1 + K2 (side stream)
      const char* hp = getenv("SMP_CSR_PROFILE");
      const bool hprof = hp && atoi(hp);
      std::vector<cudaEvent_t> hev;
      int c = 0;
      for (int64_t r0 = 0; r0 < rows; r0 += chunk, ++c) {
        const int b = ovl ? (c & 1) : 0;
        const int64_t rc = std::min(chunk, rows - r0);
        const int64_t ldk = ((rc + 63) / 64) * 64;
        // buffers b are free once the head K1 of chunk c - 2 has read them
        if (ovl && c >= 2) CK(h, cudaStreamWaitEvent(h->st, h->csr.ev_head[b], 0), "wait");
        if (rc != ldk) CK(h, cudaMemsetAsync(kmb[b], 0, kpad * ldk * 2, h->st), "memset");
        // the tail sort also densifies the head entries of these rows into xhb[b]
        cudaError_t e1 = smp::launch_sketch_csr(h->csr, pi_code(h), h->d.seed, h->k, row0 + r0, rc, a_rowptr,
                                                a_col, a_val, h->n1, two ? b_rowptr : nullptr,
                                                two ? b_col : nullptr, two ? b_val : nullptr, b_n,
                                                h->acc_sk, h->acc_nrm, h->status, h->st, lut, r0,
                                                kmb[b], ldk, (int)kpad, xhb[b], ldh, n_head);
        if (e1 != cudaSuccess) h->csr.bounds_pre = false;
        CK(h, e1, "sketch_csr");
        if (ovl) {
          CK(h, cudaEventRecord(h->csr.ev_tail[b], h->st), "event");
          CK(h, cudaStreamWaitEvent(side, h->csr.ev_tail[b], 0), "wait");
        }
        if (hprof) {
          hev.emplace_back();
          CK(h, cudaEventCreate(&hev.back()), "event");
          CK(h, cudaEventRecord(hev.back(), side), "event");
        }
        // K1 (PANEL) + K2 on the head chunk; K2 and the norm reduce add into
        // the head columns atomically (a tail entry with a non-4-bit value may
        // hit the same column concurrently)
        cudaStream_t main_st = h->st;
        h->st = side;
        smp_status s2 = sketch_dense_bf16(h, row0 + r0, rc, xhb[b], ldh, n_head, 1, 0, true, kmb[b],
                                          h->csr.head_map);
        h->st = main_st;
        if (s2 != SMP_OK) return s2;
        if (hprof) {
          hev.emplace_back();
          CK(h, cudaEventCreate(&hev.back()), "event");
          CK(h, cudaEventRecord(hev.back(), side), "event");
        }
        if (ovl) CK(h, cudaEventRecord(h->csr.ev_head[b], side), "event");
      }
      if (ovl) {  // the main stream continues after the last head K1
        CK(h, cudaEventRecord(h->csr.ev_head[0], side), "event");
        CK(h, cudaStreamWaitEvent(h->st, h->csr.ev_head[0], 0), "wait");
      }
      if (hprof) {
        float tot = 0.f;
        CK(h, cudaEventSynchronize(hev.back()), "sync");
        for (size_t i = 0; i + 1 < hev.size(); i += 2) {
          float ms = 0.f;
          cudaEventElapsedTime(&ms, hev[i], hev[i + 1]);
          tot += ms;
        }
        for (auto e : hev) cudaEventDestroy(e);
        fprintf(stderr, "K3 head over %lld rows (%d columns): K1+K2 %.3f ms (%s)\n", (long long)rows, n_head, tot,
                ovl ? "side stream, overlapped with the tail" : "serial");
      }
      h->csr.bounds_pre = false;
      h->launches += 2 + (h->csr.launches - l0);
      return SMP_OK;
    }
  }
  h->csr.ev_pool = h->timing ? &h->ev_pool : nullptr;
  cudaError_t e = smp::launch_sketch_csr(h->csr, pi_code(h), h->d.seed, h->k, row0, rows, a_rowptr,
                                         a_col, a_val, h->n1, two ? b_rowptr : nullptr,
                                         two ? b_col : nullptr, two ? b_val : nullptr,
                                         two ? h->n2 : 0, h->acc_sk, h->acc_nrm, h->status, h->st, lut);
  if (e == cudaErrorInvalidValue)
    return fail(h, SMP_EINVAL, "CSR: more than 2^26 columns are not supported");
  CK(h, e, "sketch_csr");
  h->launches += 2 + (h->csr.launches - l0);
  return SMP_OK;
}

// LELA pass 1: exact column norms only, accumulated into the same
// fp64 norm accumulators the sketch pass fills (no sketch).
smp_status smp_norms_block(smp_handle* h, int64_t row0, int64_t rows, const void* A, int64_t lda, const void* B,
                           int64_t ldb) {
  NvtxRange nvtx_("smp_norms_block");
  if (!h) return SMP_EINVAL;
  smp_status s = check_rows(h, row0, rows);
  if (s != SMP_OK) return s;
  if (h->d.input == SMP_IN_CSR_F32) return fail(h, SMP_EINVAL, "smp_norms_block: dense inputs only");
  if (rows == 0) return SMP_OK;
  const bool two = !h->d.a_is_b;
  if (!A || lda < h->n1 || (two && (!B || ldb < h->n2)))
    return fail(h, SMP_EINVAL, "null pointer or leading dimension smaller than n");
  const int bf = h->d.input == SMP_IN_DENSE_BF16 ? 1 : 0;
  h->finalized = false;
  for (int side = 0; side < (two ? 2 : 1); ++side) {
    const void* X = side ? B : A;
    const int64_t ld = side ? ldb : lda, n = side ? h->n2 : h->n1, off = side ? h->n1 : 0;
    const int64_t chunk = 1ll << 26;  // rows per launch (<= 65535 segments)
    for (int64_t r0 = 0; r0 < rows; r0 += chunk) {
      const int64_t rc = std::min(chunk, rows - r0);
      CK(h, ensure(h->lela_pn, h->lela_pn_cap, ((rc + 1023) / 1024) * n), "alloc");
      int segs = 0;
      CK(h, smp::launch_colnorms(static_cast<const uint8_t*>(X) + r0 * ld * (bf ? 2 : 4), bf, ld, rc, n,
                                 h->lela_pn, &segs, h->st), "colnorms");
      CK(h, smp::launch_reduce_norms(h->lela_pn, segs, n, h->acc_nrm + off, h->st), "reduce_norms");
      h->launches += 2;
    }
  }
  return SMP_OK;
}

// LELA pass 2: acc[s] += Σ_{t in block} A[t, I_s] B[t, J_s].
smp_status smp_exact_entries_block(smp_handle* h, int64_t row0, int64_t rows, const void* A, int64_t lda,
                                   const void* B, int64_t ldb, const int32_t* I, const int32_t* J,
                                   int64_t count, double* acc) {
  NvtxRange nvtx_("smp_exact_entries_block");
  if (!h) return SMP_EINVAL;
  smp_status s = check_rows(h, row0, rows);
  if (s != SMP_OK) return s;
  if (h->d.input == SMP_IN_CSR_F32) return fail(h, SMP_EINVAL, "smp_exact_entries_block: dense inputs only");
  if (count < 0 || (count > 0 && (!I || !J || !acc))) return fail(h, SMP_EINVAL, "bad sample arrays");
  if (rows == 0 || count == 0) return SMP_OK;
  const bool two = !h->d.a_is_b;
  if (!A || lda < h->n1 || (two && (!B || ldb < h->n2)))
    return fail(h, SMP_EINVAL, "null pointer or leading dimension smaller than n");
  const int bf = h->d.input == SMP_IN_DENSE_BF16 ? 1 : 0;
  const int64_t R = smp::lela_chunk_rows();
  CK(h, ensure(h->lela_at, h->lela_at_cap, h->n1 * R), "alloc");
  CK(h, ensure(h->lela_bt, h->lela_bt_cap, h->n2 * R), "alloc");
  CK(h, smp::launch_exact_entries(A, lda, two ? B : A, two ? ldb : lda, bf, rows, h->n1, h->n2, I, J, count, acc,
                                  h->lela_at, h->lela_bt, &h->launches, h->st), "exact_entries");
  return SMP_OK;
}

smp_status smp_set_timing(smp_handle* h, int32_t enable) {
  if (!h) return SMP_EINVAL;
  h->timing = enable != 0;
  return SMP_OK;
}

smp_status smp_kernel_timing(smp_handle* h, double* ms_total, int64_t* launches) {
  if (!h) return SMP_EINVAL;
  CK(h, cudaStreamSynchronize(h->st), "sync");
  double tot = 0.0;
  for (size_t i = 0; i + 1 < h->ev_used_n; i += 2) {
    float ms = 0.f;
    CK(h, cudaEventElapsedTime(&ms, h->ev_pool[i], h->ev_pool[i + 1]), "elapsed");
    tot += ms;
  }
  if (ms_total) *ms_total = tot;
  if (launches) *launches = (int64_t)(h->ev_used_n / 2);
  h->ev_used_n = 0;
  return SMP_OK;
}

smp_status smp_sketch_partials(smp_handle* h, float** sk, int64_t* sk_count, double** nrm,
                               int64_t* nrm_count) {
  if (!h) return SMP_EINVAL;
  if (sk) *sk = h->acc_sk;
  if (sk_count) *sk_count = h->ntot * (int64_t)h->k;
  if (nrm) *nrm = h->acc_nrm;
  if (nrm_count) *nrm_count = h->ntot;
  return SMP_OK;
}

smp_status smp_sketch_pack_partials(smp_handle* h, double** buf, int64_t* count) {
  NvtxRange nvtx_("smp_sketch_pack_partials");
  if (!h || !buf || !count) return SMP_EINVAL;
  const int64_t nsk = h->ntot * (int64_t)h->k, nn = h->ntot;
  CK(h, ensure(h->xchg, h->xchg_cap, nsk + nn), "alloc exchange");
  CK(h, smp::launch_pack_partials(h->acc_sk, nsk, h->acc_nrm, nn, h->xchg, h->st), "pack partials");
  h->launches += 1;
  *buf = h->xchg;
  *count = nsk + nn;
  return SMP_OK;
}

smp_status smp_sketch_unpack_partials(smp_handle* h) {
  NvtxRange nvtx_("smp_sketch_unpack_partials");
  if (!h) return SMP_EINVAL;
  const int64_t nsk = h->ntot * (int64_t)h->k, nn = h->ntot;
  if (!h->xchg || h->xchg_cap < nsk + nn) return fail(h, SMP_EINVAL, "call smp_sketch_pack_partials first");
  CK(h, smp::launch_unpack_partials(h->xchg, nsk, nn, h->acc_sk, h->acc_nrm, h->st), "unpack partials");
  h->launches += 1;
  h->finalized = false;
  return SMP_OK;
}

smp_status smp_finalize_norms(smp_handle* h, float* A_sk, float* B_sk, double* a_norm2,
                              double* b_norm2, double* frob2, float* a_sknorm, float* b_sknorm) {
  NvtxRange nvtx_("smp_finalize_norms");
  using namespace smp;
  if (!h) return SMP_EINVAL;
  const int k = h->k;
  const float scale = (float)(1.0 / std::sqrt((double)k));
  // h->status is cleared by smp_sketch_reset (it also carries the CSR
  // out-of-range-column bit set during the pass)
  CK(h, launch_finalize(h->acc_sk, h->acc_nrm, h->ntot, k, scale, h->fin_sk, h->fin_sknorm,
                        h->fin_D, h->status, h->st), "finalize");
  int64_t p2 = 1;
  while (p2 < std::max(h->n1, h->n2)) p2 <<= 1;
  CK(h, ensure(h->pw_scratch, h->pw_cap, 2 * p2), "alloc");
  CK(h, launch_pairwise_sum(h->acc_nrm, h->n1, h->pw_scratch, h->FAFB, h->st), "pairwise");
  CK(h, launch_pairwise_sum(h->acc_nrm + (h->d.a_is_b ? 0 : h->n1), h->n2, h->pw_scratch,
                            h->FAFB + 1, h->st), "pairwise");
  h->launches += 3;
  const int64_t boff = h->d.a_is_b ? 0 : h->n1;
  if (A_sk) CK(h, cudaMemcpyAsync(A_sk, h->fin_sk, h->n1 * k * 4, cudaMemcpyDeviceToDevice, h->st), "copy");
  if (B_sk) CK(h, cudaMemcpyAsync(B_sk, h->fin_sk + boff * k, h->n2 * k * 4, cudaMemcpyDeviceToDevice, h->st), "copy");
  if (a_norm2) CK(h, cudaMemcpyAsync(a_norm2, h->acc_nrm, h->n1 * 8, cudaMemcpyDeviceToDevice, h->st), "copy");
  if (b_norm2) CK(h, cudaMemcpyAsync(b_norm2, h->acc_nrm + boff, h->n2 * 8, cudaMemcpyDeviceToDevice, h->st), "copy");
  if (frob2) CK(h, cudaMemcpyAsync(frob2, h->FAFB, 16, cudaMemcpyDeviceToDevice, h->st), "copy");
  if (a_sknorm || b_sknorm) {
    // fp64 -> fp32 conversion of ||Ã_i||
    if (a_sknorm) CK(h, smp_convert_f64_f32(h->fin_sknorm, h->n1, a_sknorm, h->st), "convert");
    if (b_sknorm) CK(h, smp_convert_f64_f32(h->fin_sknorm + boff, h->n2, b_sknorm, h->st), "convert");
  }
  CK(h, cudaMemcpyAsync(h->h_status, h->status, sizeof(int), cudaMemcpyDeviceToHost, h->st), "copy");
  CK(h, cudaMemcpyAsync(h->h_fafb, h->FAFB, 16, cudaMemcpyDeviceToHost, h->st), "copy");
  CK(h, cudaStreamSynchronize(h->st), "sync");
  // the finalized state is usable by sample_estimate / waltmin only when every
  // check passes (a zero Frobenius norm would divide by zero in q̂)
  h->finalized = false;
  if (*h->h_status & 2) return fail(h, SMP_EINVAL, "CSR column index out of range (S:123)");
  if (*h->h_status) return fail(h, SMP_ENUMERIC, "NaN/Inf in the column norms or sketch");
  if (!(h->h_fafb[0] > 0.0) || !(h->h_fafb[1] > 0.0))
    return fail(h, SMP_ENUMERIC, "||A||_F = 0 or ||B||_F = 0");
  h->finalized = true;
  return SMP_OK;
}

static smp_status sample_multinomial(smp_handle* h, double m, uint64_t seed, int32_t est, int64_t cap,
                                     int32_t* I, int32_t* J, float* val, double* qhat, int64_t* count) {
  using namespace smp;
  const int64_t n1 = h->n1, n2 = h->n2;
  const int64_t boff = h->d.a_is_b ? 0 : n1;
  double* beta = h->alpha + n1;
  CK(h, launch_alpha_beta(h->acc_nrm, n1, h->acc_nrm + boff, n2, h->FAFB, h->alpha, beta, h->st), "alpha_beta");
  h->launches += 1;
  int64_t cnt = 0;
  cudaError_t e = run_sample_multinomial(h->mn, h->alpha, beta, n1, n2, m, seed, cap, I, J, qhat, &cnt,
                                         &h->launches, h->st);
  if (e == cudaErrorInvalidValue) return fail(h, SMP_EINVAL, "multinomial sampler: >= 2^31 entries");
  CK(h, e, "multinomial sampler");
  if (count) *count = cnt;
  if (cnt > cap) return fail(h, SMP_ECAPACITY, "|Omega| = %lld > cap = %lld", (long long)cnt, (long long)cap);
  if (cnt == 0) return SMP_OK;
  CK(h, launch_sddmm(h->fin_sk, h->fin_sk + boff * h->k, h->fin_D, h->fin_D + boff, h->k, I, J,
                     h->mn.total, cap, est == SMP_EST_PLAIN, val, h->st), "sddmm");
  h->launches += 1;
  CK(h, cudaStreamSynchronize(h->st), "sync");
  return SMP_OK;
}

smp_status smp_sample_estimate_ex(smp_handle* h, double m, uint64_t seed, int32_t est, int32_t sampler,
                                  int64_t cap, int32_t* I, int32_t* J, float* val, double* qhat,
                                  int64_t* count) {
  NvtxRange nvtx_("smp_sample_estimate_ex");
  if (!h) return SMP_EINVAL;
  if (sampler == SMP_SAMPLER_BERNOULLI) return smp_sample_estimate(h, m, seed, est, cap, I, J, val, qhat, count);
  if (sampler != SMP_SAMPLER_MULTINOMIAL) return fail(h, SMP_EINVAL, "unknown sampler");
  if (!(m > 0.0)) return fail(h, SMP_EINVAL, "m must be > 0");
  if (!h->finalized) return fail(h, SMP_EINVAL, "call smp_finalize_norms first");
  if (cap < 0 || (cap > 0 && (!I || !J || !val || !qhat))) return fail(h, SMP_EINVAL, "bad output");
  return sample_multinomial(h, m, seed, est, cap, I, J, val, qhat, count);
}

smp_status smp_sample_estimate(smp_handle* h, double m, uint64_t seed, int32_t est, int64_t cap,
                               int32_t* I, int32_t* J, float* val, double* qhat, int64_t* count) {
  NvtxRange nvtx_("smp_sample_estimate");
  using namespace smp;
  if (!h) return SMP_EINVAL;
  if (!(m > 0.0)) return fail(h, SMP_EINVAL, "m must be > 0");
  if (!h->finalized) return fail(h, SMP_EINVAL, "call smp_finalize_norms first");
  if (cap < 0 || (cap > 0 && (!I || !J || !val || !qhat))) return fail(h, SMP_EINVAL, "bad output");
  const int64_t n1 = h->n1, n2 = h->n2;
  if (n1 * n2 > (1ll << 40)) return fail(h, SMP_EINVAL, "n1*n2 too large for the Bernoulli sweep");
  const int64_t boff = h->d.a_is_b ? 0 : n1;
  double* beta = h->alpha + n1;
  CK(h, launch_alpha_beta(h->acc_nrm, n1, h->acc_nrm + boff, n2, h->FAFB, h->alpha, beta, h->st), "alpha_beta");
  const int64_t nb = omega_num_blocks(n1, n2);
  CK(h, ensure(h->blk, h->blk_cap, std::max<int64_t>(nb, 1)), "alloc");
  CK(h, launch_omega_count(h->alpha, beta, n1, n2, m, seed, h->blk, h->st), "omega_count");
  CK(h, launch_scan_counts(h->blk, nb, h->d_total, h->st), "scan");
  CK(h, launch_omega_write(h->alpha, beta, n1, n2, m, seed, h->blk, h->d_total, cap, I, J, qhat, h->st), "omega_write");
  if (cap > 0)
    CK(h, launch_sddmm(h->fin_sk, h->fin_sk + boff * h->k, h->fin_D, h->fin_D + boff, h->k, I, J,
                       h->d_total, cap, est == SMP_EST_PLAIN, val, h->st), "sddmm");
  h->launches += 5;
  CK(h, cudaMemcpyAsync(h->h_total, h->d_total, 8, cudaMemcpyDeviceToHost, h->st), "copy");
  CK(h, cudaStreamSynchronize(h->st), "sync");
  if (count) *count = *h->h_total;
  if (*h->h_total > cap)
    return fail(h, SMP_ECAPACITY, "|Omega| = %lld > cap = %lld", (long long)*h->h_total, (long long)cap);
  return SMP_OK;
}

smp_status smp_waltmin(smp_handle* h, const int32_t* I, const int32_t* J, const float* val,
                       const double* qhat, int64_t count, const smp_waltmin_desc* w, float* U,
                       float* V) {
  NvtxRange nvtx_("smp_waltmin");
  if (!h || !w) return SMP_EINVAL;
  if (!h->finalized) return fail(h, SMP_EINVAL, "call smp_finalize_norms first");
  if (w->r < 1 || w->r > 16 || w->r > h->n1 || w->r > h->n2)
    return fail(h, SMP_EINVAL, "r must satisfy 1 <= r <= min(16, n1, n2)");
  if (w->T < 1) return fail(h, SMP_EINVAL, "T must be >= 1");
  if (w->init_iters < 1) return fail(h, SMP_EINVAL, "init_iters must be >= 1");
  if (w->partition != SMP_PART_REUSE_ALL && w->partition != SMP_PART_FRESH_2T1)
    return fail(h, SMP_EINVAL, "unknown partition");
  if (w->partition == SMP_PART_FRESH_2T1 && count < 2 * (int64_t)w->T + 1)
    return fail(h, SMP_EINVAL, "FRESH_2T1 needs |Omega| >= 2T+1 (Alg. 2 line 3)");
  if (count < 0 || count > (1ll << 31) - 1 || (count > 0 && (!I || !J || !val || !qhat)) || !U || !V)
    return fail(h, SMP_EINVAL, "bad sample arrays");
  smp::WaltminArgs a{};
  a.n1 = h->n1; a.n2 = h->n2; a.count = count;
  a.r = w->r; a.T = w->T; a.init_iters = w->init_iters; a.partition = w->partition;
  a.trim_c = w->trim_c; a.lam = w->ridge; a.seed = w->seed;
  a.I = I; a.J = J; a.val = val; a.qhat = qhat;
  a.a_norm2 = h->acc_nrm; a.FA = h->FAFB;
  a.U = U; a.V = V;
  CK(h, smp::run_waltmin(a, h->st), "waltmin");
  h->launches += 10;  // CSR/CSC setup (weights, pointers, CUB radix sort, gather) + one persistent kernel
  CK(h, cudaStreamSynchronize(h->st), "sync");
  return SMP_OK;
}

}  // extern "C"

// small helper kernel (fp64 -> fp32)
__global__ void smp_f64_to_f32_kernel(const double* __restrict__ x, int64_t n, float* __restrict__ y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (float)x[i];
}
cudaError_t smp_convert_f64_f32(const double* x, int64_t n, float* y, cudaStream_t st) {
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 1024);
  if (blocks < 1) blocks = 1;
  smp_f64_to_f32_kernel<<<blocks, 256, 0, st>>>(x, n, y);
  return cudaGetLastError();
}
