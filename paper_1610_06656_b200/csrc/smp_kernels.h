// Internal launcher declarations for the SMP-PCA sm_100a kernels (not part
// of the public C ABI; see include/smp.h for that).
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

namespace smp {

// ---- K1 dense sketch (sketch_tc.cu)
struct SketchTCParams {
  int64_t rows;      // local rows of this block (TMA tensor height)
  int64_t row0;      // global row index of local row 0
  int32_t n;         // columns (TMA tensor width)
  int32_t k;         // sketch size
  int32_t n_tiles, k_tiles, splits;
  int32_t kb_total;  // ceil(rows / 64)
  int32_t kind;      // PI_*
  int32_t do_norms;
  int32_t debug;     // tuning experiments only (SMP_K1_DEBUG): 1 skip norms, 2 skip Π gen, 4 skip MMA
  uint32_t backoff_ns;  // K1: __nanosleep between barrier tests of the off-critical-path waiters (0 = spin)
  uint64_t seed;
  float* part;       // [splits][n][k]
  double* pnorm;     // [splits * k_tiles][n]
  const uint16_t* pi_panel;  // optional κ-major Π panel [k][pi_ld] for rows row0.. (else generated in-kernel)
  int64_t pi_ld;             // multiple of 64 rows, >= kb_total * 64
};
// Π(κ, t) for t in [t0, t0 + rows) into panel[κ * ld + t - t0] (bf16 bits; rows padded by the caller)
cudaError_t launch_pi_panel_kmajor(int kind, uint64_t seed, int k, int kpad, int64_t t0, int64_t rows,
                                   int64_t ld, uint16_t* panel, cudaStream_t st, int blocks_per_sm = 16);
cudaError_t launch_sketch_tc(const void* X, int64_t ldx, SketchTCParams p, cudaStream_t st);
int sketch_tc_smem_bytes();
// K1F (sketch_tc_f32.cu): fp32 X with the bf16 plane split fused in; Π from
// p.pi_panel (required); mode 3 (±1 Π, 8+8+8 bits) or 4 (Gaussian, 4+8+8);
// p.n = input columns, p.n_tiles = ceil(n / 128); part = [splits][3 n][k].
cudaError_t launch_sketch_tc_f32(const float* X, int64_t ldx, SketchTCParams p, int mode, cudaStream_t st);

// ---- combine exchange (reduce.cu): [sk (fp32 -> fp64) | nrm] in one fp64 buffer, and back
cudaError_t launch_pack_partials(const float* sk, int64_t nsk, const double* nrm, int64_t nn, double* out,
                                 cudaStream_t st);
cudaError_t launch_unpack_partials(const double* in, int64_t nsk, int64_t nn, float* sk, double* nrm,
                                   cudaStream_t st);

// ---- K2 partial reduce, fp32 split, K4 finalize (reduce.cu)
// acc[c][κ] += Σ_s Σ_pl part[s][pl*n + c][κ]   (planes pl = 0..planes-1)
// map (optional): output column of input column c is map[c] (acc is then the
// base of the whole [n_tot][k] accumulator)
cudaError_t launch_reduce_sketch(const float* part, int splits, int planes, int64_t n, int k,
                                 float* acc, cudaStream_t st, const int32_t* map = nullptr);
// nacc[c] += Σ_slot pnorm[slot][c]
cudaError_t launch_reduce_norms(const double* pnorm, int slots, int64_t n, double* nacc,
                                cudaStream_t st, const int32_t* map = nullptr);
// rows of X (fp32, or bf16 if x_bf16) -> P exact bf16 planes (mode 3: fp32
// 8+8+8 bits; mode 4: fp32 4+8+8+4; mode 2: bf16 4+4) laid out as a
// rows x (P n) matrix with leading dimension ldp, and fp64 Σx² per row segment.
cudaError_t launch_split_planes(const void* X, int x_bf16, int64_t ldx, int64_t rows, int64_t n,
                                int mode, uint16_t* planes, int64_t ldp, double* pnorm, int seg_rows,
                                cudaStream_t st);
// finalize one matrix: out = acc * scale (fp32), sknorm (fp64), D (fp64)
cudaError_t launch_finalize(const float* acc, double* nacc, int64_t n, int k, float scale,
                            float* out, double* sknorm, double* D, int* status, cudaStream_t st);
// fixed pairwise tree sum (R5) of x[0..n) into *out (single block)
cudaError_t launch_pairwise_sum(const double* x, int64_t n, double* scratch, double* out,
                                cudaStream_t st);

// ---- K3 sparse sketch (sketch_csr.cu): handle-owned workspace
struct CsrWorkspace {
  uint16_t* pi = nullptr;         // Π panel, Rp x kp bf16
  int64_t pi_cap = 0;
  uint64_t* kv_in = nullptr;      // packed (key << 32 | value bits) per tail nonzero
  uint64_t* kv_out = nullptr;     // ... sorted by key (K3d input)
  int64_t ent_cap_ki = 0, ent_cap_ko = 0;
  uint8_t* cub_tmp = nullptr;
  int64_t cub_cap = 0;
  uint32_t* hist = nullptr;       // counting sort: (panel, column, slice) counts, then starts
  uint32_t* offs = nullptr;
  int64_t hist_cap = 0, offs_cap = 0;
  uint32_t* ne_dev = nullptr;     // [0] tail entries of the panel, [1] head columns
  int64_t ne_cap = 0;
  // tensor-core head (columns with density >= SMP_CSR_HEAD_DENSITY)
  uint16_t* head_lut = nullptr;   // [ntot] slot or 0xFFFF (tail column)
  int32_t* head_map = nullptr;    // [slots] global column
  uint32_t* head_cnt = nullptr;
  uint32_t* head_flag = nullptr;  // [2 ntot]: flags, scan
  uint8_t* head_tmp = nullptr;
  int64_t head_lut_cap = 0, head_map_cap = 0, head_cnt_cap = 0, head_flag_cap = 0, head_tmp_cap = 0;
  uint16_t* xhead = nullptr;      // dense head chunk (bf16)
  int64_t xhead_cap = 0;
  uint16_t* kmaj = nullptr;       // κ-major Π of the head chunk (transposed K3 panels)
  int64_t kmaj_cap = 0;
  uint16_t* xhead1 = nullptr;     // second buffers: the head K1 of chunk c runs on a side
  int64_t xhead1_cap = 0;         // stream while the tail of chunk c + 1 fills these
  uint16_t* kmaj1 = nullptr;
  int64_t kmaj1_cap = 0;
  cudaEvent_t ev_tail[2] = {nullptr, nullptr}, ev_head[2] = {nullptr, nullptr};
  int64_t* head_h = nullptr;      // pinned

  int64_t* bounds_d = nullptr;
  int64_t bounds_cap = 0;
  int64_t* bounds_h = nullptr;    // pinned
  int64_t bounds_hcap = 0;
  bool bounds_pre = false;        // bounds_h holds the whole block's panel boundaries
  int64_t bounds_npan = 0;
  int bounds_rp = 0;
  int64_t launches = 0;           // kernels launched (counter for the bench)
  // timing of the dominant kernel (K3d) with CUDA events on the launching
  // stream: pairs appended to *ev_pool from index *ev_used (null: off)
  std::vector<cudaEvent_t>* ev_pool = nullptr;
  size_t* ev_used = nullptr;
};
// rows [row0, row0 + rows) of A (and B) in CSR (rowptr relative to any base:
// col/val are indexed from rowptr[0]) -> acc_sk[c][κ] += Σ v Π(κ, t),
// acc_nrm[c] += Σ v² for columns c of A (0..a_n) then B (a_n..a_n+b_n).
// Out-of-range columns set bit 2 of *status.  Synchronises once per call
// (panel entry counts are read back to size the sort).
cudaError_t launch_sketch_csr(CsrWorkspace& w, int kind, uint64_t seed, int k, int64_t row0,
                              int64_t rows, const int64_t* a_rowptr, const int32_t* a_col,
                              const float* a_val, int64_t a_n, const int64_t* b_rowptr,
                              const int32_t* b_col, const float* b_val, int64_t b_n, float* acc_sk,
                              double* acc_nrm, int* status, cudaStream_t st,
                              const uint16_t* head_lut = nullptr, int64_t rbase = 0,
                              uint16_t* kmaj = nullptr, int64_t kmaj_ld = 0, int kpad = 0,
                              uint16_t* xh = nullptr, int64_t ldh = 0, int n_head = 0);
// (rbase: the call covers rowptr rows [rbase, rbase + rows) of the block,
// global row0 = the global row of rowptr row rbase; kmaj: also write each
// generated Π panel into kmaj[κ][t - row0] (ld kmaj_ld, kpad κ rows) for K1;
// xh: the head entries (head_lut) of row t - row0 go to xh[(t - row0) * ldh +
// slot] as bf16, slots [0, n_head) of every row zeroed first — the dense head
// chunk K1 reads, built by the same pass that sorts the tail)
void csr_workspace_free(CsrWorkspace& w);
int csr_panel_rows(int64_t ntot);  // rows of one K3 Π panel (2^15 for up to 2^17 columns)
// read back every panel's entry boundaries for rows [0, rows) of the block
// once (one sync) so that per-chunk launch_sketch_csr calls need none
cudaError_t csr_bounds(CsrWorkspace& w, const int64_t* a_rowptr, const int64_t* b_rowptr, int64_t ntot,
                       int64_t rows, cudaStream_t st);
// head columns: count nonzeros per column over the block (over 64 evenly
// spaced segments of 4096 rows when the block is longer), select columns with
// count >= density * counted rows (slots in column order) -> w.head_lut / w.head_map;
// *n_head = number of slots (synchronises)
cudaError_t csr_select_head(CsrWorkspace& w, const int64_t* a_rowptr, const int32_t* a_col, int64_t a_n,
                            const int64_t* b_rowptr, const int32_t* b_col, int64_t b_n, int64_t rows,
                            double density, int* n_head, cudaStream_t st);

// ---- K5/K6 sampling and estimation (omega.cu)
cudaError_t launch_alpha_beta(const double* a2, int64_t n1, const double* b2, int64_t n2,
                              const double* FAFB, double* alpha, double* beta, cudaStream_t st);
int64_t omega_num_blocks(int64_t n1, int64_t n2);
cudaError_t launch_omega_count(const double* alpha, const double* beta, int64_t n1, int64_t n2,
                               double m, uint64_t seed, int64_t* blk_counts, cudaStream_t st);
cudaError_t launch_scan_counts(int64_t* blk_counts, int64_t nblk, int64_t* total, cudaStream_t st);
cudaError_t launch_omega_write(const double* alpha, const double* beta, int64_t n1, int64_t n2,
                               double m, uint64_t seed, const int64_t* blk_offsets,
                               const int64_t* total, int64_t cap, int32_t* I, int32_t* J,
                               double* qhat, cudaStream_t st);
cudaError_t launch_sddmm(const float* Ask, const float* Bsk, const double* DA, const double* DB,
                         int k, const int32_t* I, const int32_t* J, const int64_t* total,
                         int64_t cap, int plain, float* val, cudaStream_t st);

// row-multinomial Ω (R27, omega.cu): handle-owned scratch
struct MnWorkspace {
  int32_t* sig = nullptr; int64_t sig_cap = 0;        // σ (columns by β descending)
  int32_t* iota = nullptr; int64_t iota_cap = 0;
  double* bsorted = nullptr; int64_t bsorted_cap = 0; // β_σ
  double* bp = nullptr; int64_t bp_cap = 0;           // sequential prefix of β_σ
  int64_t* sat = nullptr; int64_t sat_cap = 0;        // s_i
  double* Tr = nullptr; int64_t Tr_cap = 0;           // T_i
  int64_t* offs = nullptr; int64_t offs_cap = 0;      // row entry offsets (n1 + 1)
  int32_t* jtmp = nullptr; int64_t jtmp_cap = 0;      // saturated + drawn columns
  int32_t* jsrt = nullptr; int64_t jsrt_cap = 0;      // sorted per row
  int32_t* flag = nullptr; int64_t flag_cap = 0;      // first occurrence
  int32_t* pos = nullptr; int64_t pos_cap = 0;        // output position
  uint8_t* tmp = nullptr; int64_t tmp_cap = 0;        // CUB scratch
  int64_t* total = nullptr;
  int64_t* total_h = nullptr;                         // pinned
};
void mn_workspace_free(MnWorkspace& w);
// Ω (sorted by (i, j)) with q̂; *count = |Ω| (written even when > cap, in
// which case nothing is written).  Synchronises twice.
cudaError_t run_sample_multinomial(MnWorkspace& w, const double* alpha, const double* beta, int64_t n1,
                                   int64_t n2, double m, uint64_t seed, int64_t cap, int32_t* I, int32_t* J,
                                   double* qhat, int64_t* count, int64_t* launches, cudaStream_t st);

// ---- LELA (lela.cu): pass 1 column norms, pass 2 exact entries on Ω
// pnorm[seg][c] = Σ_{t in seg} X[t, c]² (fp64, NORM_SEG-row segments; *segs set)
cudaError_t launch_colnorms(const void* X, int x_bf16, int64_t ldx, int64_t rows, int64_t n, double* pnorm,
                            int* segs, cudaStream_t st);
// acc[s] += Σ_{t < rows} A[t, I_s] B[t, J_s]; At / Bt: scratch of n1 · R / n2 · R
// floats (R = lela_chunk_rows())
cudaError_t launch_exact_entries(const void* A, int64_t lda, const void* B, int64_t ldb, int x_bf16,
                                 int64_t rows, int64_t n1, int64_t n2, const int32_t* I, const int32_t* J,
                                 int64_t cnt, double* acc, float* At, float* Bt, int64_t* launches,
                                 cudaStream_t st);
int lela_chunk_rows();

// ---- K7-K9 WAltMin (waltmin.cu)
struct WaltminArgs {
  int64_t n1, n2, count;
  int r, T, init_iters;
  int partition;          // 0 REUSE_ALL, 1 FRESH_2T1 (Alg. 2 line 3; R11)
  double trim_c, lam;
  uint64_t seed;
  const int32_t* I;
  const int32_t* J;
  const float* val;
  const double* qhat;
  const double* a_norm2;  // n1, device
  const double* FA;       // device scalar
  float* U;
  float* V;
};
// returns a cudaError_t; workspace is allocated internally from the stream's
// pool (cudaMallocAsync) and freed before return.
cudaError_t run_waltmin(const WaltminArgs& a, cudaStream_t st);

}  // namespace smp
