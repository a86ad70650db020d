/*
 * smp.h — C ABI of libsmp.so, the B200 (sm_100a) hot path of SMP-PCA
 * (Streaming Matrix Product PCA, arXiv 1610.06656).
 *
 * Citation convention: "P:L" = /root/reference/PAPER.md line L.  The problem
 * statement: A ∈ R^{d×n1}, B ∈ R^{d×n2} stored out of core; find a
 * rank-r approximation of AᵀB.  Alg. 1 takes r, k, m, T.
 *
 * Layout conventions (all calls):
 *   - Dense inputs are ROW-MAJOR d×n (one row per observation t, i.e. the
 *     rows of A that a stream delivers), leading dimension in ELEMENTS.
 *   - Sketch outputs are n×k row-major: row i is the sketched column
 *     Ã_i = Π A_i ∈ R^k, contiguous (what Eq. 2's dot products read).
 *   - Every array pointer is a DEVICE pointer owned by the caller unless the
 *     function name ends in _host; the library never frees caller memory.
 *   - Work is enqueued on the stream given to smp_sketch_init; calls return
 *     before the GPU finishes except where "synchronises" is stated.
 *   - Validation errors are returned synchronously, before anything is
 *     enqueued; the handle's last-error string says why.
 *   - Status codes mirror the error classes of the spec (IO=2, validation=3,
 *     numerical=4) plus CUDA=5, capacity=6, out-of-memory=7.
 */
#ifndef SMP_H_
#define SMP_H_

#include <stdint.h>

#if defined(__GNUC__)
#define SMP_API __attribute__((visibility("default")))
#else
#define SMP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SMP_OK = 0,
  SMP_EIO = 2,
  SMP_EINVAL = 3,      /* invalid argument / out-of-range rows / bad layout */
  SMP_ENUMERIC = 4,    /* ||A||_F = 0, ||B||_F = 0, or NaN/Inf seen        */
  SMP_ECUDA = 5,       /* CUDA runtime / driver error                       */
  SMP_ECAPACITY = 6,   /* |Ω| > cap: *count holds the size, call again      */
  SMP_ENOMEM = 7
} smp_status;

/* Π, Alg. 1 line 2: N(0,1/k) entries; P:63 admits any oblivious
 * subspace embedding.  Π is never stored: entries are regenerated from the
 * Philox4x32-10 hash of (seed, κ, global row t).
 * HADAMARD_TEST: Π(κ,t) = (-1)^popcount(κ&t)/sqrt(k), requires k = d_total a
 * power of two (then Π is orthonormal and M̃ = AᵀB exactly). */
/* Π kinds (R1, R26): Rademacher ±1, Gaussian bf16(Box–Muller),
 * the Sylvester-Hadamard test matrix (k = d, d a power of 2), and SRHT
 * (√(d/k)·S·H·D — the sketch of the paper's Spark code; H of order
 * 2^⌈log2 d_total⌉, k distinct rows; requires k <= that order). */
typedef enum {
  SMP_PI_RADEMACHER = 0,
  SMP_PI_GAUSSIAN = 1,
  SMP_PI_HADAMARD_TEST = 2,
  SMP_PI_SRHT = 3
} smp_pi;

typedef enum {
  SMP_IN_DENSE_BF16 = 0, /* bf16, 16-byte aligned base, ld % 8 == 0 (TMA)     */
  SMP_IN_DENSE_F32 = 1,  /* fp32, any alignment of 4; split into 3 bf16 terms */
  SMP_IN_CSR_F32 = 2     /* CSR rows (bag-of-words, P:9), fp32 values          */
} smp_input;

typedef enum { SMP_EST_RESCALED = 0, SMP_EST_PLAIN = 1 } smp_est;

typedef struct {
  int64_t d_total;   /* total number of rows d (all shards)                  */
  int64_t n1, n2;    /* columns of A and B (n2 ignored if a_is_b)            */
  int32_t k;         /* sketch size, 1 <= k <= 4096                           */
  int32_t pi_kind;   /* smp_pi                                                */
  uint64_t seed;     /* Π seed                                               */
  int32_t a_is_b;    /* PCA special case A = B (P:9, Remark 3 P:136)          */
  int32_t input;     /* smp_input                                             */
  int64_t row_begin; /* rows this handle may receive: [row_begin, row_end)   */
  int64_t row_end;   /* (row sharding across GPUs)             */
} smp_sketch_desc;

typedef struct smp_handle smp_handle;

/* Allocate the handle-owned workspace (fp32 sketch accumulators k×(n1+n2),
 * fp64 norm accumulators, split-K partials) on the current CUDA device and
 * zero it.  stream is a cudaStream_t (NULL = legacy default stream).
 * Errors: SMP_EINVAL (k<1 or k>4096, n<1, d<1, bad row range, HADAMARD_TEST
 * with k != d or d not a power of 2, unknown enums), SMP_ENOMEM, SMP_ECUDA. */
SMP_API smp_status smp_sketch_init(smp_handle** h, const smp_sketch_desc* desc, void* stream);

/* Step 1, the one pass: accumulate rows [row0, row0+rows) of A
 * and B into Ã = ΠA, B̃ = ΠB and the exact column norms² (fp64).  Blocks may
 * arrive in any order and must not repeat a row (not checked).  B is
 * ignored when a_is_b.  A/B: device pointers to the block's first row,
 * layout per desc.input.  Errors: SMP_EINVAL (rows outside
 * [row_begin,row_end), lda < n1, ldb < n2, misaligned bf16 pointer/ld,
 * CSR handle), SMP_ECUDA. */
SMP_API smp_status smp_sketch_block(smp_handle* h, int64_t row0, int64_t rows, const void* A, int64_t lda,
                            const void* B, int64_t ldb);

/* Same as smp_sketch_block for HOST (pageable or pinned) buffers: the
 * library streams the rows through its own double-buffered device staging
 * area in chunks of chunk_rows (0 = automatic), overlapping the copies with
 * the sketch.  Synchronises the handle's stream before returning. */
SMP_API smp_status smp_sketch_block_host(smp_handle* h, int64_t row0, int64_t rows, const void* A,
                                 int64_t lda, const void* B, int64_t ldb, int64_t chunk_rows);

/* CSR variant (SMP_IN_CSR_F32; bag-of-words inputs, P:9): row
 * t = row0 + r has entries (col[p], val[p]) for
 * p in [rowptr[r] - rowptr[0], rowptr[r+1] - rowptr[0]); rowptr has rows+1
 * entries.  Column indices must lie in [0, n): an out-of-range index is
 * reported by smp_finalize_norms (SMP_EINVAL).  Columns with density
 * >= 2% (env SMP_CSR_HEAD_DENSITY) and small-integer values go through the
 * tensor-core sketch as a dense head; the rest through the sparse kernels
 * (K3).  Norms² are exact for integer counts.  Synchronises
 * (head selection and panel sizes are read back).  Errors: SMP_EINVAL
 * (null arrays, > 2^26 columns), SMP_ECUDA. */
SMP_API smp_status smp_sketch_block_csr(smp_handle* h, int64_t row0, int64_t rows, const int64_t* a_rowptr,
                                const int32_t* a_col, const float* a_val, int64_t a_nnz,
                                const int64_t* b_rowptr, const int32_t* b_col, const float* b_val,
                                int64_t b_nnz);

/* Expose the packed partial accumulators (fp32 UNSCALED sketch sums, n_tot×k
 * with n_tot = n1 + n2 (n1 if a_is_b), then fp64 column norms² n_tot) so the
 * caller can combine shards with an all-reduce-sum in place (Spark's
 * treeAggregate, P:145 → NCCL over NVLink).  Not needed with a
 * single shard.  Pointers stay valid until smp_destroy. */
SMP_API smp_status smp_sketch_partials(smp_handle* h, float** sk, int64_t* sk_count, double** nrm,
                               int64_t* nrm_count);

/* The same partials as ONE fp64 exchange buffer for a single all-reduce-sum
 * (the north star's "one NCCL allreduce"): *buf (device, owned
 * by the handle, valid until the next pack or smp_destroy) receives
 * [n_tot·k sketch sums widened exactly to fp64 | n_tot norms²], *count its
 * length in doubles.  Enqueued on the handle's stream (no host sync): the
 * caller's collective must be ordered after it on that stream.  After the
 * all-reduce, smp_sketch_unpack_partials writes the reduced buffer back into
 * the accumulators (sketch rounded to fp32 once), ready for
 * smp_finalize_norms.  Errors: SMP_EINVAL (null handle / arguments), SMP_ECUDA. */
SMP_API smp_status smp_sketch_pack_partials(smp_handle* h, double** buf, int64_t* count);
SMP_API smp_status smp_sketch_unpack_partials(smp_handle* h);

/* Finalize: Ã = (sum)·fp32(1/sqrt(k)), ||Ã_i|| (fp64 → fp32
 * out), ||A||_F² and ||B||_F² by the fixed pairwise tree (R5).
 * Any output pointer may be NULL.  A_sk: n1×k, B_sk: n2×k (= A_sk's content
 * if a_is_b), a_norm2/b_norm2: fp64 ||A_i||², frob2[2] = {||A||_F², ||B||_F²}.
 * Keeps the finalized state in the handle for smp_sample_estimate.
 * Synchronises.  Errors: SMP_ENUMERIC (zero Frobenius norm, NaN/Inf). */
SMP_API smp_status smp_finalize_norms(smp_handle* h, float* A_sk, float* B_sk, double* a_norm2,
                              double* b_norm2, double* frob2, float* a_sknorm, float* b_sknorm);

/* Step 2: draw Ω with q̂_ij = min(1, m(||A_i||²/(2 n2 ||A||_F²) +
 * ||B_j||²/(2 n1 ||B||_F²))) (Eq. 1, Alg. 1 line 3; Bernoulli from the
 * Philox hash of (seed, i, j)) and evaluate
 * M̃_ij = ||A_i|| ||B_j|| <Ã_i,B̃_j>/(||Ã_i|| ||B̃_j||) (Eq. 2; est = PLAIN
 * gives <Ã_i,B̃_j>) on Ω.  Outputs, sorted by (i,j): I, J (int32),
 * val (fp32 M̃), qhat (fp64); *count = |Ω| (written even on overflow).
 * cap = capacity of the output arrays.  Synchronises (to return *count).
 * Errors: SMP_EINVAL (m <= 0, not finalized), SMP_ECAPACITY (|Ω| > cap;
 * nothing written; call again with cap >= *count). */
/* Ω samplers: the Bernoulli hash sweep of Alg. 1 line 3 (n1·n2 draws,
 * bit-exact, q̂ = min(1, q)) or the appendix's row-multinomial sampler
 * (P:633-639 with line 3's saturation; R27; O(n2 log n2 + m log n2)):
 * pairs with q_ij >= 1 are always in Ω (q̂ = 1); the unsaturated mass of row
 * i, T_i, is drawn M_i = floor(m T_i + u) times with replacement by CDF
 * inversion of q̃_ij ∝ α_i + β_j over the unsaturated columns; Ω holds each
 * drawn pair once, with qhat = its inclusion probability
 * 1 − (1 − π)^F (1 − fπ), π = (α_i + β_j)/T_i, F = ⌊m T_i⌋, f = m T_i − F.
 * Synchronises twice.  Errors as smp_sample_estimate, plus SMP_EINVAL when
 * the draws exceed 2^31 entries. */
enum { SMP_SAMPLER_BERNOULLI = 0, SMP_SAMPLER_MULTINOMIAL = 1 };
SMP_API smp_status smp_sample_estimate_ex(smp_handle* h, double m, uint64_t seed, int32_t est,
                                          int32_t sampler, int64_t cap, int32_t* I, int32_t* J,
                                          float* val, double* qhat, int64_t* count);

SMP_API smp_status smp_sample_estimate(smp_handle* h, double m, uint64_t seed, int32_t est, int64_t cap,
                               int32_t* I, int32_t* J, float* val, double* qhat, int64_t* count);

/* Alg. 2 line 3, R11.  REUSE_ALL: all of Ω for the init
 * and every half step (the deployed ALS).  FRESH_2T1: Ω divided into
 * 2T+1 equal random subsets — sample (i, j) keyed by Philox(ctr = (i, j, 0,
 * 4), key = waltmin seed), ranked by (key, position), rank p -> subset
 * p mod (2T+1) — Ω_0 for lines 4-5, Ω_{2t+1} for line 8 and Ω_{2t+2} for
 * line 9 of iteration t. */
typedef enum { SMP_PART_REUSE_ALL = 0, SMP_PART_FRESH_2T1 = 1 } smp_part;

typedef struct {
  int32_t r;          /* rank, 1 <= r <= 16, r <= min(n1, n2)                 */
  int32_t T;          /* ALS iterations (Alg. 2 lines 7-10), T >= 1            */
  int32_t partition;  /* smp_part (Alg. 2 line 3 reading, R11)       */
  int32_t init_iters; /* subspace iterations for line 5 (R12), >= 1 */
  double trim_c;      /* trim constant c of line 6 (R13); 0 = off   */
  double ridge;       /* λ of the normal equations (R14)            */
  uint64_t seed;      /* seed of the Rademacher start of line 5               */
} smp_waltmin_desc;

/* Step 3: WAltMin (Alg. 2) on (I, J, val, qhat) as
 * produced by smp_sample_estimate (sorted by (i,j), distinct pairs); uses
 * the handle's ||A_i|| and ||A||_F for the trim.  Outputs U (n1×r) and V
 * (n2×r) fp32 row-major with ÛV̂ᵀ ≈ (AᵀB)_r.  Synchronises.  Errors:
 * SMP_EINVAL (r outside [1, min(16, n1, n2)], T < 1, init_iters < 1, unknown
 * partition, FRESH_2T1 with count < 2T+1, null arrays), SMP_ECUDA. */
SMP_API smp_status smp_waltmin(smp_handle* h, const int32_t* I, const int32_t* J, const float* val,
                       const double* qhat, int64_t count, const smp_waltmin_desc* w, float* U,
                       float* V);

/* LELA (Bhojanapalli et al.; the paper's two-pass comparison system, P:78,
 * P:145, Table 1, runtime P:191-192; DESIGN.md NEXT-3).  Pass 1:
 * smp_norms_block accumulates ONLY the exact column norms² (fp64) of rows
 * [row0, row0+rows) into the handle (no sketch; blocks in any order), after
 * which smp_finalize_norms and smp_sample_estimate give Ω and q̂ by Eq. 1
 * exactly as for SMP-PCA (its M̃ values are then 0 and unused).  Pass 2:
 * smp_exact_entries_block adds Σ_{t in block} A[t, I_s]·B[t, J_s] (fp64) to
 * acc[s] for the count samples (I, J device int32, acc device fp64, zeroed by
 * the caller before the first block); after every row block, acc = (AᵀB)_Ω,
 * the exact entries smp_waltmin then completes (as fp32 val).  Dense inputs
 * only (bf16 or fp32, any leading dimension >= n).  Errors: SMP_EINVAL (rows
 * outside [row_begin, row_end), CSR handle, null arrays, ld < n), SMP_ECUDA. */
SMP_API smp_status smp_norms_block(smp_handle* h, int64_t row0, int64_t rows, const void* A, int64_t lda,
                                   const void* B, int64_t ldb);
SMP_API smp_status smp_exact_entries_block(smp_handle* h, int64_t row0, int64_t rows, const void* A,
                                           int64_t lda, const void* B, int64_t ldb, const int32_t* I,
                                           const int32_t* J, int64_t count, double* acc);

/* Reset the accumulators to zero (reuse the handle for another pass). */
SMP_API smp_status smp_sketch_reset(smp_handle* h);

/* Instrumentation: when enabled, the library brackets every launch of the
 * dense sketch kernel (K1) with CUDA events on the handle's stream.
 * smp_kernel_timing synchronises, returns the summed K1 device time (ms) and
 * the number of K1 launches since the previous query, and clears them. */
SMP_API smp_status smp_set_timing(smp_handle* h, int32_t enable);
SMP_API smp_status smp_kernel_timing(smp_handle* h, double* ms_total, int64_t* launches);

/* Number of kernels this handle has launched (instrumentation). */
SMP_API int64_t smp_kernel_launches(const smp_handle* h);

SMP_API void smp_destroy(smp_handle* h);
SMP_API const char* smp_last_error(const smp_handle* h);
SMP_API const char* smp_status_str(smp_status s);

#ifdef __cplusplus
}
#endif
#endif /* SMP_H_ */
