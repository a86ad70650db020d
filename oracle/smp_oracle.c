/*
 * SMP-PCA CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * This file is the plain, slow, obviously-correct fp64 reference for the hot
 * path of SMP-PCA (arXiv 1610.06656).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares
 * NO code with the CUDA path (paper_1610_06656_b200/csrc): the hash, the
 * Gaussian generator, the sampling arithmetic and WAltMin are re-implemented
 * here from the written definitions in DESIGN.md §3.
 *
 * Citation convention: "P:L" = /root/reference/PAPER.md line L.
 *
 *   Alg. 1 line 2  -> or_sketch_rows        (Step 1)
 *   Eq. 1         -> or_qhat / or_sample   (Step 2, Alg.1 l.3)
 *   Eq. 2         -> or_estimate           (Step 2, Alg.1 l.4)
 *   Alg. 2       -> or_waltmin            (Step 3, Eq. 3)
 *
 * Every floating-point quantity is fp64 unless the definition
 * fixes fp32 (the Gaussian generator G, which must produce identical bf16
 * bits on both sides).  Compile with -ffp-contract=off so that no FMA is
 * introduced where the definition does not name one.
 *
 * Parity status of each function is listed in DESIGN.md §4 ("pins").
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* H: Philox4x32-10 (Salmon et al., SC'11).  DESIGN.md §3.1.                  */
/* ------------------------------------------------------------------------ */
void or_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

static void philox_seed(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                        uint32_t out[4])
{
    uint32_t ctr[4] = {c0, c1, c2, c3};
    uint32_t key[2] = {(uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32)};
    or_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------------ */
/* Π entries (Alg. 1 line 2; "any oblivious subspace embedding"). */
/* Values are UNSCALED (±1, or a bf16-valued Gaussian); the 1/sqrt(k) factor  */
/* of N(0,1/k) is applied to the sketch at finalize (R1).           */
/* ------------------------------------------------------------------------ */
enum { OR_PI_RADEMACHER = 0, OR_PI_GAUSSIAN = 1, OR_PI_HADAMARD = 2 };

double or_pi_rademacher(uint64_t seed, int64_t kappa, int64_t t)
{
    uint32_t w[4];
    philox_seed(seed, (uint32_t)((uint64_t)t >> 7), (uint32_t)kappa,
                (uint32_t)((uint64_t)t >> 39), 1u, w);
    /* row offset b = t & 127 lives in word b >> 5; inside the word, element
       e = b & 31 sits at bit (e >> 1) + 16 (e & 1): even rows use bits 0..15,
       odd rows bits 16..31. */
    unsigned b = (unsigned)(t & 127);
    unsigned e = b & 31u;
    unsigned pos = (e >> 1) + ((e & 1u) << 4);
    unsigned bit = (w[b >> 5] >> pos) & 1u;
    return bit ? -1.0 : 1.0;
}

static float u32_as_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f32_as_u32(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* Round fp32 to the nearest bf16 (ties to even); returned as the fp32 value. */
static float bf16_rne(float x)
{
    uint32_t u = f32_as_u32(x);
    uint32_t lsb = (u >> 16) & 1u;
    u = (u + 0x7FFFu + lsb) & 0xFFFF0000u;
    return u32_as_f32(u);
}

/* G: stated fp32 Box–Muller.  Only IEEE correctly-rounded  */
/* fp32 operations (+, *, fmaf, sqrtf, exact int<->float) are used, each in   */
/* the order written, so that the CUDA side produces identical bits.          */
static void gauss_pair(uint32_t wa, uint32_t wb, float *z0, float *z1)
{
    /* ln(1+y) = y * P(y), P of degree 9, coefficients fp32. */
    static const float L[10] = {
        0x1.000000p+0f, -0x1.000000p-1f, 0x1.5555c6p-2f, -0x1.00003ep-2f, 0x1.996178p-3f,
        -0x1.54e596p-3f, 0x1.28ce66p-3f, -0x1.0e2b8ep-3f, 0x1.ac49bap-4f, -0x1.6e4bbap-5f};
    const float LN2 = 0x1.62e430p-1f;
    /* sin(pi x/2) = x*(S1 + x2*(S3 + ...)), cos(pi x/2) = 1 + x2*(C2 + ...) */
    const float S1 = 0x1.921fb6p+0f, S3 = -0x1.4abbcep-1f, S5 = 0x1.466bc6p-4f,
                S7 = -0x1.32d2ccp-8f, S9 = 0x1.507834p-13f;
    const float C2 = -0x1.3bd3ccp+0f, C4 = 0x1.03c1f0p-2f, C6 = -0x1.55d3c8p-6f,
                C8 = 0x1.e1f506p-11f, C10 = -0x1.a6d1f2p-16f;

    /* u1 in (0,1] */
    uint32_t v1 = (wa >> 8) + 1u;
    float u1 = (float)v1 * 0x1p-24f;           /* exact */
    uint32_t bits = f32_as_u32(u1);
    int e = (int)(bits >> 23) - 127;
    uint32_t mant = bits & 0x7FFFFFu;
    float f;
    if (mant >= 0x400000u) {                   /* f >= 1.5: use f/2 in [0.75,1) */
        f = u32_as_f32(mant | 0x3F000000u);
        e += 1;
    } else {
        f = u32_as_f32(mant | 0x3F800000u);
    }
    float y = f - 1.0f;                        /* exact (Sterbenz) */
    float p = L[9];
    for (int i = 8; i >= 0; --i) p = fmaf(p, y, L[i]);
    float lnf = y * p;
    float lnu = fmaf((float)e, LN2, lnf);
    float r2 = -2.0f * lnu;                    /* exact */
    float rho = sqrtf(r2);

    /* angle 2*pi*u2, u2 = v2 * 2^-24 in [0,1) */
    uint32_t v2 = wb >> 8;
    uint32_t qn = (v2 + 0x200000u) >> 22;      /* nearest quadrant, 0..4 */
    int32_t xi = (int32_t)v2 - (int32_t)(qn << 22);
    float x = (float)xi * 0x1p-22f;            /* exact, in [-0.5,0.5) */
    float x2 = x * x;
    float sp = fmaf(fmaf(fmaf(fmaf(S9, x2, S7), x2, S5), x2, S3), x2, S1);
    float sn = x * sp;
    float cs = fmaf(fmaf(fmaf(fmaf(fmaf(C10, x2, C8), x2, C6), x2, C4), x2, C2), x2, 1.0f);
    float c, s;
    switch (qn & 3u) {
    case 0: c = cs; s = sn; break;
    case 1: c = -sn; s = cs; break;
    case 2: c = -cs; s = -sn; break;
    default: c = sn; s = -cs; break;
    }
    *z0 = bf16_rne(rho * c);
    *z1 = bf16_rne(rho * s);
}

double or_pi_gaussian(uint64_t seed, int64_t kappa, int64_t t)
{
    uint32_t w[4];
    philox_seed(seed, (uint32_t)((uint64_t)t >> 2), (uint32_t)kappa,
                (uint32_t)((uint64_t)t >> 34), 2u, w);
    unsigned sel = (unsigned)(t & 3);
    float z0, z1;
    if (sel < 2) gauss_pair(w[0], w[1], &z0, &z1);
    else gauss_pair(w[2], w[3], &z0, &z1);
    return (double)((sel & 1u) ? z1 : z0);
}

static int popcount64(uint64_t x)
{
    int c = 0;
    while (x) { c += (int)(x & 1u); x >>= 1; }
    return c;
}

double or_pi_hadamard(int64_t kappa, int64_t t)
{
    return (popcount64((uint64_t)kappa & (uint64_t)t) & 1) ? -1.0 : 1.0;
}

/* ------------------------------------------------------------------------ */
/* SRHT (the sketch the paper's Spark code used, P:145 and its footnote;     */
/* SURVEY §8f NEXT-1; R26):  Π = sqrt(d/k) S H D with H the        */
/* normalised Sylvester-Hadamard matrix of order 2^L >= d, D = diag(±1) and  */
/* S k distinct rows of H sampled without replacement.  Unscaled entries:    */
/*   Π(κ, t) = D_t · (−1)^popcount(s_κ & t),  s_κ = F_L(κ),                 */
/* D_t: bit of Philox(ctr = (t>>7, 0, t>>39, 6)) in the Rademacher layout;   */
/* F_L: a bijection of [0, 2^L) — 4-round unbalanced Feistel, halves        */
/* a = L/2 (high) and b = L − a (low) bits; even rounds hi ^= f(lo) mod 2^a, */
/* odd rounds lo ^= f(hi) mod 2^b, f(v) = word 0 of                         */
/* Philox(ctr = (v, round, L, 7)).  Internal kind code: 16 + L.              */
/* ------------------------------------------------------------------------ */
int64_t or_srht_row(uint64_t seed, int L, int64_t kappa)
{
    const int a = L / 2, b = L - a;
    const uint64_t mb = b >= 64 ? ~0ull : ((1ull << b) - 1), ma = a >= 64 ? ~0ull : ((1ull << a) - 1);
    uint64_t lo = (uint64_t)kappa & mb, hi = ((uint64_t)kappa >> b) & ma;
    for (int r = 0; r < 4; ++r) {
        uint32_t w[4];
        if ((r & 1) == 0) {
            philox_seed(seed, (uint32_t)lo, (uint32_t)r, (uint32_t)L, 7u, w);
            hi ^= (uint64_t)w[0] & ma;
        } else {
            philox_seed(seed, (uint32_t)hi, (uint32_t)r, (uint32_t)L, 7u, w);
            lo ^= (uint64_t)w[0] & mb;
        }
    }
    return (int64_t)((hi << b) | lo);
}

double or_srht_sign(uint64_t seed, int64_t t)
{
    uint32_t w[4];
    philox_seed(seed, (uint32_t)((uint64_t)t >> 7), 0u, (uint32_t)((uint64_t)t >> 39), 6u, w);
    unsigned b = (unsigned)(t & 127);
    unsigned e = b & 31u;
    unsigned pos = (e >> 1) + ((e & 1u) << 4);
    return ((w[b >> 5] >> pos) & 1u) ? -1.0 : 1.0;
}

double or_pi_srht(uint64_t seed, int L, int64_t kappa, int64_t t)
{
    const int64_t s = or_srht_row(seed, L, kappa);
    const double h = (popcount64((uint64_t)s & (uint64_t)t) & 1) ? -1.0 : 1.0;
    return or_srht_sign(seed, t) * h;
}

double or_pi_entry(int kind, uint64_t seed, int64_t kappa, int64_t t)
{
    if (kind == OR_PI_RADEMACHER) return or_pi_rademacher(seed, kappa, t);
    if (kind == OR_PI_GAUSSIAN) return or_pi_gaussian(seed, kappa, t);
    if (kind >= 16) return or_pi_srht(seed, kind - 16, kappa, t);
    return or_pi_hadamard(kappa, t);
}

/* ------------------------------------------------------------------------ */
/* Step 1: one pass over rows of X (Alg. 1 line 2).           */
/*   sk[c*k + kappa] += Π(kappa, t) * X[t, c]     (unscaled, fp64)           */
/*   norm2[c]        += X[t, c]^2                 (fp64)                     */
/* X is row-major with leading dimension ldx; dtype 0 = fp64, 1 = fp32,      */
/* 2 = bf16 (raw uint16).  Global row of local row r is row0 + r.            */
/* ------------------------------------------------------------------------ */
static double load_elem(const void *X, int dtype, int64_t idx)
{
    if (dtype == 0) return ((const double *)X)[idx];
    if (dtype == 1) return (double)((const float *)X)[idx];
    uint32_t u = (uint32_t)((const uint16_t *)X)[idx] << 16;
    return (double)u32_as_f32(u);
}

void or_sketch_rows(int kind, uint64_t seed, int k, int64_t row0, int64_t rows, int64_t n,
                    const void *X, int dtype, int64_t ldx, double *sk, double *norm2)
{
    const int64_t RB = 256;                    /* Π materialised per 256-row block */
    double *pi = (double *)malloc(sizeof(double) * (size_t)RB * (size_t)k);
    for (int64_t r0 = 0; r0 < rows; r0 += RB) {
        int64_t rb = rows - r0 < RB ? rows - r0 : RB;
        #pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < rb; ++r)
            for (int kp = 0; kp < k; ++kp)
                pi[r * k + kp] = or_pi_entry(kind, seed, kp, row0 + r0 + r);
        #pragma omp parallel for schedule(static)
        for (int64_t c = 0; c < n; ++c) {
            double *skc = sk + c * (int64_t)k;
            for (int64_t r = 0; r < rb; ++r) {
                double x = load_elem(X, dtype, (r0 + r) * ldx + c);
                norm2[c] += x * x;
                const double *pr = pi + r * k;
                for (int kp = 0; kp < k; ++kp) skc[kp] += pr[kp] * x;
            }
        }
    }
    free(pi);
}

/* Sketch of a single column subset (sampled parity at full size): columns    */
/* cols[0..nc) of X over rows [0, rows), same accumulation order as above.    */
void or_sketch_cols(int kind, uint64_t seed, int k, int64_t row0, int64_t rows,
                    int64_t nc, const int64_t *cols, const void *X, int dtype, int64_t ldx,
                    double *sk, double *norm2)
{
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t ci = 0; ci < nc; ++ci) {
        double *skc = sk + ci * (int64_t)k;
        int64_t c = cols[ci];
        for (int64_t r = 0; r < rows; ++r) {
            double x = load_elem(X, dtype, r * ldx + c);
            norm2[ci] += x * x;
            if (x != 0.0)
                for (int kp = 0; kp < k; ++kp)
                    skc[kp] += or_pi_entry(kind, seed, kp, row0 + r) * x;
        }
    }
}

/* CSR rows (bag-of-words input, P:9): row t has entries             */
/* (col[p], val[p]) for p in [rowptr[t], rowptr[t+1]).                       */
void or_sketch_csr(int kind, uint64_t seed, int k, int64_t row0, int64_t rows, int64_t n,
                   const int64_t *rowptr, const int32_t *col, const float *val,
                   double *sk, double *norm2)
{
    /* Π(:, t) for the non-empty rows of each 256-row block (generation only;
       the accumulation below runs in row order, entry by entry). */
    const int64_t RB = 256;
    double *pi = (double *)malloc(sizeof(double) * (size_t)RB * (size_t)k);
    (void)n;
    for (int64_t r0 = 0; r0 < rows; r0 += RB) {
        int64_t rb = rows - r0 < RB ? rows - r0 : RB;
        #pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < rb; ++r) {
            if (rowptr[r0 + r] == rowptr[r0 + r + 1]) continue;
            for (int kp = 0; kp < k; ++kp) pi[r * k + kp] = or_pi_entry(kind, seed, kp, row0 + r0 + r);
        }
        for (int64_t r = 0; r < rb; ++r) {
            const double *pr = pi + r * k;
            for (int64_t p = rowptr[r0 + r]; p < rowptr[r0 + r + 1]; ++p) {
                int64_t c = col[p - rowptr[0]];
                double x = (double)val[p - rowptr[0]];
                norm2[c] += x * x;
                double *skc = sk + c * (int64_t)k;
                for (int kp = 0; kp < k; ++kp) skc[kp] += pr[kp] * x;
            }
        }
    }
    free(pi);
}

/* Column norms only: norm2[c] += Σ_t X[t, c]^2 in fp64 (the norm half of    */
/* Step 1), for full-size Ω parity without the full sketch.         */
void or_colnorms(int64_t rows, int64_t n, const void *X, int dtype, int64_t ldx, double *norm2)
{
    #pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < n; ++c) {
        double s = norm2[c];
        for (int64_t r = 0; r < rows; ++r) {
            double x = load_elem(X, dtype, r * ldx + c);
            s += x * x;
        }
        norm2[c] = s;
    }
}

/* ------------------------------------------------------------------------ */
/* Finalize (D_A/D_B definition).                                */
/* ------------------------------------------------------------------------ */
/* R5: Frobenius^2 by a fixed pairwise tree over the column norms^2:        */
/* pad to a power of two with zeros, sum adjacent pairs level by level.      */
double or_pairwise_sum(const double *x, int64_t n)
{
    if (n <= 0) return 0.0;
    int64_t p = 1;
    while (p < n) p <<= 1;
    double *buf = (double *)calloc((size_t)p, sizeof(double));
    memcpy(buf, x, sizeof(double) * (size_t)n);
    while (p > 1) {
        p >>= 1;
        for (int64_t i = 0; i < p; ++i) buf[i] = buf[2 * i] + buf[2 * i + 1];
    }
    double s = buf[0];
    free(buf);
    return s;
}

/* Scales the unscaled sketch sk (n x k) by 1/sqrt(k) into out (n x k),      */
/* and computes sknorm[c] = ||Ã_c|| and D[c] = ||X_c|| / ||Ã_c|| (0 if 0).  */
/* DESIGN.md R25: a column whose norm² is below 2^-200 is the zero column     */
/* (norm2[c] is set to 0, so Eq. 1 and D see an exact zero).                 */
void or_finalize(int k, int64_t n, const double *sk, double *norm2,
                 double *out, double *sknorm, double *D)
{
    double scale = 1.0 / sqrt((double)k);
    for (int64_t c = 0; c < n; ++c) {
        double s2 = 0.0;
        for (int kp = 0; kp < k; ++kp) {
            double v = sk[c * k + kp] * scale;
            out[c * k + kp] = v;
            s2 += v * v;
        }
        if (norm2[c] < 0x1p-200) norm2[c] = 0.0;
        sknorm[c] = sqrt(s2);
        D[c] = sknorm[c] > 0.0 ? sqrt(norm2[c]) / sknorm[c] : 0.0;
    }
}

/* ------------------------------------------------------------------------ */
/* Eq. 1 with q̂ = min(1, q) (Alg. 1 line 3).                */
/* R6: alpha_i = a2_i / ((2 n2) FA), beta_j = b2_j / ((2 n1) FB),            */
/*     q = m * (alpha_i + beta_j), no FMA.                                   */
/* ------------------------------------------------------------------------ */
void or_alpha_beta(int64_t n1, int64_t n2, const double *a2, const double *b2,
                   double FA, double FB, double *alpha, double *beta)
{
    double da = (2.0 * (double)n2) * FA;
    double db = (2.0 * (double)n1) * FB;
    for (int64_t i = 0; i < n1; ++i) alpha[i] = a2[i] / da;
    for (int64_t j = 0; j < n2; ++j) beta[j] = b2[j] / db;
}

double or_qhat(double m, double alpha_i, double beta_j)
{
    double q = m * (alpha_i + beta_j);
    return q < 1.0 ? q : 1.0;
}

/* ------------------------------------------------------------------------ */
/* Row-multinomial sampler (the paper's appendix, with Alg. 1     */
/* line 3's saturation q̂ = min(1, q)     */
/* R27).  With α, β from or_alpha_beta and q_ij = m(α_i + β_j) (Eq. 1, R6):  */
/*  * σ orders the columns by β descending (ties: column index ascending);   */
/*    Bp[p] = β_σ(0) + ... + β_σ(p) (sequential, fp64), Btot = Bp[n2-1].     */
/*  * Row i's saturated pairs — q_ij >= 1, always in Ω with q̂ = 1 as in the  */
/*    Bernoulli model — are the prefix p < s_i of σ (q is non-increasing     */
/*    in p): s_i = the first p with m(α_i + β_σ(p)) < 1 (binary search).     */
/*  * The unsaturated mass T_i = (n2 − s_i)·α_i + (Btot − Bp[s_i−1]) (the     */
/*    appendix's m_i/m restricted to unsaturated columns; Bp[−1] = 0) is      */
/*    drawn row-wise multinomially: m_i = m·T_i, M_i = floor(m_i + u_i),      */
/*    u_i = U53(Philox(i, 0, 0, 8)) 2^-53; draw d: target = U53(Philox(i, d,   */
/*    0, 9)) 2^-53 · T_i, p = the first p >= s_i with                        */
/*    C_i(p) = (p − s_i + 1)·α_i + (Bp[p] − Bp[s_i−1]) > target (n2−1 if       */
/*    none): inversion of the affine CDF of q̃_ij ∝ α_i + β_j ("only   */
/*    update the linear shift and scale"); column j = σ(p).                   */
/*  * Ω = saturated pairs ∪ the SET of drawn pairs, sorted by (i, j).  A      */
/*    drawn pair's inclusion probability, with π = (α_i + β_j)/T_i,          */
/*    F = floor(m_i), f = m_i − F (M_i = F + 1 w.p. f):                       */
/*      q̂_ij = 1 − (1−π)^F (1 − fπ) = −expm1(F·log1p(−π) + log1p(−fπ))      */
/*    (π >= 1: q̂ = 1 if F >= 1, else f); WAltMin weights it 1/q̂ (Alg. 2    */
/*    line 2).  For q ≪ 1, q̂ → q (the Bernoulli marginal).                  */
/* O(n2 log n2 + n1 log n2 + m log n2) work (P:633-639's O(m log n)).        */
/* ------------------------------------------------------------------------ */
static double u53(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t tag)
{
    uint32_t w[4];
    philox_seed(seed, c0, c1, 0u, tag, w);
    uint64_t v = (((uint64_t)w[1] << 32) | (uint64_t)w[0]) >> 11;
    return (double)v * 0x1p-53;
}

static int cmp_i32(const void *a, const void *b)
{
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

typedef struct { double b; int64_t j; } beta_rec;

static int cmp_beta_desc(const void *a, const void *b)
{
    const beta_rec *x = (const beta_rec *)a, *y = (const beta_rec *)b;
    if (x->b != y->b) return x->b > y->b ? -1 : 1;
    return (x->j > y->j) - (x->j < y->j);
}

typedef struct {
    int64_t n2;
    int64_t *sig;   /* σ */
    double *bp;     /* Bp */
    double btot;
} mn_ctx;

static void mn_setup(mn_ctx *c, int64_t n2, const double *beta)
{
    beta_rec *r = (beta_rec *)malloc(sizeof(beta_rec) * (size_t)(n2 > 0 ? n2 : 1));
    for (int64_t j = 0; j < n2; ++j) { r[j].b = beta[j]; r[j].j = j; }
    qsort(r, (size_t)n2, sizeof(beta_rec), cmp_beta_desc);
    c->n2 = n2;
    c->sig = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n2 > 0 ? n2 : 1));
    c->bp = (double *)malloc(sizeof(double) * (size_t)(n2 > 0 ? n2 : 1));
    double acc = 0.0;
    for (int64_t p = 0; p < n2; ++p) {
        c->sig[p] = r[p].j;
        acc = acc + r[p].b;
        c->bp[p] = acc;
    }
    c->btot = n2 > 0 ? c->bp[n2 - 1] : 0.0;
    free(r);
}

static void mn_free(mn_ctx *c) { free(c->sig); free(c->bp); }

/* s_i and T_i of row i */
static void mn_row(const mn_ctx *c, double m, double alpha_i, const double *beta, int64_t *s_out,
                   double *T_out)
{
    int64_t lo = 0, hi = c->n2;                 /* first p with q < 1, n2 if none */
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        const double q = m * (alpha_i + beta[c->sig[mid]]);
        if (q < 1.0) hi = mid; else lo = mid + 1;
    }
    const double base = lo > 0 ? c->bp[lo - 1] : 0.0;
    *s_out = lo;
    *T_out = (double)(c->n2 - lo) * alpha_i + (c->btot - base);
}

/* column of draw d of row i (given s_i, T_i) */
static int64_t mn_draw(const mn_ctx *c, uint64_t seed, int64_t i, int64_t d, double alpha_i, int64_t s,
                       double T)
{
    const double target = u53(seed, (uint32_t)i, (uint32_t)d, 9u) * T;
    const double base = s > 0 ? c->bp[s - 1] : 0.0;
    int64_t lo = s, hi = c->n2 - 1;             /* first p >= s with C(p) > target, else n2-1 */
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        const double cdf = (double)(mid - s + 1) * alpha_i + (c->bp[mid] - base);
        if (cdf > target) hi = mid; else lo = mid + 1;
    }
    return c->sig[lo];
}

static int64_t mn_count(uint64_t seed, double m, int64_t i, double T)
{
    return (int64_t)floor(m * T + u53(seed, (uint32_t)i, 0u, 8u));
}

/* Raw multinomial draws of the unsaturated part (with replacement, sorted   */
/* by (i, j), duplicates kept); sat[i] (optional) receives s_i.              */
int64_t or_multinomial_draws(uint64_t seed, double m, int64_t n1, int64_t n2, const double *alpha,
                             const double *beta, int64_t cap, int32_t *I, int32_t *J, int64_t *sat)
{
    mn_ctx c;
    mn_setup(&c, n2, beta);
    int64_t cnt = 0;
    for (int64_t i = 0; i < n1; ++i) {
        int64_t s;
        double T;
        mn_row(&c, m, alpha[i], beta, &s, &T);
        if (sat) sat[i] = s;
        const int64_t Mi = s < n2 ? mn_count(seed, m, i, T) : 0;
        const int64_t c0 = cnt;
        for (int64_t d = 0; d < Mi; ++d) {
            const int64_t j = mn_draw(&c, seed, i, d, alpha[i], s, T);
            if (cnt < cap) { I[cnt] = (int32_t)i; J[cnt] = (int32_t)j; }
            ++cnt;
        }
        if (cnt <= cap && cnt > c0) qsort(J + c0, (size_t)(cnt - c0), sizeof(int32_t), cmp_i32);
    }
    mn_free(&c);
    return cnt;
}

/* q̂_ij of a drawn (unsaturated) pair; T_i as above. */
double or_mn_qhat(double m, double alpha_i, double beta_j, double T_i)
{
    const double mi = m * T_i;
    const double F = floor(mi);
    const double f = mi - F;
    const double pi = (alpha_i + beta_j) / T_i;
    if (!(pi > 0.0)) return 0.0;
    if (pi >= 1.0) return F >= 1.0 ? 1.0 : f;
    return -expm1(F * log1p(-pi) + log1p(-f * pi));
}

/* Ω of the multinomial model; returns |Ω|, writes at most cap entries.     */
int64_t or_sample_multinomial(uint64_t seed, double m, int64_t n1, int64_t n2, const double *alpha,
                              const double *beta, int64_t cap, int32_t *I, int32_t *J, double *q)
{
    mn_ctx c;
    mn_setup(&c, n2, beta);
    int32_t *row = (int32_t *)malloc(sizeof(int32_t) * 64);
    int64_t rcap = 64;
    int64_t cnt = 0;
    for (int64_t i = 0; i < n1; ++i) {
        int64_t s;
        double T;
        mn_row(&c, m, alpha[i], beta, &s, &T);
        const int64_t Mi = s < n2 ? mn_count(seed, m, i, T) : 0;
        if (s + Mi > rcap) {
            rcap = s + Mi;
            row = (int32_t *)realloc(row, sizeof(int32_t) * (size_t)rcap);
        }
        for (int64_t p = 0; p < s; ++p) row[p] = (int32_t)c.sig[p];
        for (int64_t d = 0; d < Mi; ++d) row[s + d] = (int32_t)mn_draw(&c, seed, i, d, alpha[i], s, T);
        qsort(row, (size_t)(s + Mi), sizeof(int32_t), cmp_i32);
        for (int64_t e = 0; e < s + Mi; ++e) {
            if (e > 0 && row[e] == row[e - 1]) continue;          /* the set Ω */
            if (cnt < cap) {
                const int32_t j = row[e];
                const double qq = m * (alpha[i] + beta[j]);
                I[cnt] = (int32_t)i;
                J[cnt] = j;
                q[cnt] = qq >= 1.0 ? 1.0 : or_mn_qhat(m, alpha[i], beta[j], T);
            }
            ++cnt;
        }
    }
    free(row);
    mn_free(&c);
    return cnt;
}

/* s_i and T_i per row (tests) */
void or_mn_rows(double m, int64_t n1, int64_t n2, const double *alpha, const double *beta, int64_t *s,
                double *T)
{
    mn_ctx c;
    mn_setup(&c, n2, beta);
    for (int64_t i = 0; i < n1; ++i) mn_row(&c, m, alpha[i], beta, &s[i], &T[i]);
    mn_free(&c);
}

/* Bernoulli draw for pair (i,j): U53 from Philox(ctr=(i,j,0,3), key=seed).  */
int or_draw(uint64_t seed, int64_t i, int64_t j, double qhat)
{
    uint32_t w[4];
    philox_seed(seed, (uint32_t)i, (uint32_t)j, 0u, 3u, w);
    uint64_t u53 = (((uint64_t)w[1] << 32) | (uint64_t)w[0]) >> 11;
    double u = (double)u53 * 0x1p-53;          /* exact */
    return u < qhat;
}

/* Ω in (i,j) order.  Returns the count; writes at most cap entries.        */
int64_t or_sample(uint64_t seed, double m, int64_t n1, int64_t n2,
                  const double *alpha, const double *beta, int64_t cap,
                  int32_t *I, int32_t *J, double *qhat)
{
    int64_t cnt = 0;
    for (int64_t i = 0; i < n1; ++i)
        for (int64_t j = 0; j < n2; ++j) {
            double q = or_qhat(m, alpha[i], beta[j]);
            if (or_draw(seed, i, j, q)) {
                if (cnt < cap) { I[cnt] = (int32_t)i; J[cnt] = (int32_t)j; qhat[cnt] = q; }
                ++cnt;
            }
        }
    return cnt;
}

/* Eq. 2: M̃_ij = ||A_i|| ||B_j|| <Ã_i,B̃_j> / (||Ã_i|| ||B̃_j||)    */
/*              = D_A[i] * D_B[j] * <Ã_i, B̃_j>.                  */
/* plain != 0 gives the JL estimator <Ã_i, B̃_j>.                     */
void or_estimate(int k, int64_t cnt, const int32_t *I, const int32_t *J,
                 const double *Ask, const double *Bsk, const double *DA, const double *DB,
                 int plain, double *out)
{
    for (int64_t s = 0; s < cnt; ++s) {
        const double *a = Ask + (int64_t)I[s] * k;
        const double *b = Bsk + (int64_t)J[s] * k;
        double dot = 0.0;
        for (int kp = 0; kp < k; ++kp) dot += a[kp] * b[kp];
        out[s] = plain ? dot : DA[I[s]] * DB[J[s]] * dot;
    }
}

/* ------------------------------------------------------------------------ */
/* WAltMin (Alg. 2).                                              */
/* ------------------------------------------------------------------------ */
/* Thin Householder QR of Z (n x r, row-major), Z <- Q (n x r).  Columns with */
/* no remaining energy become zero (rank-deficient input, R12).    */
static void householder_q(int64_t n, int r, double *Z)
{
    double *V = (double *)calloc((size_t)n * (size_t)r, sizeof(double));
    double *beta = (double *)calloc((size_t)r, sizeof(double));
    int *dead = (int *)calloc((size_t)r, sizeof(int));
    double *A = (double *)malloc(sizeof(double) * (size_t)n * (size_t)r);
    memcpy(A, Z, sizeof(double) * (size_t)n * (size_t)r);
    double fro = 0.0;
    for (int64_t i = 0; i < n * r; ++i) fro += A[i] * A[i];
    fro = sqrt(fro);
    for (int j = 0; j < r && j < n; ++j) {
        double nrm = 0.0;
        for (int64_t i = j; i < n; ++i) nrm += A[i * r + j] * A[i * r + j];
        nrm = sqrt(nrm);
        if (nrm <= 1e-14 * (fro > 0 ? fro : 1.0)) { dead[j] = 1; beta[j] = 0.0; continue; }
        double a0 = A[(int64_t)j * r + j];
        double alpha = a0 >= 0 ? -nrm : nrm;
        for (int64_t i = 0; i < n; ++i) V[i * r + j] = 0.0;
        V[(int64_t)j * r + j] = a0 - alpha;
        for (int64_t i = j + 1; i < n; ++i) V[i * r + j] = A[i * r + j];
        double vv = 0.0;
        for (int64_t i = j; i < n; ++i) vv += V[i * r + j] * V[i * r + j];
        beta[j] = vv > 0 ? 2.0 / vv : 0.0;
        for (int c = j; c < r; ++c) {
            double s = 0.0;
            for (int64_t i = j; i < n; ++i) s += V[i * r + j] * A[i * r + c];
            s *= beta[j];
            for (int64_t i = j; i < n; ++i) A[i * r + c] -= s * V[i * r + j];
        }
    }
    /* Q = H_0 H_1 ... H_{r-1} [I_r; 0] */
    for (int64_t i = 0; i < n * r; ++i) Z[i] = 0.0;
    for (int j = 0; j < r && j < n; ++j) Z[(int64_t)j * r + j] = dead[j] ? 0.0 : 1.0;
    for (int j = (r < n ? r : (int)n) - 1; j >= 0; --j) {
        if (dead[j]) continue;
        for (int c = 0; c < r; ++c) {
            double s = 0.0;
            for (int64_t i = j; i < n; ++i) s += V[i * r + j] * Z[i * r + c];
            s *= beta[j];
            for (int64_t i = j; i < n; ++i) Z[i * r + c] -= s * V[i * r + j];
        }
    }
    free(V); free(beta); free(dead); free(A);
}

/* Solve (G + lam*tr(G)/r * I) x = h by Cholesky, fp64.  Returns 0 if the   */
/* system is empty/singular (x = 0).                                          */
static int ridge_cholesky_solve(int r, const double *G, const double *h, double lam, double *x)
{
    double tr = 0.0;
    for (int a = 0; a < r; ++a) tr += G[a * r + a];
    for (int a = 0; a < r; ++a) x[a] = 0.0;
    if (!(tr > 0.0)) return 0;
    double L[32 * 32];
    double shift = lam * tr / (double)r;
    for (int a = 0; a < r; ++a)
        for (int b = 0; b < r; ++b) L[a * r + b] = G[a * r + b] + (a == b ? shift : 0.0);
    for (int j = 0; j < r; ++j) {
        double s = L[j * r + j];
        for (int p = 0; p < j; ++p) s -= L[j * r + p] * L[j * r + p];
        if (!(s > 0.0)) return 0;
        double d = sqrt(s);
        L[j * r + j] = d;
        for (int i = j + 1; i < r; ++i) {
            double t = L[i * r + j];
            for (int p = 0; p < j; ++p) t -= L[i * r + p] * L[j * r + p];
            L[i * r + j] = t / d;
        }
    }
    double y[32];
    for (int i = 0; i < r; ++i) {
        double t = h[i];
        for (int p = 0; p < i; ++p) t -= L[i * r + p] * y[p];
        y[i] = t / L[i * r + i];
    }
    for (int i = r - 1; i >= 0; --i) {
        double t = y[i];
        for (int p = i + 1; p < r; ++p) t -= L[p * r + i] * x[p];
        x[i] = t / L[i * r + i];
    }
    return 1;
}

/* One weighted least-squares half step (Alg. 2 lines 8/9; closed form       */
/* P:596-604).  For each output row o, over the samples s with side[s] == o: */
/*   G_o = sum w_s x_{other(s)} x_{other(s)}^T,  h_o = sum w_s M_s x_other   */
/* and out[o] = (G_o + lam tr(G_o)/r I)^{-1} h_o.                            */
void or_als_half(int r, int64_t n_out, int64_t cnt, const int32_t *side, const int32_t *other,
                 const double *val, const double *w, const double *X_other, double lam,
                 double *out)
{
    double *G = (double *)calloc((size_t)n_out * r * r, sizeof(double));
    double *h = (double *)calloc((size_t)n_out * r, sizeof(double));
    for (int64_t s = 0; s < cnt; ++s) {
        int64_t o = side[s];
        const double *x = X_other + (int64_t)other[s] * r;
        for (int a = 0; a < r; ++a) {
            h[o * r + a] += w[s] * val[s] * x[a];
            for (int b = 0; b < r; ++b) G[(o * r + a) * r + b] += w[s] * x[a] * x[b];
        }
    }
    for (int64_t o = 0; o < n_out; ++o)
        ridge_cholesky_solve(r, G + o * r * r, h + o * r, lam, out + o * r);
    free(G); free(h);
}

/* Alg. 2 line 3: "Divide Ω in 2T+1 equal uniformly random subsets"  */
/* (R11, the FRESH_2T1 partition).  Sample s = (i, j) gets the key  */
/* K_s = (w1 << 32) | w0 of Philox(ctr = (i, j, 0, 4), key = seed); samples   */
/* are ranked by (K_s, i, j, s) and the sample of rank p goes to subset       */
/* p mod nsub (nsub = 2T+1): subset sizes differ by at most one, and the      */
/* assignment is a uniformly random equal split (keys i.i.d. uniform).        */
typedef struct { uint64_t key; int32_t i, j; int64_t s; } part_rec;

static int cmp_part(const void *a, const void *b)
{
    const part_rec *x = (const part_rec *)a, *y = (const part_rec *)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    if (x->i != y->i) return x->i < y->i ? -1 : 1;
    if (x->j != y->j) return x->j < y->j ? -1 : 1;
    return (x->s > y->s) - (x->s < y->s);
}

void or_partition(uint64_t seed, int nsub, int64_t cnt, const int32_t *I, const int32_t *J, int32_t *sub)
{
    part_rec *r = (part_rec *)malloc(sizeof(part_rec) * (size_t)(cnt > 0 ? cnt : 1));
    for (int64_t s = 0; s < cnt; ++s) {
        uint32_t w[4];
        philox_seed(seed, (uint32_t)I[s], (uint32_t)J[s], 0u, 4u, w);
        r[s].key = ((uint64_t)w[1] << 32) | (uint64_t)w[0];
        r[s].i = I[s];
        r[s].j = J[s];
        r[s].s = s;
    }
    qsort(r, (size_t)cnt, sizeof(part_rec), cmp_part);
    for (int64_t p = 0; p < cnt; ++p) sub[r[p].s] = (int32_t)(p % nsub);
    free(r);
}

/* Samples of phase ph: all of Ω (REUSE_ALL) or subset Ω_ph (FRESH_2T1),   */
/* compacted in their original (i, j) order.                                 */
static int64_t phase_samples(int partition, int ph, int64_t cnt, const int32_t *sub, const int32_t *I,
                             const int32_t *J, const double *val, const double *w, int32_t *pI,
                             int32_t *pJ, double *pv, double *pw)
{
    int64_t c = 0;
    for (int64_t s = 0; s < cnt; ++s) {
        if (partition != 0 && sub[s] != ph) continue;
        pI[c] = I[s]; pJ[c] = J[s]; pv[c] = val[s]; pw[c] = w[s];
        ++c;
    }
    return c;
}

/* Full WAltMin (Alg. 2).  partition 0 = REUSE_ALL (all of Ω in */
/* every phase, as the deployed ALS; R11), 1 = FRESH_2T1    */
/* (line 3: Ω_0 for the init, Ω_{2t+1} / Ω_{2t+2} for iteration t):          */
/*   w = 1/q̂ (line 2); R = w .* P_Ω0(M̃) (line 4);                          */
/*   U0 = top-r left singular subspace of R by subspace iteration from a     */
/*        Rademacher start (line 5; R12), init_iters iterations;    */
/*   trim rows of U0 with norm > trim_c sqrt(r) ||A_i||/||A||_F (line 6,     */
/*        P:237; R13), re-orthonormalise;                          */
/*   T x { V = argmin on Ω_{2t+1} (line 8); U = argmin on Ω_{2t+2} (l. 9) }. */
void or_waltmin(int64_t n1, int64_t n2, int r, int T, int init_iters, double trim_c,
                double lam, uint64_t seed, int partition, int64_t cnt, const int32_t *I,
                const int32_t *J, const double *val, const double *qhat, const double *a_norm,
                double frobA, double *U, double *V)
{
    const size_t c1 = (size_t)(cnt > 0 ? cnt : 1);
    double *w = (double *)malloc(sizeof(double) * c1);
    for (int64_t s = 0; s < cnt; ++s) w[s] = qhat[s] > 0.0 ? 1.0 / qhat[s] : 0.0;
    int32_t *sub = (int32_t *)calloc(c1, sizeof(int32_t));
    if (partition != 0) or_partition(seed, 2 * T + 1, cnt, I, J, sub);
    int32_t *pI = (int32_t *)malloc(sizeof(int32_t) * c1), *pJ = (int32_t *)malloc(sizeof(int32_t) * c1);
    double *pv = (double *)malloc(sizeof(double) * c1), *pw = (double *)malloc(sizeof(double) * c1);
    double *Y = (double *)calloc((size_t)n2 * r, sizeof(double));
    double *Z = (double *)calloc((size_t)n1 * r, sizeof(double));
    /* Y0[j][l] = ±1 from Philox(ctr=(j,l,0,5), key=seed), bit 0 of word 0 */
    for (int64_t j = 0; j < n2; ++j)
        for (int l = 0; l < r; ++l) {
            uint32_t o[4];
            philox_seed(seed, (uint32_t)j, (uint32_t)l, 0u, 5u, o);
            Y[j * r + l] = (o[0] & 1u) ? -1.0 : 1.0;
        }
    int64_t pc = phase_samples(partition, 0, cnt, sub, I, J, val, w, pI, pJ, pv, pw);
    for (int it = 0; it < init_iters; ++it) {
        for (int64_t i = 0; i < n1 * r; ++i) Z[i] = 0.0;
        for (int64_t s = 0; s < pc; ++s)
            for (int l = 0; l < r; ++l) Z[(int64_t)pI[s] * r + l] += pw[s] * pv[s] * Y[(int64_t)pJ[s] * r + l];
        householder_q(n1, r, Z);
        for (int64_t j = 0; j < n2 * r; ++j) Y[j] = 0.0;
        for (int64_t s = 0; s < pc; ++s)
            for (int l = 0; l < r; ++l) Y[(int64_t)pJ[s] * r + l] += pw[s] * pv[s] * Z[(int64_t)pI[s] * r + l];
        householder_q(n2, r, Y);
    }
    /* trim */
    if (trim_c > 0.0 && frobA > 0.0) {
        for (int64_t i = 0; i < n1; ++i) {
            double rn = 0.0;
            for (int l = 0; l < r; ++l) rn += Z[i * r + l] * Z[i * r + l];
            rn = sqrt(rn);
            double thr = trim_c * sqrt((double)r) * a_norm[i] / frobA;
            if (rn > thr)
                for (int l = 0; l < r; ++l) Z[i * r + l] = 0.0;
        }
        householder_q(n1, r, Z);
    }
    memcpy(U, Z, sizeof(double) * (size_t)n1 * r);
    if (T == 0)
        for (int64_t j = 0; j < n2 * r; ++j) V[j] = 0.0;
    for (int t = 0; t < T; ++t) {
        pc = phase_samples(partition, 2 * t + 1, cnt, sub, I, J, val, w, pI, pJ, pv, pw);
        or_als_half(r, n2, pc, pJ, pI, pv, pw, U, lam, V);
        pc = phase_samples(partition, 2 * t + 2, cnt, sub, I, J, val, w, pI, pJ, pv, pw);
        or_als_half(r, n1, pc, pI, pJ, pv, pw, V, lam, U);
    }
    free(w); free(sub); free(pI); free(pJ); free(pv); free(pw); free(Y); free(Z);
}

/* ------------------------------------------------------------------------ */
/* LELA (Bhojanapalli et al.; the paper's two-pass comparison system,  */
/* P:145, Table 1): pass 1 = the column  */
/* norms (or_colnorms), Ω from the same Eq. 1 (or_sample); pass 2 computes   */
/* the EXACT entries of AᵀB on Ω ("needs a second pass to compute the  */
/* sampled entries"):  out[s] += Σ_t A[t, I_s] · B[t, J_s]  (fp64), over the  */
/* rows of the block; then WAltMin on (Ω, exact entries, q̂) (or_waltmin).   */
/* ------------------------------------------------------------------------ */
void or_exact_entries(int64_t rows, const void *A, int adtype, int64_t lda, const void *B, int bdtype,
                      int64_t ldb, int64_t cnt, const int32_t *I, const int32_t *J, double *out)
{
    #pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < cnt; ++s) {
        double acc = out[s];
        for (int64_t t = 0; t < rows; ++t)
            acc += load_elem(A, adtype, t * lda + I[s]) * load_elem(B, bdtype, t * ldb + J[s]);
        out[s] = acc;
    }
}

/* Threads the oracle's OpenMP loops use (reported as the CPU baseline's cores). */
#ifdef _OPENMP
#include <omp.h>
int or_num_threads(void) { return omp_get_max_threads(); }
#else
int or_num_threads(void) { return 1; }
#endif
