"""Pins for the CPU oracle (oracle/): each test checks an oracle function
against something other than itself — a library routine, a closed form, an
invariant of the paper, brute force, or a printed value of the paper.

Citations: "P:L" = PAPER.md line L (section/equation named inline).
"""
import json
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest
import scipy.linalg
import scipy.stats

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- H: Philox
def test_philox_random123_kat(golden_dir):
    """Published Random123 known-answer vectors (tests/golden, cited)."""
    with open(os.path.join(golden_dir, "philox4x32_10_kat.txt")) as f:
        rows = [ln.split() for ln in f if ln.strip() and not ln.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        words = [int(x, 16) for x in r[2:]]
        out = oracle.philox4x32_10(words[0:4], words[4:6])
        assert [int(x) for x in out] == words[6:10]


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_philox_vs_curand_host():
    """The CUDA toolkit's curand_Philox4x32_10 (a library routine), run on the
    host, agrees with the oracle on 2000 random (ctr, key) pairs."""
    src = os.path.join(ROOT, "tests", "helpers", "curand_philox_kat.cu")
    rng = np.random.default_rng(123)
    words = rng.integers(0, 2**32, size=(2000, 6), dtype=np.uint64)
    with tempfile.TemporaryDirectory() as td:
        exe = os.path.join(td, "kat")
        subprocess.check_call(["nvcc", "-O1", "-Wno-deprecated-gpu-targets", "-o", exe, src])
        inp = "\n".join(" ".join("%x" % int(x) for x in row) for row in words) + "\n"
        out = subprocess.run([exe], input=inp, capture_output=True, text=True, check=True).stdout
    got = [[int(x, 16) for x in ln.split()] for ln in out.strip().splitlines()]
    for row, ref in zip(words, got):
        mine = oracle.philox4x32_10(row[:4], row[4:6])
        assert [int(x) for x in mine] == ref


# ---------------------------------------------------------------- Π
def test_rademacher_values_and_balance():
    k, d = 64, 4096
    P = oracle.pi_matrix(oracle.PI_RADEMACHER, 7, k, 0, d)
    assert set(np.unique(P)) <= {-1.0, 1.0}
    # binomial balance test (two-sided, alpha = 1e-4)
    n_neg = int((P < 0).sum())
    pval = scipy.stats.binomtest(n_neg, P.size, 0.5).pvalue
    assert pval > 1e-4
    # independence across rows/cols: correlation of adjacent entries ~ 0
    c1 = np.mean(P[:, 1:] * P[:, :-1])
    c2 = np.mean(P[1:, :] * P[:-1, :])
    assert abs(c1) < 5 / math.sqrt(P.size) and abs(c2) < 5 / math.sqrt(P.size)


def test_rademacher_counter_layout():
    """row t's sign is bit (e>>1) + 16(e&1), e = t & 31, of word
    (t & 127) >> 5 of Philox(ctr=(t>>7, κ, t>>39, 1))."""
    seed = 0x1234_5678_9ABC
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for kappa, t in [(0, 0), (3, 127), (200, 128), (17, 1000003), (5, 2**33 + 77)]:
        w = oracle.philox4x32_10([(t >> 7) & 0xFFFFFFFF, kappa, (t >> 39) & 0xFFFFFFFF, 1], key)
        b = t & 127
        e = b & 31
        bit = (int(w[b >> 5]) >> ((e >> 1) + 16 * (e & 1))) & 1
        assert oracle.pi_entry(oracle.PI_RADEMACHER, seed, kappa, t) == (-1.0 if bit else 1.0)


def _bf16_round(x):
    """Independent fp64 -> bf16 (round to nearest even) via float32 bits."""
    f = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    lsb = (f >> 16) & 1
    f = ((f + 0x7FFF + lsb) & 0xFFFF0000).astype(np.uint32)
    return f.view(np.float32).astype(np.float64)


def test_gaussian_matches_libm_box_muller():
    """G is a polynomial Box–Muller: compare to fp64 libm
    Box–Muller on the same Philox words; at most 1 bf16 ulp apart."""
    seed = 99
    key = [seed, 0]
    errs = 0
    n = 0
    for kappa in range(8):
        for tq in range(0, 400):
            w = [int(x) for x in oracle.philox4x32_10([tq, kappa, 0, 2], key)]
            for p in range(2):
                wa, wb = w[2 * p], w[2 * p + 1]
                u1 = ((wa >> 8) + 1) * 2.0**-24
                u2 = (wb >> 8) * 2.0**-24
                rho = math.sqrt(-2.0 * math.log(u1))
                zc, zs = rho * math.cos(2 * math.pi * u2), rho * math.sin(2 * math.pi * u2)
                g0 = oracle.pi_entry(oracle.PI_GAUSSIAN, seed, kappa, 4 * tq + 2 * p)
                g1 = oracle.pi_entry(oracle.PI_GAUSSIAN, seed, kappa, 4 * tq + 2 * p + 1)
                for g, z in ((g0, zc), (g1, zs)):
                    ulp = 2.0 ** (math.floor(math.log2(max(abs(z), 1e-30))) - 7)
                    n += 1
                    if abs(g - z) > ulp * 1.0001:
                        errs += 1
    assert n == 8 * 400 * 4
    assert errs == 0


def test_gaussian_distribution():
    """Mean 0, variance 1 (unscaled), KS vs N(0,1) over 2e5 draws."""
    k, d = 50, 4000
    P = oracle.pi_matrix(oracle.PI_GAUSSIAN, 3, k, 0, d).ravel()
    assert abs(P.mean()) < 5 / math.sqrt(P.size)
    assert abs(P.var() - 1.0) < 0.02
    # bf16 quantisation perturbs values by <= 2^-9 relative; KS still passes
    assert scipy.stats.kstest(P, "norm").pvalue > 1e-4
    # bf16-valued
    assert np.array_equal(_bf16_round(P), P)


def test_hadamard_is_sylvester():
    """Π(κ,t) = (-1)^popcount(κ & t) equals scipy's Sylvester Hadamard matrix."""
    d = 64
    P = oracle.pi_matrix(oracle.PI_HADAMARD, 0, d, 0, d)
    assert np.array_equal(P, scipy.linalg.hadamard(d).astype(np.float64))


def test_jl_norm_band():
    """Lemma randomJLT / S:150: ||Πx||^2 within 1 ± 0.5 for >= 99% of
    unit vectors at k=200, d=2000 (Rademacher and Gaussian)."""
    rng = np.random.default_rng(5)
    d, k, nv = 2000, 200, 200
    X = rng.standard_normal((d, nv))
    X /= np.linalg.norm(X, axis=0)
    for kind in (oracle.PI_RADEMACHER, oracle.PI_GAUSSIAN):
        sk, _ = oracle.sketch_rows(kind, 11, k, X)
        out, sknorm, _ = oracle.finalize(k, sk, np.ones(nv))
        frac = np.mean(np.abs(sknorm**2 - 1.0) <= 0.5)
        assert frac >= 0.99


# ---------------------------------------------------------------- Step 1
@pytest.mark.parametrize("kind", [oracle.PI_RADEMACHER, oracle.PI_GAUSSIAN])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_sketch_bruteforce(kind, dtype):
    """Brute force: materialised Π @ X and (X**2).sum(0)."""
    rng = np.random.default_rng(0)
    d, n, k = 300, 17, 24
    X = rng.standard_normal((d, n)).astype(dtype)
    sk, n2 = oracle.sketch_rows(kind, 5, k, X, row0=1000)
    P = oracle.pi_matrix(kind, 5, k, 1000, d)
    ref = (P @ X.astype(np.float64)).T
    np.testing.assert_allclose(sk, ref, rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(n2, (X.astype(np.float64) ** 2).sum(0), rtol=1e-13)


def test_sketch_bf16_input():
    rng = np.random.default_rng(1)
    d, n, k = 200, 9, 16
    X32 = rng.standard_normal((d, n)).astype(np.float32)
    bits = X32.view(np.uint32) >> 16  # truncation to bf16 bits (any bf16 value works)
    Xbf = bits.astype(np.uint16)
    Xval = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    sk, n2 = oracle.sketch_rows(oracle.PI_RADEMACHER, 2, k, Xbf)
    P = oracle.pi_matrix(oracle.PI_RADEMACHER, 2, k, 0, d)
    np.testing.assert_allclose(sk, (P @ Xval).T, rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(n2, (Xval**2).sum(0), rtol=1e-13)


def test_sketch_order_and_shard_invariance():
    """One pass in arbitrary block order and merge of shards:
    the sum over row blocks equals the whole (exactly up to fp64 rounding)."""
    rng = np.random.default_rng(2)
    d, n, k = 512, 11, 32
    X = rng.standard_normal((d, n))
    whole, wn = oracle.sketch_rows(oracle.PI_RADEMACHER, 9, k, X)
    sk = np.zeros((n, k))
    nn = np.zeros(n)
    for b in [3, 0, 2, 1]:
        oracle.sketch_rows(oracle.PI_RADEMACHER, 9, k, X[b * 128:(b + 1) * 128], row0=b * 128,
                           sk=sk, norm2=nn)
    np.testing.assert_allclose(sk, whole, rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(nn, wn, rtol=1e-13)


def test_sketch_cols_matches_rows():
    rng = np.random.default_rng(3)
    X = rng.standard_normal((400, 30))
    full, fn = oracle.sketch_rows(oracle.PI_GAUSSIAN, 4, 20, X, row0=77)
    cols = np.array([0, 5, 29, 13])
    sub, sn = oracle.sketch_cols(oracle.PI_GAUSSIAN, 4, 20, X, cols, row0=77)
    np.testing.assert_allclose(sub, full[cols], rtol=1e-12, atol=1e-11)
    np.testing.assert_allclose(sn, fn[cols], rtol=1e-13)


def test_sketch_csr_matches_dense():
    rng = np.random.default_rng(4)
    d, n, k = 150, 40, 16
    D = rng.poisson(0.3, size=(d, n)).astype(np.float32)
    rowptr = np.concatenate([[0], np.cumsum((D != 0).sum(1))]).astype(np.int64)
    col = np.concatenate([np.nonzero(D[t])[0] for t in range(d)]).astype(np.int32)
    val = np.concatenate([D[t][D[t] != 0] for t in range(d)]).astype(np.float32)
    sk, n2 = oracle.sketch_csr(oracle.PI_GAUSSIAN, 8, k, n, rowptr, col, val, row0=10)
    ref, rn = oracle.sketch_rows(oracle.PI_GAUSSIAN, 8, k, D, row0=10)
    np.testing.assert_allclose(sk, ref, rtol=1e-12, atol=1e-11)
    assert np.array_equal(n2, rn)  # integer counts: exact
    # a block whose rowptr does not start at 0 (col/val indexed from rowptr[0])
    a, b = 37, 121
    sk2, n22 = oracle.sketch_csr(oracle.PI_GAUSSIAN, 8, k, n, rowptr[a:b + 1], col[rowptr[a]:],
                                 val[rowptr[a]:], row0=10 + a)
    ref2, rn2 = oracle.sketch_rows(oracle.PI_GAUSSIAN, 8, k, D[a:b], row0=10 + a)
    np.testing.assert_allclose(sk2, ref2, rtol=1e-12, atol=1e-11)
    assert np.array_equal(n22, rn2)


def test_colnorms_closed_form():
    """Σ_t X[t,c]² against its definition (numpy fp64), bf16/fp32/fp64 inputs."""
    rng = np.random.default_rng(9)
    X = (rng.standard_normal((513, 37)) * np.exp(rng.uniform(-5, 5, 37))).astype(np.float32)
    np.testing.assert_allclose(oracle.colnorms(X), (X.astype(np.float64) ** 2).sum(0), rtol=1e-13)
    Xd = X.astype(np.float64)
    np.testing.assert_allclose(oracle.colnorms(Xd), (Xd ** 2).sum(0), rtol=1e-13)
    bits = (X.view(np.uint32) >> 16).astype(np.uint16)
    Xb = (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    np.testing.assert_allclose(oracle.colnorms(bits), (Xb ** 2).sum(0), rtol=1e-13)
    # equals the norm half of the one-pass sketch
    _, n2 = oracle.sketch_rows(oracle.PI_RADEMACHER, 1, 8, X)
    np.testing.assert_allclose(oracle.colnorms(X), n2, rtol=1e-13)


def test_pairwise_sum_exact_cases():
    """R5 tree: exact on integers, equals math.fsum on benign data."""
    x = np.arange(1, 1001, dtype=np.float64)
    assert oracle.pairwise_sum(x) == 500500.0
    assert oracle.pairwise_sum(np.array([])) == 0.0
    rng = np.random.default_rng(0)
    y = rng.random(777)
    assert abs(oracle.pairwise_sum(y) - math.fsum(y)) <= 1e-12 * math.fsum(y)


# ---------------------------------------------------------------- Eq. 2 closed forms
def test_hadamard_kd_gives_exact_product():
    """North star (a): k = d and Π orthonormal (Sylvester-Hadamard / sqrt(k)) =>
    ÃᵀB̃ = AᵀB, ||Ã_i|| = ||A_i||, hence M̃ = AᵀB exactly (Eq. 2)."""
    rng = np.random.default_rng(6)
    d = 64
    A = rng.standard_normal((d, 12))
    B = rng.standard_normal((d, 9))
    skA, a2 = oracle.sketch_rows(oracle.PI_HADAMARD, 0, d, A)
    skB, b2 = oracle.sketch_rows(oracle.PI_HADAMARD, 0, d, B)
    As, asn, DA = oracle.finalize(d, skA, a2)
    Bs, bsn, DB = oracle.finalize(d, skB, b2)
    np.testing.assert_allclose(asn, np.sqrt(a2), rtol=1e-12)
    np.testing.assert_allclose(DA, 1.0, rtol=1e-12)
    I, J = np.meshgrid(np.arange(12), np.arange(9), indexing="ij")
    Mt = oracle.estimate(d, I.ravel(), J.ravel(), As, Bs, DA, DB)
    np.testing.assert_allclose(Mt.reshape(12, 9), A.T @ B, rtol=1e-10, atol=1e-10)


def test_a_equals_b_diagonal():
    """North star (b) / S:202: A = B => M̃_ii = ||A_i||^2 for any Π."""
    rng = np.random.default_rng(7)
    A = rng.standard_normal((300, 15)) * rng.uniform(0.1, 10, 15)
    sk, a2 = oracle.sketch_rows(oracle.PI_RADEMACHER, 3, 16, A)
    As, _, DA = oracle.finalize(16, sk, a2)
    idx = np.arange(15)
    Mt = oracle.estimate(16, idx, idx, As, As, DA, DA)
    np.testing.assert_allclose(Mt, (A**2).sum(0), rtol=1e-12)


def test_fig2a_mse(golden_dir):
    """Fig. 2a: rescaled-JL MSE 0.053 vs JL MSE 0.129 at d=1000,
    k=10; closed forms (8/15)/k and (4/3)/k for cos ~ U[-1,1] (R24)."""
    g = json.load(open(os.path.join(golden_dir, "fig2a_mse.json")))
    d, k, npairs = g["d"], g["k"], 4000
    rng = np.random.default_rng(8)
    c = rng.uniform(-1, 1, npairs)
    a = rng.standard_normal((d, npairs))
    a /= np.linalg.norm(a, axis=0)
    p = rng.standard_normal((d, npairs))
    p -= a * (a * p).sum(0)
    p /= np.linalg.norm(p, axis=0)
    b = c * a + np.sqrt(1 - c**2) * p
    mse_r, mse_j = [], []
    for s in range(3):  # three independent Π
        skA, a2 = oracle.sketch_rows(oracle.PI_GAUSSIAN, 100 + s, k, a)
        skB, b2 = oracle.sketch_rows(oracle.PI_GAUSSIAN, 100 + s, k, b)
        As, _, DA = oracle.finalize(k, skA, a2)
        Bs, _, DB = oracle.finalize(k, skB, b2)
        idx = np.arange(npairs)
        mr = oracle.estimate(k, idx, idx, As, Bs, DA, DB)
        mj = oracle.estimate(k, idx, idx, As, Bs, DA, DB, plain=True)
        mse_r.append(np.mean((mr - c) ** 2))
        mse_j.append(np.mean((mj - c) ** 2))
    mr, mj = np.mean(mse_r), np.mean(mse_j)
    assert mr < mj
    assert abs(mj - g["mse_jl"]) / g["mse_jl"] < 0.15
    assert abs(mr - g["mse_rescaled_jl"]) / g["mse_rescaled_jl"] < 0.2
    assert abs(mj - (4 / 3) / k) / ((4 / 3) / k) < 0.15


def test_lemma_jl_scaling():
    """Lemma JL: max |M̃_ij - A_iᵀB_j| / (||A_i|| ||B_j||) shrinks
    like 1/sqrt(k): quadrupling k roughly halves it."""
    rng = np.random.default_rng(9)
    A = rng.standard_normal((1024, 20))
    B = A[:, :20] + 0.5 * rng.standard_normal((1024, 20))
    exact = A.T @ B
    scale = np.outer(np.linalg.norm(A, axis=0), np.linalg.norm(B, axis=0))
    I, J = np.meshgrid(np.arange(20), np.arange(20), indexing="ij")
    errs = []
    for k in (64, 256, 1024):
        e = []
        for s in range(4):
            skA, a2 = oracle.sketch_rows(oracle.PI_RADEMACHER, 50 + s, k, A)
            skB, b2 = oracle.sketch_rows(oracle.PI_RADEMACHER, 50 + s, k, B)
            As, _, DA = oracle.finalize(k, skA, a2)
            Bs, _, DB = oracle.finalize(k, skB, b2)
            Mt = oracle.estimate(k, I.ravel(), J.ravel(), As, Bs, DA, DB).reshape(20, 20)
            e.append(np.sqrt(np.mean(((Mt - exact) / scale) ** 2)))
        errs.append(np.mean(e))
    assert 1.4 < errs[0] / errs[1] < 2.8
    assert 1.4 < errs[1] / errs[2] < 2.8


# ---------------------------------------------------------------- Eq. 1
def test_q_sums_to_m():
    """sum_ij q_ij = m when no entry saturates (Eq. 1 identity)."""
    rng = np.random.default_rng(10)
    a2 = rng.uniform(0.5, 2, 37)
    b2 = rng.uniform(0.5, 2, 23)
    FA, FB = oracle.pairwise_sum(a2), oracle.pairwise_sum(b2)
    al, be = oracle.alpha_beta(a2, b2, FA, FB)
    m = 50.0
    total = math.fsum(oracle.qhat(m, x, y) for x in al for y in be)
    assert abs(total - m) < 1e-9 * m


def test_q_uniform_and_single_column():
    """equal norms => q = m/n^2; single nonzero A column i0 =>
    q_{i0 j} = m(1/(2 n2) + b2_j/(2 n1 FB)), other rows m b2_j/(2 n1 FB)."""
    n = 8
    al, be = oracle.alpha_beta(np.ones(n), np.ones(n), float(n), float(n))
    assert all(abs(oracle.qhat(3.0, a, b) - 3.0 / n**2) < 1e-15 for a in al for b in be)
    a2 = np.zeros(5)
    a2[2] = 4.0
    b2 = np.array([1.0, 2.0, 3.0, 4.0])
    FA, FB = 4.0, 10.0
    al, be = oracle.alpha_beta(a2, b2, FA, FB)
    m = 2.0
    for j in range(4):
        assert abs(oracle.qhat(m, al[2], be[j]) - m * (1 / 8 + b2[j] / (2 * 5 * FB))) < 1e-15
        assert abs(oracle.qhat(m, al[0], be[j]) - m * b2[j] / (2 * 5 * FB)) < 1e-15


def test_omega_saturation_and_empty():
    al, be = oracle.alpha_beta(np.ones(6), np.ones(5), 6.0, 5.0)
    I, J, q = oracle.sample(0, 1e9, al, be)
    assert len(I) == 30 and np.all(q == 1.0)
    assert list(zip(I, J)) == [(i, j) for i in range(6) for j in range(5)]
    I, J, q = oracle.sample(0, 0.0, al, be)
    assert len(I) == 0


def test_omega_inclusion_chi2():
    """per-entry inclusion frequencies over independent seeds match q̂
    (chi-squared, alpha = 1e-3)."""
    rng = np.random.default_rng(11)
    a2 = rng.uniform(0.2, 3, 10)
    b2 = rng.uniform(0.2, 3, 8)
    al, be = oracle.alpha_beta(a2, b2, oracle.pairwise_sum(a2), oracle.pairwise_sum(b2))
    m = 30.0
    trials = 3000
    counts = np.zeros((10, 8))
    for s in range(trials):
        I, J, _ = oracle.sample(1000 + s, m, al, be)
        np.add.at(counts, (I, J), 1)
    q = np.array([[oracle.qhat(m, x, y) for y in be] for x in al])
    exp = q * trials
    chi2 = np.sum((counts - exp) ** 2 / (exp * (1 - q)))
    assert scipy.stats.chi2.sf(chi2, df=80) > 1e-3


def test_omega_sorted_and_draw_definition():
    rng = np.random.default_rng(12)
    a2 = rng.uniform(0.2, 3, 30)
    b2 = rng.uniform(0.2, 3, 40)
    FA, FB = oracle.pairwise_sum(a2), oracle.pairwise_sum(b2)
    al, be = oracle.alpha_beta(a2, b2, FA, FB)
    I, J, q = oracle.sample(77, 200.0, al, be)
    keys = I.astype(np.int64) * 40 + J
    assert np.all(np.diff(keys) > 0)
    # U53 from Philox(ctr=(i,j,0,3), key=seed) < q̂
    for i, j in [(0, 0), (3, 7), (29, 39)]:
        w = oracle.philox4x32_10([i, j, 0, 3], [77, 0])
        u = ((int(w[1]) << 32 | int(w[0])) >> 11) * 2.0**-53
        qq = oracle.qhat(200.0, al[i], be[j])
        inc = any(ii == i and jj == j for ii, jj in zip(I, J))
        assert inc == (u < qq)


# ---------------------------------------------------------------- WAltMin (Alg. 2)
def test_als_half_bruteforce():
    """Alg. 2 line 8 closed form: per-column weighted least squares
    equals numpy lstsq on sqrt(w)-scaled rows (λ -> 0)."""
    rng = np.random.default_rng(13)
    n1, n2, r = 30, 25, 3
    U = rng.standard_normal((n1, r))
    mask = rng.random((n1, n2)) < 0.4
    I, J = np.nonzero(mask)
    val = rng.standard_normal(len(I))
    w = rng.uniform(0.5, 3, len(I))
    V = oracle.als_half(r, n2, J, I, val, w, U, lam=0.0)
    for j in range(n2):
        sel = J == j
        if sel.sum() == 0:
            assert np.all(V[j] == 0)
            continue
        sw = np.sqrt(w[sel])
        ref, *_ = np.linalg.lstsq(U[I[sel]] * sw[:, None], val[sel] * sw, rcond=None)
        np.testing.assert_allclose(V[j], ref, rtol=1e-8, atol=1e-10)


def test_waltmin_full_observation_exact_rank():
    """fully observed (q̂ = 1), exact rank r => UVᵀ = M."""
    rng = np.random.default_rng(14)
    n1, n2, r = 40, 30, 4
    M = rng.standard_normal((n1, r)) @ rng.standard_normal((r, n2))
    I, J = np.meshgrid(np.arange(n1), np.arange(n2), indexing="ij")
    I, J = I.ravel().astype(np.int32), J.ravel().astype(np.int32)
    U, V = oracle.waltmin(n1, n2, r, 5, I, J, M.ravel(), np.ones(len(I)),
                          np.ones(n1), 1.0, trim_c=0.0)
    np.testing.assert_allclose(U @ V.T, M, rtol=1e-8, atol=1e-8 * np.abs(M).max())


def test_waltmin_init_matches_svd():
    """Alg. 2 line 5: subspace iteration gives the top-r left singular subspace
    of R_Ω (materialised densely; LAPACK SVD), principal angles ~ 0."""
    rng = np.random.default_rng(15)
    n1, n2, r = 40, 30, 3
    L = rng.standard_normal((n1, r)) * [10, 6, 3] @ rng.standard_normal((r, n2))
    M = L + 0.05 * rng.standard_normal((n1, n2))
    mask = rng.random((n1, n2)) < 0.5
    I, J = np.nonzero(mask)
    q = np.full(len(I), 0.5)
    # T = 0: output U is the trimmed init (trim disabled)
    U, _ = oracle.waltmin(n1, n2, r, 0, I, J, M[I, J], q, np.ones(n1), 1.0, init_iters=200,
                          trim_c=0.0)
    R = np.zeros((n1, n2))
    R[I, J] = M[I, J] / 0.5
    Us = np.linalg.svd(R)[0][:, :r]
    s = np.linalg.svd(Us.T @ U, compute_uv=False)
    assert np.all(s > 1 - 1e-8)
    np.testing.assert_allclose(U.T @ U, np.eye(r), atol=1e-10)


def test_waltmin_trim():
    """Alg. 2 line 6 / P:237: rows of U0 with norm above c sqrt(r)||A_i||/||A||_F
    are zeroed.  A spiked row of R with tiny ||A_i|| is removed."""
    rng = np.random.default_rng(16)
    n1, n2, r = 30, 20, 2
    M = rng.standard_normal((n1, r)) @ rng.standard_normal((r, n2))
    M[5] *= 50.0
    I, J = np.meshgrid(np.arange(n1), np.arange(n2), indexing="ij")
    I, J = I.ravel(), J.ravel()
    a_norm = np.ones(n1)
    a_norm[5] = 1e-6
    frob = float(np.sqrt((a_norm**2).sum()))
    U, _ = oracle.waltmin(n1, n2, r, 0, I, J, M[I, J], np.ones(len(I)), a_norm, frob,
                          init_iters=30, trim_c=1.0)
    assert np.all(U[5] == 0)
    thr = 1.0 * math.sqrt(r) * a_norm / frob
    np.testing.assert_allclose(U.T @ U, np.eye(r), atol=1e-10)
    assert np.sum(np.linalg.norm(U, axis=1) > thr + 1e-9) <= n1  # post-check is informative


def test_waltmin_objective_nonincreasing():
    """Eq. 3's objective does not increase across half-steps (REUSE_ALL)."""
    rng = np.random.default_rng(17)
    n1, n2, r = 30, 25, 3
    M = rng.standard_normal((n1, r)) @ rng.standard_normal((r, n2)) + 0.3 * rng.standard_normal((n1, n2))
    mask = rng.random((n1, n2)) < 0.5
    I, J = np.nonzero(mask)
    val = M[I, J]
    w = rng.uniform(1, 3, len(I))
    U = rng.standard_normal((n1, r))
    obj = lambda U, V: float(np.sum(w * (np.sum(U[I] * V[J], 1) - val) ** 2))
    V = oracle.als_half(r, n2, J, I, val, w, U, lam=0.0)
    prev = obj(U, V)
    for _ in range(5):
        U = oracle.als_half(r, n1, I, J, val, w, V, lam=0.0)
        cur = obj(U, V)
        assert cur <= prev * (1 + 1e-12)
        prev = cur
        V = oracle.als_half(r, n2, J, I, val, w, U, lam=0.0)
        cur = obj(U, V)
        assert cur <= prev * (1 + 1e-12)
        prev = cur


def test_phase_transition():
    """Fig. 4a / P:160: error at m = 6 n r ln n is >= 10x below the error at
    m = 0.5 n r ln n (exact rank-r product, exact entries)."""
    rng = np.random.default_rng(18)
    n, r = 150, 3
    Ut = rng.standard_normal((n, r))
    Vt = rng.standard_normal((n, r))
    M = Ut @ Vt.T
    a2 = np.ones(n)
    al, be = oracle.alpha_beta(a2, a2, float(n), float(n))

    def err(m):
        I, J, q = oracle.sample(5, m, al, be)
        U, V = oracle.waltmin(n, n, r, 10, I, J, M[I, J], q, np.ones(n), math.sqrt(n),
                              init_iters=50)
        return np.linalg.norm(U @ V.T - M, 2) / np.linalg.norm(M, 2)

    lo = err(0.5 * n * r * math.log(n))
    hi = err(6 * n * r * math.log(n))
    assert hi < 1e-3 and lo > 10 * hi


def test_pipeline_hadamard_saturated_exact_rank():
    """Whole Alg. 1 closed form: Hadamard Π (k = d), saturated sampling
    (q̂ = 1) and exact-rank AᵀB => ÛV̂ᵀ = AᵀB."""
    rng = np.random.default_rng(19)
    d, n, r = 64, 12, 3
    Z = rng.standard_normal((d, r))
    A = Z @ rng.standard_normal((r, n))
    B = Z @ rng.standard_normal((r, n)) + 0.0
    res = oracle.smp_pca(A, B, k=d, r=r, m=1e12, T=5, pi_kind=oracle.PI_HADAMARD, trim_c=0.0)
    assert len(res["I"]) == n * n
    np.testing.assert_allclose(res["U"] @ res["V"].T, A.T @ B, rtol=1e-7,
                               atol=1e-7 * np.abs(A.T @ B).max())


def test_pipeline_error_reported_vs_optimal():
    """Theorem 1 has unspecified constants, so the guarantee is
    checked as: on a tiny shared-axis cone instance above the phase transition,
    SMP-PCA's spectral error is within a small factor of ||M̃ - AᵀB|| plus the
    optimal rank-r error, and beats SVD(ÃᵀB̃)."""
    rng = np.random.default_rng(20)
    d, n, r, k = 2000, 60, 3, 256
    x = rng.standard_normal(d)
    x /= np.linalg.norm(x)

    def cone(m, theta):
        t = rng.standard_normal((d, m)) * (math.tan(theta / 2) / math.sqrt(d))
        y = x[:, None] + t
        y *= rng.choice([-1, 1], m)
        return y / np.linalg.norm(y, axis=0)

    A, B = cone(n, 0.3), cone(n, 0.3)
    M = A.T @ B
    m = 6 * n * r * math.log(n)
    res = oracle.smp_pca(A, B, k=k, r=r, m=m, T=10, pi_kind=oracle.PI_GAUSSIAN, seed=3)
    nrm = np.linalg.norm(M, 2)
    err = np.linalg.norm(res["U"] @ res["V"].T - M, 2) / nrm
    s = np.linalg.svd(M, compute_uv=False)
    opt = s[r] / nrm
    Ms = res["Ask"] @ res["Bsk"].T
    u, sv, vt = np.linalg.svd(Ms)
    err_svd = np.linalg.norm((u[:, :r] * sv[:r]) @ vt[:r] - M, 2) / nrm
    assert err <= err_svd
    assert err < 0.1
    assert opt <= err + 1e-12


# ------------------------------------------------------------------ SRHT (NEXT-1, R26)
def test_srht_feistel_is_a_bijection():
    """F_L permutes [0, 2^L): the k sampled Hadamard rows are distinct
    (sampling without replacement, the S of S·H·D)."""
    for L in (1, 2, 3, 5, 8, 11):
        rows = [oracle.srht_row(7, L, i) for i in range(1 << L)]
        assert sorted(rows) == list(range(1 << L)), L


def test_srht_sign_layout_and_balance():
    """D_t from raw Philox words of stream 6 (the Rademacher bit layout)."""
    seed = 0x1234
    for t in (0, 1, 2, 31, 32, 127, 128, 1000, (1 << 40) + 77):
        w = oracle.philox4x32_10([(t >> 7) & 0xFFFFFFFF, 0, (t >> 39) & 0xFFFFFFFF, 6],
                                 [seed & 0xFFFFFFFF, seed >> 32])
        b = t & 127
        e = b & 31
        bit = (int(w[b >> 5]) >> ((e >> 1) + ((e & 1) << 4))) & 1
        assert oracle.srht_sign(seed, t) == (-1.0 if bit else 1.0)
    s = np.array([oracle.srht_sign(3, t) for t in range(20000)])
    assert abs(s.mean()) < 4.5 / np.sqrt(len(s))


def test_srht_entries_are_signed_hadamard():
    d = 1000
    kind = oracle.pi_srht(d)
    L = kind - 16
    assert (1 << L) >= d > (1 << (L - 1))
    H = scipy.linalg.hadamard(1 << L)
    for kap in (0, 3, 17):
        s = oracle.srht_row(5, L, kap)
        for t in (0, 1, 77, 999):
            assert oracle.pi_entry(kind, 5, kap, t) == oracle.srht_sign(5, t) * H[s, t]


def test_srht_full_rank_gives_exact_product():
    """k = d = 2^L: Π is a row-permuted, column-signed Hadamard matrix, so
    ΠᵀΠ = d I and the (1/√k-scaled) sketch preserves all inner products:
    M̃ = AᵀB exactly (the SRHT analogue of north-star check (a))."""
    d, n = 256, 12
    kind = oracle.pi_srht(d)
    rng = np.random.default_rng(2)
    A = rng.standard_normal((d, n))
    B = rng.standard_normal((d, n))
    P = oracle.pi_matrix(kind, 9, d, 0, d)
    np.testing.assert_allclose(P.T @ P, d * np.eye(d), atol=1e-9)
    skA, a2 = oracle.sketch_rows(kind, 9, d, A)
    skB, b2 = oracle.sketch_rows(kind, 9, d, B)
    As, _, DA = oracle.finalize(d, skA, a2)
    Bs, _, DB = oracle.finalize(d, skB, b2)
    I, J = np.meshgrid(np.arange(n, dtype=np.int32), np.arange(n, dtype=np.int32), indexing="ij")
    M = oracle.estimate(d, I.ravel(), J.ravel(), As, Bs, DA, DB)
    np.testing.assert_allclose(M.reshape(n, n), A.T @ B, rtol=1e-9, atol=1e-9)


def test_srht_jl_band():
    """Subsampled at k < d, SRHT is still a JL map: ‖Πx‖²/k ≈ ‖x‖²."""
    d, k, trials = 2048, 256, 40
    kind = oracle.pi_srht(d)
    rng = np.random.default_rng(4)
    X = rng.standard_normal((d, trials))
    sk, n2 = oracle.sketch_rows(kind, 11, k, X)
    ratio = (sk ** 2).sum(1) / k / n2
    assert np.all(np.abs(ratio - 1) < 0.5) and abs(ratio.mean() - 1) < 0.1


# ------------------------------------------------------------------ row-multinomial Ω (NEXT-2, R27)
def _ab(n1, n2, seed):
    rng = np.random.default_rng(seed)
    a2 = rng.exponential(size=n1) ** 2
    b2 = rng.exponential(size=n2) ** 2
    return oracle.alpha_beta(a2, b2, oracle.pairwise_sum(a2), oracle.pairwise_sum(b2))


def _mn_ref_rows(m, al, be):
    """Brute force of R27's row quantities from their definitions: s_i =
    #{j : q_ij >= 1}, T_i = Σ_{j: q_ij < 1} (α_i + β_j)."""
    q = m * (al[:, None] + be[None, :])
    sat = q >= 1.0
    s = sat.sum(1)
    T = np.where(sat, 0.0, al[:, None] + be[None, :]).sum(1)
    return s, T, sat


def test_multinomial_row_counts_match_appendix():
    """Saturated prefix s_i and unsaturated mass T_i against brute force;
    E[M_i] = m T_i (the appendix's m_i on the unsaturated columns);
    Σ_i s_i + Σ_i m T_i = Σ_ij min(1, q_ij) (same expected size as Alg. 1's
    Bernoulli Ω before merging repeats)."""
    n1, n2, m = 40, 30, 500.0
    al, be = _ab(n1, n2, 1)
    s_ref, T_ref, sat = _mn_ref_rows(m, al, be)
    s, T = oracle.mn_rows(m, al, be)
    assert np.array_equal(s, s_ref) and s.max() > 0 and s.min() < n2
    np.testing.assert_allclose(T, T_ref, rtol=1e-12, atol=1e-15)
    q = m * (al[:, None] + be[None, :])
    assert abs(s.sum() + m * T.sum() - np.minimum(q, 1).sum()) < 1e-9 * m
    counts = np.zeros(n1)
    seeds = 400
    for sd in range(seeds):
        I, J = oracle.multinomial_draws(sd, m, al, be)
        counts += np.bincount(I, minlength=n1)
        assert np.all(np.diff(I) >= 0)
        same = I[1:] == I[:-1]
        assert np.all(J[1:][same] >= J[:-1][same])       # sorted by (i, j)
        assert not sat[I, J].any()                        # draws avoid saturated pairs
    est = counts / seeds
    # M_i = floor(m T_i + u): |mean - m T_i| within a few standard errors (var <= 1/4)
    assert np.all(np.abs(est - m * T) < 5 * 0.5 / np.sqrt(seeds) + 1e-12)


def test_multinomial_draws_follow_q_tilde():
    """Within a row, unsaturated columns are drawn ∝ α_i + β_j:
    expected count of (i, j) per draw-set = q_ij (unsaturated), 0 on
    saturated pairs; chi-squared over seeds."""
    n1, n2, m = 3, 25, 300.0
    al, be = _ab(n1, n2, 2)
    _, _, sat = _mn_ref_rows(m, al, be)
    assert sat.any() and not sat.all()
    freq = np.zeros((n1, n2))
    seeds = 200
    for sd in range(seeds):
        I, J = oracle.multinomial_draws(sd + 1000, m, al, be)
        np.add.at(freq, (I, J), 1)
    assert freq[sat].sum() == 0
    expect = seeds * m * (al[:, None] + be[None, :])
    u = ~sat
    chi2 = ((freq[u] - expect[u]) ** 2 / expect[u]).sum()
    dof = int(u.sum())
    assert chi2 < dof + 5 * np.sqrt(2 * dof)


def test_multinomial_inversion_matches_linear_search():
    """Draw d of row i is the first p >= s_i with C_i(p) > u T_i in the
    β-descending order σ, column σ(p) — recomputed here from raw Philox words
    and a linear scan of the same fp64 CDF values (the definition)."""
    n1, n2, m, seed = 6, 50, 300.0, 7
    al, be = _ab(n1, n2, 3)
    be[10] = be[11]                                  # a tie in σ (index order)
    I, J = oracle.multinomial_draws(seed, m, al, be)
    sig = np.lexsort((np.arange(n2), -be))
    bp = np.cumsum(be[sig])      # sequential fp64 sums, as the definition
    key = [seed & 0xFFFFFFFF, seed >> 32]
    s_ref, T_ref, _ = _mn_ref_rows(m, al, be)
    for i in range(n1):
        s = int(s_ref[i])
        base = bp[s - 1] if s > 0 else 0.0
        T = (n2 - s) * al[i] + (bp[-1] - base)
        w = oracle.philox4x32_10([i, 0, 0, 8], key)
        Mi = int(np.floor(m * T + ((int(w[1]) << 32 | int(w[0])) >> 11) * 2.0 ** -53)) if s < n2 else 0
        cols = []
        for d in range(Mi):
            w = oracle.philox4x32_10([i, d, 0, 9], key)
            target = ((int(w[1]) << 32 | int(w[0])) >> 11) * 2.0 ** -53 * T
            C = (np.arange(1, n2 - s + 1) * al[i]) + (bp[s:] - base)
            hits = np.nonzero(C > target)[0]
            cols.append(int(sig[s + hits[0]]) if len(hits) else int(sig[n2 - 1]))
        assert list(J[I == i]) == sorted(cols)


def test_multinomial_omega_is_the_set_of_draws():
    """Ω of the multinomial model (R27) = saturated pairs ∪ the distinct drawn
    pairs, in (i, j) order, no duplicates; q̂ = 1 exactly on saturated pairs."""
    n1, n2, m = 20, 15, 200.0
    al, be = _ab(n1, n2, 5)
    _, _, sat = _mn_ref_rows(m, al, be)
    for seed in range(5):
        dI, dJ = oracle.multinomial_draws(seed, m, al, be)
        I, J, q = oracle.sample_multinomial(seed, m, al, be)
        ref = sorted(set(zip(dI.tolist(), dJ.tolist())) | set(zip(*np.nonzero(sat))))
        assert list(zip(I.tolist(), J.tolist())) == [(int(a), int(b)) for a, b in ref]
        assert len(set(zip(dI.tolist(), dJ.tolist()))) < len(dI)    # repeats were merged
        assert np.all(q[sat[I, J]] == 1.0)
        assert np.all((q > 0) & (q <= 1))


def test_multinomial_qhat_closed_form():
    """q̂ = 1 − (1−π)^F (1 − fπ) (R27) against direct evaluation in exact
    rational arithmetic (fractions) and its limits: q̂ → q = m(α+β) when
    q ≪ 1; π = 1 ⇒ q̂ = 1 (F ≥ 1) or f (F = 0)."""
    from fractions import Fraction as Fr
    for (m, a, b, T) in [(50.0, 1e-3, 2e-3, 0.04), (3.7, 0.1, 0.05, 0.6), (1e4, 1e-9, 3e-9, 1e-4),
                         (0.3, 0.2, 0.1, 0.5)]:
        mi = Fr(m) * Fr(T)
        F = mi.numerator // mi.denominator
        f = mi - F
        pi = (Fr(a) + Fr(b)) / Fr(T)
        exact = 1 - (1 - pi) ** F * (1 - f * pi)
        got = oracle.mn_qhat(m, a, b, T)
        assert abs(got - float(exact)) <= 1e-13 * float(exact)
    # small-q limit: q̂/q -> 1 with relative deviation ~ q/2
    q = 50.0 * (1e-7 + 2e-7)
    g = oracle.mn_qhat(50.0, 1e-7, 2e-7, 0.3)
    assert abs(g / q - 1) < 2 * q
    assert oracle.mn_qhat(5.0, 0.5, 0.5, 1.0) == 1.0
    assert abs(oracle.mn_qhat(0.4, 0.5, 0.5, 1.0) - 0.4) < 1e-15


def test_multinomial_inclusion_frequency_equals_qhat():
    """P((i, j) ∈ Ω) = q̂_ij (R27): empirical inclusion frequencies over seeds
    against q̂ (z-test per pair and chi-squared over all pairs), saturated
    pairs always in.  A dropped f term or q̂ = q fails it on the heavy pairs."""
    n1, n2, m = 4, 12, 30.0
    al, be = _ab(n1, n2, 9)
    seeds = 3000
    hits = np.zeros((n1, n2))
    qmat = None
    for s in range(seeds):
        I, J, q = oracle.sample_multinomial(s + 77, m, al, be)
        hits[I, J] += 1
        if qmat is None or len(I) == n1 * n2:
            qm = np.full((n1, n2), np.nan)
            qm[I, J] = q
            qmat = qm if qmat is None else np.where(np.isnan(qmat), qm, qmat)
    s_i, T_i = oracle.mn_rows(m, al, be)
    qq = m * (al[:, None] + be[None, :])
    qh = np.array([[1.0 if qq[i, j] >= 1 else oracle.mn_qhat(m, al[i], be[j], T_i[i]) for j in range(n2)]
                   for i in range(n1)])
    ok = ~np.isnan(qmat)
    np.testing.assert_allclose(qmat[ok], qh[ok], rtol=1e-14)
    p = hits / seeds
    z = (p - qh) / np.sqrt(qh * (1 - qh) / seeds + 1e-300)
    inner = (qh > 0) & (qh < 1)
    assert np.all(np.abs(z[inner]) < 4.5)
    chi2 = (z[inner] ** 2).sum()
    dof = int(inner.sum())
    assert chi2 < dof + 5 * np.sqrt(2 * dof)
    assert (qq >= 1).any() and np.max(qh[qq < 1]) > 0.4    # saturated and heavy unsaturated pairs


def test_multinomial_error_within_factor_two_of_bernoulli():
    """"the error in this model is bounded up to a factor of 2 of the
    error achieved by the Binomial model".  Exact entries of a skewed-norm
    rank-r product (GD-like column scales), same m, WAltMin on each Ω;
    median over seeds."""
    rng = np.random.default_rng(31)
    n, r, d = 120, 3, 400
    G = rng.standard_normal((d, n))
    Dg = 1.0 / np.arange(1, n + 1) ** 0.7
    A = G * Dg
    M = A.T @ A
    a2 = (A * A).sum(0)
    FA = oracle.pairwise_sum(a2)
    al, be = oracle.alpha_beta(a2, a2, FA, FA)
    m = 4 * n * r * math.log(n)
    Ms = np.linalg.svd(M, compute_uv=False)
    opt = Ms[r] / Ms[0]
    errs = {"bernoulli": [], "multinomial": []}
    for s in range(5):
        for name, fn in (("bernoulli", oracle.sample), ("multinomial", oracle.sample_multinomial)):
            I, J, q = fn(100 + s, m, al, be)
            U, V = oracle.waltmin(n, n, r, 10, I, J, M[I, J], q, np.sqrt(a2), math.sqrt(FA),
                                  init_iters=50, seed=s)
            errs[name].append(np.linalg.norm(U @ V.T - M, 2) / Ms[0])
    eb, em = np.median(errs["bernoulli"]), np.median(errs["multinomial"])
    assert eb < 5 * opt + 0.05
    assert em <= 2.0 * eb + 1e-3, (em, eb)


# ------------------------------------------------------------------ WAltMin weights, trim, partition
def test_waltmin_init_is_weighted_subspace():
    """Alg. 2 lines 2, 4, 5: the init subspace is the top-r left singular
    subspace of R = w .* P_Ω(M̃) with w = 1/q̂ — for NON-uniform q̂ (log-uniform
    on [0.05, 1]) — from LAPACK on the dense R, and it measurably differs from
    the unweighted subspace (so w = 1 or w = q̂ fail)."""
    rng = np.random.default_rng(41)
    n1, n2, r = 50, 40, 3
    M = (rng.standard_normal((n1, r)) * [10, 5, 2]) @ rng.standard_normal((r, n2))
    M += 0.5 * rng.standard_normal((n1, n2))
    qfull = np.exp(rng.uniform(np.log(0.05), 0.0, (n1, n2)))
    mask = rng.random((n1, n2)) < qfull
    I, J = np.nonzero(mask)
    q = qfull[I, J]
    U, V = oracle.waltmin(n1, n2, r, 0, I, J, M[I, J], q, np.ones(n1), 1.0, init_iters=300,
                          trim_c=0.0)
    R = np.zeros((n1, n2))
    R[I, J] = M[I, J] / q
    Uw = np.linalg.svd(R)[0][:, :r]
    cw = np.linalg.svd(Uw.T @ U, compute_uv=False)
    assert np.all(cw > 1 - 1e-8)
    R1 = np.zeros((n1, n2))
    R1[I, J] = M[I, J]
    Uu = np.linalg.svd(R1)[0][:, :r]
    cu = np.linalg.svd(Uu.T @ U, compute_uv=False)
    assert cu.min() < 1 - 1e-4       # the weighting matters on this instance
    Rq = np.zeros((n1, n2))
    Rq[I, J] = M[I, J] * q
    cq = np.linalg.svd(np.linalg.svd(Rq)[0][:, :r].T @ U, compute_uv=False)
    assert cq.min() < 1 - 1e-4
    assert np.all(V == 0)


def test_waltmin_one_iteration_is_weighted_lstsq():
    """Alg. 2 lines 8-9 with w = 1/q̂ (non-uniform): T = 1 equals numpy lstsq
    with sqrt(w) row scaling — V from the init U0, then U from V — with U0
    from LAPACK (the init pin above)."""
    rng = np.random.default_rng(42)
    n1, n2, r = 45, 35, 2
    M = rng.standard_normal((n1, r)) @ rng.standard_normal((r, n2)) + 0.3 * rng.standard_normal((n1, n2))
    qfull = np.exp(rng.uniform(np.log(0.05), 0.0, (n1, n2)))
    mask = rng.random((n1, n2)) < np.maximum(qfull, 0.3)
    I, J = np.nonzero(mask)
    q = qfull[I, J]
    U, V = oracle.waltmin(n1, n2, r, 1, I, J, M[I, J], q, np.ones(n1), 1.0, init_iters=400,
                          trim_c=0.0, lam=0.0)
    w = 1.0 / q
    R = np.zeros((n1, n2))
    R[I, J] = M[I, J] * w
    U0 = np.linalg.svd(R)[0][:, :r]
    V1 = np.zeros((n2, r))
    for j in range(n2):
        s = J == j
        sw = np.sqrt(w[s])
        V1[j] = np.linalg.lstsq(U0[I[s]] * sw[:, None], M[I[s], j] * sw, rcond=None)[0]
    U1 = np.zeros((n1, r))
    for i in range(n1):
        s = I == i
        sw = np.sqrt(w[s])
        U1[i] = np.linalg.lstsq(V1[J[s]] * sw[:, None], M[i, J[s]] * sw, rcond=None)[0]
    # U0 is defined up to a rotation; U1 V1ᵀ is not
    np.testing.assert_allclose(U @ V.T, U1 @ V1.T, rtol=1e-7, atol=1e-7 * np.abs(M).max())
    # and the unweighted fit differs
    U1u = np.zeros((n1, r))
    for i in range(n1):
        s = I == i
        U1u[i] = np.linalg.lstsq(V1[J[s]], M[i, J[s]], rcond=None)[0]
    assert np.abs(U1u @ V1.T - U1 @ V1.T).max() > 1e-3 * np.abs(M).max()


def test_waltmin_trim_threshold_exact():
    """Alg. 2 line 6 (R13): a row of U0 is zeroed iff
    ‖U0_i‖ > c·sqrt(r)·‖A_i‖/‖A‖_F.  Row norms of U0 are the leverage scores of
    R (rotation invariant; LAPACK).  ‖A_i‖ is placed so that row 3 sits at
    1.01× its threshold (zeroed) and row 7 at 0.99× (kept); every other row
    far below.  Dropping sqrt(r) or comparing squares moves one of them."""
    rng = np.random.default_rng(43)
    n1, n2, r, c = 30, 25, 3, 8.0
    M = (rng.standard_normal((n1, r)) * [6, 3, 1]) @ rng.standard_normal((r, n2))
    I, J = np.meshgrid(np.arange(n1), np.arange(n2), indexing="ij")
    I, J = I.ravel(), J.ravel()
    lev = np.linalg.norm(np.linalg.svd(M)[0][:, :r], axis=1)
    frob = 2.0
    a_norm = np.full(n1, 10.0)                 # threshold 8·sqrt(3)·10/2 ≫ 1 >= lev
    a_norm[3] = lev[3] / 1.01 * frob / (c * math.sqrt(r))
    a_norm[7] = lev[7] / 0.99 * frob / (c * math.sqrt(r))
    U, _ = oracle.waltmin(n1, n2, r, 0, I, J, M[I, J], np.ones(len(I)), a_norm, frob,
                          init_iters=200, trim_c=c)
    assert np.all(U[3] == 0)
    assert np.linalg.norm(U[7]) > 0
    # re-orthonormalised basis of the trimmed U0
    U0 = np.linalg.svd(M)[0][:, :r].copy()
    U0[3] = 0
    Q = np.linalg.qr(U0)[0]
    np.testing.assert_allclose(np.linalg.svd(Q.T @ U, compute_uv=False), 1.0, atol=1e-8)
    np.testing.assert_allclose(U.T @ U, np.eye(r), atol=1e-10)


def test_partition_equal_random_subsets():
    """Alg. 2 line 3 (R11 FRESH_2T1): 2T+1 subsets whose sizes differ by
    at most one; every sample in exactly one; the assignment recomputed from
    raw Philox words (the definition); uniform over subsets (chi-squared over
    seeds for fixed pairs)."""
    rng = np.random.default_rng(44)
    I = rng.integers(0, 300, 1001).astype(np.int32)
    J = rng.integers(0, 200, 1001).astype(np.int32)
    order = np.lexsort((J, I))
    I, J = I[order], J[order]
    for T in (1, 3, 10):
        sub = oracle.partition(5, T, I, J)
        sizes = np.bincount(sub, minlength=2 * T + 1)
        assert len(sizes) == 2 * T + 1 and sizes.max() - sizes.min() <= 1 and sizes.sum() == len(I)
    T = 3
    key = [5, 0]
    keys = []
    for s in range(len(I)):
        w = oracle.philox4x32_10([int(I[s]), int(J[s]), 0, 4], key)
        keys.append((int(w[1]) << 32 | int(w[0]), int(I[s]), int(J[s]), s))
    ref = np.empty(len(I), np.int32)
    for p, kk in enumerate(sorted(keys)):
        ref[kk[3]] = p % (2 * T + 1)
    assert np.array_equal(oracle.partition(5, T, I, J), ref)
    # uniformity: the subset of the first 20 pairs over 700 seeds
    cnt = np.zeros((20, 2 * T + 1))
    for sd in range(700):
        sub = oracle.partition(sd, T, I, J)
        cnt[np.arange(20), sub[:20]] += 1
    e = 700 / (2 * T + 1)
    chi2 = ((cnt - e) ** 2 / e).sum()
    dof = 20 * 2 * T
    assert chi2 < dof + 5 * np.sqrt(2 * dof)


def test_waltmin_fresh_partition_pipeline():
    """FRESH_2T1 (Alg. 2 lines 3-9 literally): init on Ω_0 only, V on Ω_1, U on
    Ω_2 (T = 1) — against numpy: LAPACK subspace of R_Ω0, lstsq per row with
    sqrt(w) scaling on the named subsets."""
    rng = np.random.default_rng(45)
    n1, n2, r, T = 60, 50, 2, 1
    M = rng.standard_normal((n1, r)) @ rng.standard_normal((r, n2)) + 0.2 * rng.standard_normal((n1, n2))
    qfull = np.exp(rng.uniform(np.log(0.3), 0.0, (n1, n2)))
    mask = rng.random((n1, n2)) < qfull
    I, J = np.nonzero(mask)
    I, J = I.astype(np.int32), J.astype(np.int32)
    q = qfull[I, J]
    U, V = oracle.waltmin(n1, n2, r, T, I, J, M[I, J], q, np.ones(n1), 1.0, init_iters=400,
                          trim_c=0.0, lam=0.0, seed=9, partition=oracle.PART_FRESH_2T1)
    sub = oracle.partition(9, T, I, J)
    w = 1.0 / q
    s0 = sub == 0
    R = np.zeros((n1, n2))
    R[I[s0], J[s0]] = M[I[s0], J[s0]] * w[s0]
    U0 = np.linalg.svd(R)[0][:, :r]
    V1 = np.zeros((n2, r))
    for j in range(n2):
        s = (J == j) & (sub == 1)
        sw = np.sqrt(w[s])
        V1[j] = np.linalg.lstsq(U0[I[s]] * sw[:, None], M[I[s], j] * sw, rcond=None)[0]
    U1 = np.zeros((n1, r))
    for i in range(n1):
        s = (I == i) & (sub == 2)
        sw = np.sqrt(w[s])
        U1[i] = np.linalg.lstsq(V1[J[s]] * sw[:, None], M[i, J[s]] * sw, rcond=None)[0]
    np.testing.assert_allclose(U @ V.T, U1 @ V1.T, rtol=1e-7, atol=1e-7 * np.abs(M).max())
    Ur, Vr = oracle.waltmin(n1, n2, r, T, I, J, M[I, J], q, np.ones(n1), 1.0, init_iters=400,
                            trim_c=0.0, lam=0.0, seed=9)
    assert np.abs(Ur @ Vr.T - U @ V.T).max() > 1e-3     # REUSE_ALL is a different reading


# ------------------------------------------------------------------ Theorem 1
def _eta_hat(A, B, k, m, r, seed, pi_kind):
    M = A.T @ B
    U_, s, Vt = np.linalg.svd(M)
    Mr = (U_[:, :r] * s[:r]) @ Vt[:r]
    res = oracle.smp_pca(A, B, k=k, r=r, m=m, T=15, pi_kind=pi_kind, seed=seed, init_iters=60)
    err = np.linalg.norm(Mr - res["U"] @ res["V"].T, 2)
    tail = np.sqrt((s[r:] ** 2).sum())
    return err / (tail + s[r - 1])


def test_theorem1_implied_eta_below_one_and_shrinks():
    """Eq. 7: ‖(AᵀB)_r − ÛV̂ᵀ‖ ≤ η‖AᵀB − (AᵀB)_r‖_F + ζ + η σ_r*.  With
    ζ = 0 (T = 15 ≥ log((‖A‖_F+‖B‖_F)/ζ) is not checkable; ζ absorbed) the
    implied η̂ = err/(‖AᵀB − (AᵀB)_r‖_F + σ_r*) must be < 1, shrink with k at
    saturated m (Eq. 5: η ∝ 1/√k), and shrink with m at exact M̃ (Hadamard
    k = d, Eq. 6: η ∝ 1/√m).  Medians over seeds.  GD-type inputs."""
    rng = np.random.default_rng(46)
    d, n, r = 512, 48, 3
    G = rng.standard_normal((d, n))
    A = G * (1.0 / np.arange(1, n + 1))
    B = (G + 0.5 * rng.standard_normal((d, n))) * (1.0 / np.arange(1, n + 1) ** 0.5)
    eta_k = [np.median([_eta_hat(A, B, k, 1e12, r, s, oracle.PI_GAUSSIAN) for s in range(3)])
             for k in (32, 128, 512)]
    assert eta_k[2] < 1.0
    assert eta_k[0] > eta_k[1] > eta_k[2], eta_k
    assert eta_k[0] / eta_k[2] > 2.0              # ~ sqrt(16) = 4 expected
    base = n * r * math.log(n)
    eta_m = [np.median([_eta_hat(A, B, d, c * base, r, s, oracle.PI_HADAMARD) for s in range(3)])
             for c in (1.5, 3.0, 8.0)]
    assert eta_m[2] < 1.0
    assert eta_m[0] > eta_m[1] > eta_m[2], eta_m


# ------------------------------------------------------------------ LELA (NEXT-3)
def test_exact_entries_equal_matmul_and_block_additivity():
    """LELA's pass 2 against the library matmul (AᵀB)[I, J]; fp32 and bf16
    inputs read exactly; row blocks in any order sum to the whole."""
    rng = np.random.default_rng(51)
    d, n1, n2 = 700, 40, 30
    A = rng.standard_normal((d, n1))
    B = rng.standard_normal((d, n2))
    I = rng.integers(0, n1, 200).astype(np.int32)
    J = rng.integers(0, n2, 200).astype(np.int32)
    ref = (A.T @ B)[I, J]
    np.testing.assert_allclose(oracle.exact_entries(A, B, I, J), ref, rtol=1e-12, atol=1e-12)
    out = np.zeros(200)
    for r0, r1 in [(300, 700), (0, 120), (120, 300)]:
        oracle.exact_entries(A[r0:r1], B[r0:r1], I, J, out)
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)
    A32 = A.astype(np.float32)
    Abf = (A32.view(np.uint32) >> 16).astype(np.uint16)
    Aval = (Abf.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    np.testing.assert_allclose(oracle.exact_entries(Abf, B, I, J), (Aval.T @ B)[I, J], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(oracle.exact_entries(A32, B, I, J), (A32.astype(np.float64).T @ B)[I, J],
                               rtol=1e-12, atol=1e-12)


def test_lela_exact_rank_saturated_and_beats_smp_pca():
    """LELA with saturated sampling on an exact rank-r product recovers it
    (exact entries, full observation); on a noisy GD instance LELA's
    error is at most SMP-PCA's ("LELA always achieves a smaller spectral
    norm error than SMP-PCA"), both above the optimal rank-r error."""
    rng = np.random.default_rng(52)
    d, n, r = 300, 30, 3
    Z = rng.standard_normal((d, r))
    A = Z @ rng.standard_normal((r, n))
    B = Z @ rng.standard_normal((r, n))
    res = oracle.lela(A, B, r, 1e12, 5, trim_c=0.0)
    assert len(res["I"]) == n * n
    np.testing.assert_allclose(res["U"] @ res["V"].T, A.T @ B, rtol=1e-7, atol=1e-7 * np.abs(A.T @ B).max())
    d, n, r = 2000, 80, 5
    G = rng.standard_normal((d, n))
    A = G * (1.0 / np.arange(1, n + 1))
    M = A.T @ A
    s = np.linalg.svd(M, compute_uv=False)
    m = 4 * n * r * math.log(n)
    el, es = [], []
    for sd in range(3):
        L = oracle.lela(A, A, r, m, 10, seed=sd)
        S = oracle.smp_pca(A, A, k=128, r=r, m=m, T=10, pi_kind=oracle.PI_GAUSSIAN, seed=sd, a_is_b=True)
        el.append(np.linalg.norm(L["U"] @ L["V"].T - M, 2) / s[0])
        es.append(np.linalg.norm(S["U"] @ S["V"].T - M, 2) / s[0])
    assert s[r] / s[0] <= np.median(el) + 1e-9
    assert np.median(el) <= np.median(es) + 1e-9, (el, es)


def test_finalize_flushes_negligible_norms_r25():
    """R25: a column whose norm² is below 2^-200 is the zero column: D = 0 and
    its norm² becomes an exact 0 (so Eq. 1 gives α = 0); a column just above
    the threshold keeps its value."""
    k = 8
    sk = np.ones((3, k))
    norm2 = np.array([2.0 ** -210, 2.0 ** -190, 4.0])
    out, sn, D = oracle.finalize(k, sk, norm2)
    assert norm2[0] == 0.0 and D[0] == 0.0
    assert norm2[1] == 2.0 ** -190 and D[1] > 0
    np.testing.assert_allclose(D[2], 2.0 / np.sqrt(k * (1.0 / k)), rtol=1e-15)
