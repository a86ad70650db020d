"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element, on seeded inputs (DESIGN.md §4 lists the tolerances and why).

  sketch Ã, B̃      ||Ã_i^gpu - Ã_i^or|| / ||Ã_i^or|| <= 1e-5 per column (north star)
  norms ||A_i||²   relative 2e-7 (bf16: exact fp32 squares summed in fp32 over 4-row
                   chunks, fp64 across chunks: <= 3·2^-24 relative worst case, R4)
  Ω, indices        bit-exact;  q̂ relative 1e-12
  M̃                |M̃^gpu - M̃^or| <= 1e-4 ||A_i|| ||B_j||   (R22, Lemma JL scale P:318)
  factors           ||UVᵀ_gpu - UVᵀ_or||_2 / ||AᵀB||_2 <= 1e-3
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

PI = {"rademacher": 0, "gaussian": 1, "hadamard": 2}


def _smp():
    import paper_1610_06656_b200 as smp
    return smp


def _to_np(X):
    if X.dtype == torch.bfloat16:
        return synth.bf16_bits(X)
    return X.detach().cpu().numpy()


def gpu_sketch(A, B, k, pi, seed=0, row0=0, d_total=None, blocks=None, a_is_b=False):
    smp = _smp()
    inp = smp.IN_DENSE_BF16 if A.dtype == torch.bfloat16 else smp.IN_DENSE_F32
    d = A.shape[0] + row0 if d_total is None else d_total
    sk = smp.SMPSketch(d, A.shape[1], A.shape[1] if a_is_b else B.shape[1], k, pi=pi, seed=seed,
                       a_is_b=a_is_b, input=inp)
    Ad = A.cuda()
    Bd = None if a_is_b else B.cuda()
    if blocks is None:
        sk.block(row0, Ad, Bd)
    else:
        for (r0, r1) in blocks:
            sk.block(row0 + r0, Ad[r0:r1], None if a_is_b else Bd[r0:r1])
    fin = sk.finalize()
    return sk, fin


def oracle_sketch(A, B, k, pi, seed=0, row0=0, a_is_b=False):
    skA, a2 = oracle.sketch_rows(pi, seed, k, _to_np(A), row0=row0)
    if a_is_b:
        skB, b2 = skA, a2
    else:
        skB, b2 = oracle.sketch_rows(pi, seed, k, _to_np(B), row0=row0)
    As, asn, DA = oracle.finalize(k, skA, a2)
    Bs, bsn, DB = oracle.finalize(k, skB, b2)
    return dict(As=As, Bs=Bs, a2=a2, b2=b2, DA=DA, DB=DB, asn=asn, bsn=bsn,
                FA=oracle.pairwise_sum(a2), FB=oracle.pairwise_sum(b2))


def col_rel_err(gpu, ref):
    g = gpu.detach().cpu().double().numpy()
    num = np.linalg.norm(g - ref, axis=1)
    den = np.linalg.norm(ref, axis=1)
    return np.where(den > 0, num / np.where(den > 0, den, 1), num)


NORM_RTOL = 2e-7   # 3·2^-24 (R4): worst-case bound of the 4-row fp32 chunk sums


def check_sketch(fin, orc, tol=1e-5):
    ea = col_rel_err(fin["A_sk"], orc["As"])
    eb = col_rel_err(fin["B_sk"], orc["Bs"])
    assert ea.max() <= tol, f"A sketch max col rel err {ea.max():.3e}"
    assert eb.max() <= tol, f"B sketch max col rel err {eb.max():.3e}"
    a2 = fin["a_norm2"].cpu().numpy()
    b2 = fin["b_norm2"].cpu().numpy()
    np.testing.assert_allclose(a2, orc["a2"], rtol=NORM_RTOL, atol=0)
    np.testing.assert_allclose(b2, orc["b2"], rtol=NORM_RTOL, atol=0)
    fr = fin["frob2"].cpu().numpy()
    np.testing.assert_allclose(fr, [orc["FA"], orc["FB"]], rtol=NORM_RTOL)


# ------------------------------------------------------------------ Step 1
@pytest.mark.parametrize("d,n1,n2,k,pi", [
    (2000, 100, 100, 64, "rademacher"),     # cfg0 shape
    (4096, 300, 520, 256, "rademacher"),    # several n-tiles, ragged n
    (3001, 257, 33, 130, "rademacher"),     # ragged d, k not a multiple of 128
    (2500, 64, 96, 384, "gaussian"),        # two κ tiles
    (1000, 40, 40, 512, "gaussian"),
])
def test_sketch_bf16_parity(d, n1, n2, k, pi):
    A = synth.gaussian_small(d, n1, seed=1, scale_cols=True).to(torch.bfloat16)
    B = synth.gaussian_small(d, n2, seed=2).to(torch.bfloat16)
    _, fin = gpu_sketch(A, B, k, PI[pi], seed=7)
    orc = oracle_sketch(A, B, k, PI[pi], seed=7)
    check_sketch(fin, orc)


@pytest.mark.parametrize("gen_sets", ["", "2", "3", "4"])
def test_sketch_generator_sets(monkeypatch, gen_sets):
    """K1 with 2, 3 or 4 Π generator warp sets (TMEM ring of 2·GS stages; the
    default picks 3 when several κ tiles share an X tile): same sketch as the
    oracle — every set's K-block pairs, the ring phases and the Philox
    prefetch of the next pair are exercised (k = 700: 3 κ tiles, ragged)."""
    if gen_sets:
        monkeypatch.setenv("SMP_K1_GEN_SETS", gen_sets)
    d, n1, n2, k = 24000, 300, 200, 700
    A = synth.gaussian_small(d, n1, seed=11, scale_cols=True).to(torch.bfloat16)
    B = synth.gaussian_small(d, n2, seed=12).to(torch.bfloat16)
    _, fin = gpu_sketch(A, B, k, PI["rademacher"], seed=13)
    orc = oracle_sketch(A, B, k, PI["rademacher"], seed=13)
    check_sketch(fin, orc)


@pytest.mark.parametrize("d,n,k,pi", [(2000, 100, 64, "rademacher"), (1500, 70, 256, "gaussian")])
def test_sketch_f32_parity(d, n, k, pi):
    """fp32 inputs go through the exact 3-term bf16 split."""
    A, B = synth.cone_tiny(d, n, seed=0)
    _, fin = gpu_sketch(A, B, k, PI[pi], seed=0)
    orc = oracle_sketch(A, B, k, PI[pi], seed=0)
    check_sketch(fin, orc)


def test_sketch_f32_norms_extreme_magnitudes():
    """K1F accumulates Σx² as fp32 double-float pairs while x² and its FMA
    residual are normal fp32 numbers (|x| in [2^-40, 2^41)) and in fp64
    otherwise: columns scaled from 1e-30 to 1e18 (x² under- and overflows
    fp32 at both ends) must still give the oracle's fp64 norms, and the
    sketch its 1e-5 (the plane split is scale-free)."""
    d, n = 4096, 128
    A = synth.gaussian_small(d, n, seed=31).float()
    B = synth.gaussian_small(d, n, seed=32).float()
    exps = torch.tensor([-30, -22, -13, -12, -6, 0, 5, 12, 13, 18], dtype=torch.float64)
    sa = (10.0 ** exps[torch.arange(n) % len(exps)]).float()
    A = A * sa[None, :]
    B = B * sa.flip(0)[None, :]
    B[::3, 7] = 0.0   # exact zeros mixed into a tiny-magnitude column
    _, fin = gpu_sketch(A, B, 64, PI["rademacher"], seed=3)
    orc = oracle_sketch(A, B, 64, PI["rademacher"], seed=3)
    ea = col_rel_err(fin["A_sk"], orc["As"])
    eb = col_rel_err(fin["B_sk"], orc["Bs"])
    assert ea.max() <= 1e-5 and eb.max() <= 1e-5, (ea.max(), eb.max())
    np.testing.assert_allclose(fin["a_norm2"].cpu().numpy(), orc["a2"], rtol=1e-12, atol=0)
    np.testing.assert_allclose(fin["b_norm2"].cpu().numpy(), orc["b2"], rtol=1e-12, atol=0)


def test_sketch_unaligned_row0_and_blocks():
    """Global row offsets not multiple of 32/64 exercise the generic Π path;
    blocks in arbitrary order sum to the whole."""
    d, n, k = 1900, 150, 128
    A = synth.gaussian_small(d, n, seed=3).to(torch.bfloat16)
    B = synth.gaussian_small(d, n, seed=4).to(torch.bfloat16)
    row0 = 77
    blocks = [(1200, 1900), (0, 333), (333, 1200)]
    _, fin = gpu_sketch(A, B, k, 0, seed=5, row0=row0, d_total=row0 + d, blocks=blocks)
    orc = oracle_sketch(A, B, k, 0, seed=5, row0=row0)
    check_sketch(fin, orc)


def test_sketch_a_equals_b():
    d, n, k = 1024, 96, 64
    A = synth.gaussian_small(d, n, seed=9).to(torch.bfloat16)
    _, fin = gpu_sketch(A, None, k, 1, seed=2, a_is_b=True)
    orc = oracle_sketch(A, A, k, 1, seed=2, a_is_b=True)
    check_sketch(fin, orc)


def test_zero_and_sparse_columns():
    """Degenerate columns: an all-zero column (norm 0, D = 0, never sampled
    beyond the B-side term) and a column with a single nonzero entry."""
    d, n, k = 777, 40, 64
    A = synth.gaussian_small(d, n, seed=13)
    A[:, 3] = 0.0
    A[:, 5] = 0.0
    A[100, 5] = 2.5
    A[:, 7] = 2.0 ** -110          # norm² ~ 2^-210: the zero column of R25 on both sides
    A = A.to(torch.bfloat16)
    B = synth.gaussian_small(d, n, seed=14).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, k, 0, seed=1)
    orc = oracle_sketch(A, B, k, 0, seed=1)
    check_sketch(fin, orc)
    assert float(fin["a_norm2"][3]) == 0.0 and float(fin["a_norm2"][5]) == 6.25
    assert float(fin["a_norm2"][7]) == 0.0 and orc["a2"][7] == 0.0
    I, J, val, qh = sk.sample_estimate(500.0, 4)
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    Io, Jo, qo = oracle.sample(4, 500.0, al, be)
    assert np.array_equal(I.cpu().numpy(), Io) and np.array_equal(J.cpu().numpy(), Jo)
    v = val.cpu().numpy()
    assert np.all(v[I.cpu().numpy() == 3] == 0.0)  # D_A = 0 for the zero column


def test_hadamard_k_equals_d_exact_product():
    """North star (a): Hadamard Π with k = d gives M̃ = AᵀB (fully sampled)."""
    smp = _smp()
    d, n = 256, 24
    A = synth.gaussian_small(d, n, seed=11).to(torch.bfloat16)
    B = synth.gaussian_small(d, n, seed=12).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, d, smp.PI_HADAMARD_TEST, seed=0)
    I, J, val, qh = sk.sample_estimate(1e12, 0)
    assert I.numel() == n * n
    M = (A.double().T @ B.double()).numpy()
    got = np.zeros((n, n))
    got[I.cpu().numpy(), J.cpu().numpy()] = val.cpu().numpy()
    scale = np.outer(np.linalg.norm(A.double().numpy(), axis=0), np.linalg.norm(B.double().numpy(), axis=0))
    assert np.max(np.abs(got - M) / scale) < 1e-5


# ------------------------------------------------------------------ Step 2
@pytest.mark.parametrize("n1,n2,m_coef", [(100, 100, 0.3), (600, 450, 4.0), (300, 257, 50.0)])
def test_omega_bit_exact_and_mtilde(n1, n2, m_coef):
    d, k = 3000, 128
    A = synth.gaussian_small(d, n1, seed=21, scale_cols=True).to(torch.bfloat16)
    B = synth.gaussian_small(d, n2, seed=22, scale_cols=True).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, k, 0, seed=3)
    orc = oracle_sketch(A, B, k, 0, seed=3)
    m = m_coef * max(n1, n2) * 5 * math.log(max(n1, n2))
    I, J, val, qh = sk.sample_estimate(m, 99)
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    Io, Jo, qo = oracle.sample(99, m, al, be)
    assert np.array_equal(I.cpu().numpy(), Io) and np.array_equal(J.cpu().numpy(), Jo)
    np.testing.assert_allclose(qh.cpu().numpy(), qo, rtol=2 * NORM_RTOL)
    Mo = oracle.estimate(k, Io, Jo, orc["As"], orc["Bs"], orc["DA"], orc["DB"])
    scale = np.sqrt(orc["a2"][Io] * orc["b2"][Jo])
    err = np.abs(val.cpu().double().numpy() - Mo) / scale
    assert err.max() <= 1e-4, err.max()
    # plain JL estimator as well
    I2, J2, v2, _ = sk.sample_estimate(m, 99, plain=True)
    Mp = oracle.estimate(k, Io, Jo, orc["As"], orc["Bs"], orc["DA"], orc["DB"], plain=True)
    assert np.max(np.abs(v2.cpu().double().numpy() - Mp) / scale) <= 1e-4


def test_omega_capacity_and_empty():
    smp = _smp()
    d, n, k = 512, 50, 64
    A = synth.gaussian_small(d, n, seed=31).to(torch.bfloat16)
    B = synth.gaussian_small(d, n, seed=32).to(torch.bfloat16)
    sk, _ = gpu_sketch(A, B, k, 0)
    I, J, v, q = sk.sample_estimate(200.0, 1, cap=5)  # grows internally
    assert I.numel() > 5
    I2, J2, v2, q2 = sk.sample_estimate(1e-9, 1)
    assert I2.numel() == 0


# ------------------------------------------------------------------ Step 3
def _uvt_err(U1, V1, U2, V2, M):
    P1 = U1 @ V1.T
    P2 = U2 @ V2.T
    return np.linalg.norm(P1 - P2, 2) / np.linalg.norm(M, 2)


@pytest.mark.parametrize("n1,n2,r,m_coef", [(120, 100, 5, 4.0), (300, 200, 10, 6.0)])
def test_waltmin_parity_identical_inputs(n1, n2, r, m_coef):
    """WAltMin (Alg. 2) on the ORACLE's Ω, M̃ (rounded to fp32) and q̂ —
    identical inputs on both sides — agrees to 1e-3 of ||AᵀB||."""
    d, k = 2000, 256
    Z = synth.gaussian_small(d, r, seed=41).double()
    A = (Z @ synth.gaussian_small(r, n1, seed=42).double() + 0.1 * synth.gaussian_small(d, n1, seed=43).double()).to(torch.bfloat16)
    B = (Z @ synth.gaussian_small(r, n2, seed=44).double() + 0.1 * synth.gaussian_small(d, n2, seed=45).double()).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, k, 0, seed=1)
    orc = oracle_sketch(A, B, k, 0, seed=1)
    m = m_coef * max(n1, n2) * r * math.log(max(n1, n2))
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    Io, Jo, qo = oracle.sample(5, m, al, be)
    Mo = oracle.estimate(k, Io, Jo, orc["As"], orc["Bs"], orc["DA"], orc["DB"]).astype(np.float32)
    Uo, Vo = oracle.waltmin(n1, n2, r, 10, Io, Jo, Mo.astype(np.float64), qo, np.sqrt(orc["a2"]),
                            math.sqrt(orc["FA"]), init_iters=30, seed=9)
    dev = torch.device("cuda")
    Ug, Vg = sk.waltmin(torch.tensor(Io, device=dev), torch.tensor(Jo, device=dev),
                        torch.tensor(Mo, device=dev), torch.tensor(qo, device=dev), r, 10,
                        init_iters=30, seed=9)
    M = (A.double().T @ B.double()).numpy()
    err = _uvt_err(Ug.cpu().double().numpy(), Vg.cpu().double().numpy(), Uo, Vo, M)
    assert err <= 1e-3, err


@pytest.mark.parametrize("thr", ["40", "0"])
def test_waltmin_heavy_rows_parity(thr, monkeypatch):
    """WAltMin with rows split over a CTA's warps (SMP_WM_HEAVY = split
    threshold; 40 forces most rows and columns of this skewed Ω through the
    CTA-cooperative path, 0 disables it): agrees with the oracle on identical
    inputs to 1e-3 of ||AᵀB||, and both GPU paths agree to 1e-9."""
    n1, n2, r, d, k = 200, 150, 6, 2000, 256
    Z = synth.gaussian_small(d, r, seed=51).double()
    # column scales 1/sqrt(i+1): skewed norms -> a few long rows/columns in Ω
    sa = torch.arange(1, n1 + 1, dtype=torch.float64).rsqrt()
    sb = torch.arange(1, n2 + 1, dtype=torch.float64).rsqrt()
    A = ((Z @ synth.gaussian_small(r, n1, seed=52).double() + 0.1 * synth.gaussian_small(d, n1, seed=53).double())
         * sa).to(torch.bfloat16)
    B = ((Z @ synth.gaussian_small(r, n2, seed=54).double() + 0.1 * synth.gaussian_small(d, n2, seed=55).double())
         * sb).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, k, 0, seed=1)
    orc = oracle_sketch(A, B, k, 0, seed=1)
    m = 2.0 * n1 * r * math.log(n1)
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    Io, Jo, qo = oracle.sample(5, m, al, be)
    rows = np.bincount(Io, minlength=n1)
    assert (rows > 40).sum() >= 20 and (rows <= 40).sum() >= 20, rows  # both paths exercised
    Mo = oracle.estimate(k, Io, Jo, orc["As"], orc["Bs"], orc["DA"], orc["DB"]).astype(np.float32)
    Uo, Vo = oracle.waltmin(n1, n2, r, 10, Io, Jo, Mo.astype(np.float64), qo, np.sqrt(orc["a2"]),
                            math.sqrt(orc["FA"]), init_iters=30, seed=9)
    dev = torch.device("cuda")
    args = (torch.tensor(Io, device=dev), torch.tensor(Jo, device=dev), torch.tensor(Mo, device=dev),
            torch.tensor(qo, device=dev), r, 10)
    monkeypatch.setenv("SMP_WM_HEAVY", thr)
    Ug, Vg = sk.waltmin(*args, init_iters=30, seed=9)
    M = (A.double().T @ B.double()).numpy()
    Pg = Ug.cpu().double().numpy() @ Vg.cpu().double().numpy().T
    err = _uvt_err(Ug.cpu().double().numpy(), Vg.cpu().double().numpy(), Uo, Vo, M)
    assert err <= 1e-3, err
    monkeypatch.setenv("SMP_WM_HEAVY", "0")
    U0, V0 = sk.waltmin(*args, init_iters=30, seed=9)
    P0 = U0.cpu().double().numpy() @ V0.cpu().double().numpy().T
    assert np.linalg.norm(Pg - P0, 2) / np.linalg.norm(M, 2) <= 1e-9


@pytest.mark.parametrize("r,n,switch", [(5, 4200, "SMP_WM_L1"), (10, 2304, "SMP_WM_L1"),
                                        (5, 1024, "SMP_WM_CACHE"), (10, 600, "SMP_WM_CACHE"),
                                        (5, 1024, "SMP_WM_STAGE")])
def test_waltmin_gather_paths_bit_identical(r, n, switch, monkeypatch):
    """Data-path switches that must not change a bit of the factors (all read
    on every smp_waltmin call):
    SMP_WM_L1 — factor-row gathers through L1 (16-byte pieces for even r) vs
    L2-only, when the rows are too many to stage in SMEM (n r 8 B > 160 KB:
    4200·5·8 = 168 KB, 2304·10·8 = 184 KB): the grid barrier's fences make L1
    reads coherent; SMP_WM_CACHE — each CTA's sample indices/weights read
    from its SMEM copy vs from global; SMP_WM_STAGE — factor rows staged in
    SMEM vs gathered from global."""
    d, k = 4096, 256
    Z = synth.gaussian_small(d, r, seed=61)
    A = (Z @ synth.gaussian_small(r, n, seed=62) + 0.1 * synth.gaussian_small(d, n, seed=63)).to(torch.bfloat16)
    B = (Z @ synth.gaussian_small(r, n, seed=64) + 0.1 * synth.gaussian_small(d, n, seed=65)).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, k, 0, seed=2)
    I, J, val, qh = sk.sample_estimate(4 * n * r * math.log(n), 3)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv(switch, mode)
        U, V = sk.waltmin(I, J, val, qh, r, 10, init_iters=30, seed=3)
        out[mode] = (U.cpu(), V.cpu())
    assert torch.equal(out["1"][0], out["0"][0]) and torch.equal(out["1"][1], out["0"][1])
    assert float(out["1"][0].abs().sum()) > 0


def test_waltmin_rank_deficient_and_empty_rows():
    """Degenerate WAltMin inputs on identical data: R_Ω of rank 2 < r = 4
    (the init pads with zero directions) and rows/columns without any
    sample (their factor rows are 0, R14)."""
    n1, n2, r = 90, 70, 4
    rng = np.random.default_rng(71)
    M = rng.standard_normal((n1, 2)) @ rng.standard_normal((2, n2))
    mask = rng.random((n1, n2)) < 0.5
    mask[[3, 40]] = False
    mask[:, [7, 55]] = False
    Io, Jo = np.nonzero(mask)
    Io, Jo = Io.astype(np.int32), Jo.astype(np.int32)
    qo = np.full(len(Io), 0.5)
    Mo = M[Io, Jo].astype(np.float32)
    Uo, Vo = oracle.waltmin(n1, n2, r, 8, Io, Jo, Mo.astype(np.float64), qo, np.ones(n1), math.sqrt(n1),
                            init_iters=30, seed=4, trim_c=0.0)
    smp = _smp()
    A = synth.gaussian_small(64, n1, seed=1).to(torch.bfloat16)
    B = synth.gaussian_small(64, n2, seed=2).to(torch.bfloat16)
    sk, _ = gpu_sketch(A, B, 32, 0)
    dev = torch.device("cuda")
    Ug, Vg = sk.waltmin(torch.tensor(Io, device=dev), torch.tensor(Jo, device=dev), torch.tensor(Mo, device=dev),
                        torch.tensor(qo, device=dev), r, 8, init_iters=30, seed=4, trim_c=0.0)
    Ug, Vg = Ug.cpu().double().numpy(), Vg.cpu().double().numpy()
    assert np.all(Ug[[3, 40]] == 0) and np.all(Vg[[7, 55]] == 0)
    assert _uvt_err(Ug, Vg, Uo, Vo, M) <= 1e-3
    assert np.linalg.norm(Ug @ Vg.T - M, 2) / np.linalg.norm(M, 2) < 1e-3 + \
        np.linalg.norm(M[[3, 40]], 2) / np.linalg.norm(M, 2) + np.linalg.norm(M[:, [7, 55]], 2) / np.linalg.norm(M, 2)


def test_cfg0_literal_m_identical_inputs():
    """cfg0 as BASELINE states it (fp32 cone, k = 64, m = 0.3 n r ln n = 691,
    r = 5, T = 10): sketch, norms and Ω through the GPU against the oracle, then
    WAltMin on identical inputs.  This m is far below the phase transition
    (many rows have < r samples): the ALS diverges (error ~150
    ||AᵀB||) and its output moves by ~1e-3 ||AᵀB|| when M̃ moves by ONE fp32
    ulp (R14).  The factor gap is therefore held to the larger of the north
    star's 1e-3 and 4x the oracle's own 1-ulp sensitivity, measured here."""
    cfg = synth.CONFIGS["cfg0"]
    A, B = synth.cone_tiny(cfg["d"], cfg["n1"], seed=cfg["seed"])
    sk, fin = gpu_sketch(A, B, cfg["k"], 0, seed=0)
    orc = oracle_sketch(A, B, cfg["k"], 0, seed=0)
    check_sketch(fin, orc)
    m = synth.m_of(cfg)
    assert abs(m - 690.78) < 0.01
    I, J, val, qh = sk.sample_estimate(m, 0)
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    Io, Jo, qo = oracle.sample(0, m, al, be)
    assert np.array_equal(I.cpu().numpy(), Io) and np.array_equal(J.cpu().numpy(), Jo)
    assert (np.bincount(Io, minlength=100) < 5).sum() > 10
    v = val.cpu().numpy().astype(np.float64)
    Uo, Vo = oracle.waltmin(100, 100, 5, 10, Io, Jo, v, qh.cpu().numpy(), np.sqrt(orc["a2"]),
                            math.sqrt(orc["FA"]), init_iters=30, seed=0)
    Ug, Vg = sk.waltmin(I, J, val, qh, 5, 10, init_iters=30, seed=0)
    M = (A.double().T @ B.double()).numpy()
    vu = (val.cpu().numpy() * np.float32(1 + 2 ** -23)).astype(np.float64)   # M̃ one fp32 ulp up
    Uu, Vu = oracle.waltmin(100, 100, 5, 10, Io, Jo, vu, qh.cpu().numpy(), np.sqrt(orc["a2"]),
                            math.sqrt(orc["FA"]), init_iters=30, seed=0)
    sens = _uvt_err(Uu, Vu, Uo, Vo, M)
    gap = _uvt_err(Ug.cpu().double().numpy(), Vg.cpu().double().numpy(), Uo, Vo, M)
    print(f"cfg0 literal m: GPU-oracle factor gap {gap:.3e}, oracle 1-ulp sensitivity {sens:.3e}")
    assert gap <= max(1e-3, 4 * sens), (gap, sens)


def test_pipeline_end_to_end_vs_oracle():
    """Alg. 1 end to end from the same A, B on both sides (cfg1-like regime,
    m = 4 n r ln n): factors within 1e-3 of ||AᵀB||_2."""
    smp = _smp()
    d, n, r, k = 8192, 256, 5, 256
    VA = synth.lowrank_factors(n, 20, 1, 0, "cpu")
    VB = synth.lowrank_factors(n, 20, 1, 1, "cpu")
    A, B = synth.lowrank_block(0, d, n, 1, VA, VB, device="cpu")
    m = 4 * n * r * math.log(n)
    res = smp.smp_pca(A.cuda(), B.cuda(), k=k, r=r, m=m, T=10, seed=1, init_iters=30)
    orc = oracle.smp_pca(synth.bf16_bits(A), synth.bf16_bits(B), k=k, r=r, m=m, T=10, seed=1,
                         init_iters=30)
    assert np.array_equal(res["I"].cpu().numpy(), orc["I"])
    assert np.array_equal(res["J"].cpu().numpy(), orc["J"])
    M = (A.double().T @ B.double()).numpy()
    err = _uvt_err(res["U"].cpu().double().numpy(), res["V"].cpu().double().numpy(),
                   orc["U"], orc["V"], M)
    assert err <= 1e-3, err


# ------------------------------------------------------------------ Step 1, sparse (K3)
def _csr(d, n, nnz_row, seed, tag, perm=None):
    rp, col, val = synth.csr_block(0, d, n, nnz_row, seed, tag, device="cpu")
    if perm is not None:  # heavy columns away from the low indices (R18 note)
        col = torch.from_numpy(perm[col.numpy()].astype(np.int32))
        # keep rows ascending in column (CSR convention; K3 does not need it)
        rows = [col[i * nnz_row:(i + 1) * nnz_row].sort() for i in range(d)]
        val = torch.cat([val[i * nnz_row:(i + 1) * nnz_row][r.indices] for i, r in enumerate(rows)])
        col = torch.cat([r.values for r in rows])
    return rp, col, val


def gpu_sketch_csr(d, n1, n2, k, pi, seed, A, B, row0=0, splits=None):
    smp = _smp()
    sk = smp.SMPSketch(row0 + d, n1, n2, k, pi=pi, seed=seed, input=smp.IN_CSR_F32)
    splits = splits or [(0, d)]
    for (r0, r1) in splits:
        a_rp, a_col, a_val = A
        b_rp, b_col, b_val = B
        # col/val start at entry rowptr[0] of the block (include/smp.h)
        ea, eb = int(a_rp[r0]), int(b_rp[r0])
        sk.block_csr(row0 + r0, r1 - r0, a_rp[r0:r1 + 1].cuda(), a_col[ea:].cuda(), a_val[ea:].cuda(),
                     b_rp[r0:r1 + 1].cuda(), b_col[eb:].cuda(), b_val[eb:].cuda())
    return sk, sk.finalize()


@pytest.mark.parametrize("d,n1,n2,za,zb,k,pi,row0,permute", [
    (3000, 300, 200, 20, 16, 512, "gaussian", 0, False),      # cfg3 shape in miniature
    (2500, 257, 130, 12, 9, 130, "rademacher", 77, True),     # ragged k, unaligned rows, permuted heavy cols
    (70000, 40, 24, 3, 2, 64, "gaussian", 5, False),          # several Π panels (> 2^15 rows)
])
def test_sketch_csr_parity(d, n1, n2, za, zb, k, pi, row0, permute):
    perm_a = np.random.default_rng(1).permutation(n1) if permute else None
    perm_b = np.random.default_rng(2).permutation(n2) if permute else None
    A = _csr(d, n1, za, 3, 0, perm_a)
    B = _csr(d, n2, zb, 3, 1, perm_b)
    half = d // 3
    sk, fin = gpu_sketch_csr(d, n1, n2, k, PI[pi], 11, A, B, row0=row0,
                             splits=[(half, d), (0, half)])   # blocks in any order
    skA, a2 = oracle.sketch_csr(PI[pi], 11, k, n1, A[0].numpy(), A[1].numpy(), A[2].numpy(), row0=row0)
    skB, b2 = oracle.sketch_csr(PI[pi], 11, k, n2, B[0].numpy(), B[1].numpy(), B[2].numpy(), row0=row0)
    As, _, _ = oracle.finalize(k, skA, a2)
    Bs, _, _ = oracle.finalize(k, skB, b2)
    ea = col_rel_err(fin["A_sk"], As)
    eb = col_rel_err(fin["B_sk"], Bs)
    assert ea.max() <= 1e-5 and eb.max() <= 1e-5, (ea.max(), eb.max())
    # integer counts: fp64 norms are exact sums of exact squares -> bit-exact
    assert np.array_equal(fin["a_norm2"].cpu().numpy(), a2)
    assert np.array_equal(fin["b_norm2"].cpu().numpy(), b2)
    # Ω is therefore bit-exact too
    m = 4 * max(n1, n2) * 5 * math.log(max(n1, n2))
    I, J, val, qh = sk.sample_estimate(m, 5)
    al, be = oracle.alpha_beta(a2, b2, oracle.pairwise_sum(a2), oracle.pairwise_sum(b2))
    Io, Jo, qo = oracle.sample(5, m, al, be)
    assert np.array_equal(I.cpu().numpy(), Io) and np.array_equal(J.cpu().numpy(), Jo)


@pytest.mark.parametrize("density,frac_vals,chunk", [
    ("0", False, None),       # no tensor-core head: every nonzero through the sorted tail
    ("1e-9", False, None),    # every non-empty column is a head column
    ("0.02", True, None),     # head columns holding non-4-bit values: those entries stay in the tail
    ("0.02", True, "32768"),  # 3 head chunks: head K1 on the side stream, double-buffered
])
def test_sketch_csr_head_split_parity(density, frac_vals, chunk, monkeypatch):
    """The head/tail split of K3 never changes the result:
    the same CSR sketched with no head, an all-head split, head columns
    that carry values tcgen05 cannot take exactly (R21), and the head K1 of
    one chunk overlapped with the next chunk's tail all match the oracle."""
    monkeypatch.setenv("SMP_CSR_HEAD_DENSITY", density)
    if chunk:
        monkeypatch.setenv("SMP_CSR_HEAD_CHUNK", chunk)
        monkeypatch.setenv("SMP_CSR_HEAD_OVERLAP", "1")
    d, n1, n2, k = (70000 if chunk else 40000), 90, 70, 200
    A = _csr(d, n1, 12, 8, 0)
    B = _csr(d, n2, 9, 8, 1)
    if frac_vals:   # every 7th entry gets a value with > 4 significant bits
        for rp, col, val in (A, B):
            val[::7] = val[::7] * 1.3 + 0.01
    half = 20001   # a block boundary inside a Π panel, not 4-row aligned (generic Π panel path)
    sk, fin = gpu_sketch_csr(d, n1, n2, k, PI["gaussian"], 13, A, B, splits=[(0, half), (half, d)])
    skA, a2 = oracle.sketch_csr(PI["gaussian"], 13, k, n1, A[0].numpy(), A[1].numpy(), A[2].numpy())
    skB, b2 = oracle.sketch_csr(PI["gaussian"], 13, k, n2, B[0].numpy(), B[1].numpy(), B[2].numpy())
    As, _, _ = oracle.finalize(k, skA, a2)
    Bs, _, _ = oracle.finalize(k, skB, b2)
    ea = col_rel_err(fin["A_sk"], As)
    eb = col_rel_err(fin["B_sk"], Bs)
    assert ea.max() <= 1e-5 and eb.max() <= 1e-5, (ea.max(), eb.max())
    if frac_vals:
        np.testing.assert_allclose(fin["a_norm2"].cpu().numpy(), a2, rtol=1e-12)
        np.testing.assert_allclose(fin["b_norm2"].cpu().numpy(), b2, rtol=1e-12)
    else:
        assert np.array_equal(fin["a_norm2"].cpu().numpy(), a2)
        assert np.array_equal(fin["b_norm2"].cpu().numpy(), b2)


def test_sketch_csr_many_columns_radix_path():
    """More columns than the SMEM counting sort holds (ntot > 40960): the
    per-panel radix-sort path of K3, no tensor-core head."""
    d, n1, n2, k = 3000, 30000, 20000, 96
    A = _csr(d, n1, 6, 4, 0)
    B = _csr(d, n2, 5, 4, 1)
    sk, fin = gpu_sketch_csr(d, n1, n2, k, PI["gaussian"], 17, A, B, splits=[(0, 1000), (1000, d)])
    skA, a2 = oracle.sketch_csr(PI["gaussian"], 17, k, n1, A[0].numpy(), A[1].numpy(), A[2].numpy())
    skB, b2 = oracle.sketch_csr(PI["gaussian"], 17, k, n2, B[0].numpy(), B[1].numpy(), B[2].numpy())
    As, _, _ = oracle.finalize(k, skA, a2)
    Bs, _, _ = oracle.finalize(k, skB, b2)
    assert col_rel_err(fin["A_sk"], As).max() <= 1e-5 and col_rel_err(fin["B_sk"], Bs).max() <= 1e-5
    assert np.array_equal(fin["a_norm2"].cpu().numpy(), a2)
    assert np.array_equal(fin["b_norm2"].cpu().numpy(), b2)


def test_sketch_csr_dense_and_empty_rows():
    """Ragged CSR: a row holding every column of A (30,000 nonzeros: a scatter
    batch of its own, beyond the per-batch row-id capacity), runs of empty
    rows, and rows of one nonzero, with the tensor-core head on."""
    d, n1, n2, k = 3000, 30000, 9000, 64
    rng = np.random.default_rng(5)
    cols_a, cols_b, rpa, rpb = [], [], [0], [0]
    for t in range(d):
        if t == 1234:
            ca = np.arange(n1)
        elif 500 <= t < 700:
            ca = np.array([], dtype=np.int64)
        elif t % 97 == 0:
            ca = rng.choice(n1, 1)
        else:
            ca = np.sort(rng.choice(n1, 6, replace=False))
        cb = np.array([], dtype=np.int64) if 600 <= t < 900 else np.sort(rng.choice(n2, 4, replace=False))
        cols_a.append(ca)
        cols_b.append(cb)
        rpa.append(rpa[-1] + len(ca))
        rpb.append(rpb[-1] + len(cb))
    ca = np.concatenate(cols_a).astype(np.int32)
    cb = np.concatenate(cols_b).astype(np.int32)
    va = rng.integers(1, 6, len(ca)).astype(np.float32)
    vb = rng.integers(1, 6, len(cb)).astype(np.float32)
    A = (torch.tensor(rpa, dtype=torch.int64), torch.from_numpy(ca), torch.from_numpy(va))
    B = (torch.tensor(rpb, dtype=torch.int64), torch.from_numpy(cb), torch.from_numpy(vb))
    sk, fin = gpu_sketch_csr(d, n1, n2, k, PI["gaussian"], 19, A, B, splits=[(0, 1500), (1500, d)])
    skA, a2 = oracle.sketch_csr(PI["gaussian"], 19, k, n1, A[0].numpy(), A[1].numpy(), A[2].numpy())
    skB, b2 = oracle.sketch_csr(PI["gaussian"], 19, k, n2, B[0].numpy(), B[1].numpy(), B[2].numpy())
    As, _, _ = oracle.finalize(k, skA, a2)
    Bs, _, _ = oracle.finalize(k, skB, b2)
    assert col_rel_err(fin["A_sk"], As).max() <= 1e-5 and col_rel_err(fin["B_sk"], Bs).max() <= 1e-5
    assert np.array_equal(fin["a_norm2"].cpu().numpy(), a2)
    assert np.array_equal(fin["b_norm2"].cpu().numpy(), b2)


def test_sketch_csr_bad_column_rejected():
    smp = _smp()
    d, n = 100, 10
    rp = torch.arange(0, d + 1, dtype=torch.int64) * 2
    col = torch.zeros(2 * d, dtype=torch.int32)
    col[17] = n + 3   # out of range
    val = torch.ones(2 * d)
    sk = smp.SMPSketch(d, n, n, 32, pi=0, seed=0, input=smp.IN_CSR_F32)
    sk.block_csr(0, d, rp.cuda(), col.cuda(), val.cuda(), rp.cuda(), torch.zeros_like(col).cuda(), val.cuda())
    with pytest.raises(Exception):
        sk.finalize()


@pytest.mark.parametrize("pi", ["gaussian", "rademacher", "srht"])
def test_pi_bit_exact_sampled_rows(pi):
    """Π itself, bit for bit: X has one 1 per column at a random row t_c over
    a long row range, so Ã[:, c]·√k = Π[:, t_c] exactly (a1, R2/R3)."""
    smp = _smp()
    d, n, k, seed = 1 << 21, 256, 512, 4
    rng = np.random.default_rng(7)
    t = np.sort(rng.choice(d, n, replace=False))
    X = torch.zeros(d, n, dtype=torch.bfloat16)
    X[torch.as_tensor(t), torch.arange(n)] = 1.0
    gpu_kind = smp.PI_SRHT if pi == "srht" else PI[pi]
    or_kind = oracle.pi_srht(d) if pi == "srht" else PI[pi]
    sk = smp.SMPSketch(d, n, n, k, pi=gpu_kind, seed=seed, a_is_b=True, input=smp.IN_DENSE_BF16)
    sk.block(0, X.cuda())
    fin = sk.finalize()
    got = fin["A_sk"].cpu().numpy()                       # fp32: Π(κ, t_c) · fp32(1/√k), RN
    want = np.array([[oracle.pi_entry(or_kind, seed, kap, int(tc)) for kap in range(k)] for tc in t])
    want32 = want.astype(np.float32) * np.float32(1.0 / np.sqrt(k))
    bad = got != want32
    assert bad.sum() == 0, f"{bad.sum()} of {bad.size} Π entries differ, e.g. {np.argwhere(bad)[:5]}"


# ------------------------------------------------------------------ SRHT (NEXT-1, R26)
@pytest.mark.parametrize("d,n,k,row0,blocks", [
    (3000, 300, 256, 0, None),            # several n-tiles, Hadamard order 4096
    (2500, 96, 130, 77, [(900, 2500), (0, 900)]),   # unaligned rows (generic path), ragged k
])
def test_sketch_srht_parity(d, n, k, row0, blocks):
    smp = _smp()
    A = synth.gaussian_small(d, n, seed=1, scale_cols=True).to(torch.bfloat16)
    B = synth.gaussian_small(d, n, seed=2).to(torch.bfloat16)
    dt = row0 + d
    _, fin = gpu_sketch(A, B, k, smp.PI_SRHT, seed=5, row0=row0, d_total=dt, blocks=blocks)
    kind = oracle.pi_srht(dt)
    orc = oracle_sketch(A, B, k, kind, seed=5, row0=row0)
    check_sketch(fin, orc)


def test_sketch_csr_srht_parity():
    smp = _smp()
    d, n1, n2, k = 2000, 120, 80, 128
    A = _csr(d, n1, 10, 5, 0)
    B = _csr(d, n2, 8, 5, 1)
    sk, fin = gpu_sketch_csr(d, n1, n2, k, smp.PI_SRHT, 11, A, B)
    kind = oracle.pi_srht(d)
    skA, a2 = oracle.sketch_csr(kind, 11, k, n1, A[0].numpy(), A[1].numpy(), A[2].numpy())
    skB, b2 = oracle.sketch_csr(kind, 11, k, n2, B[0].numpy(), B[1].numpy(), B[2].numpy())
    As, _, _ = oracle.finalize(k, skA, a2)
    Bs, _, _ = oracle.finalize(k, skB, b2)
    assert col_rel_err(fin["A_sk"], As).max() <= 1e-5 and col_rel_err(fin["B_sk"], Bs).max() <= 1e-5
    assert np.array_equal(fin["a_norm2"].cpu().numpy(), a2)


def test_srht_full_rank_exact_product():
    """SRHT with k = d = 2^L: M̃ = AᵀB (fully sampled), as with Hadamard."""
    smp = _smp()
    d, n = 256, 24
    A = synth.gaussian_small(d, n, seed=11).to(torch.bfloat16)
    B = synth.gaussian_small(d, n, seed=12).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, d, smp.PI_SRHT, seed=3)
    I, J, val, qh = sk.sample_estimate(1e12, 0)
    assert I.numel() == n * n
    M = (A.double().T @ B.double()).numpy()
    got = np.zeros((n, n))
    got[I.cpu().numpy(), J.cpu().numpy()] = val.cpu().numpy()
    scale = np.outer(np.linalg.norm(A.double().numpy(), axis=0), np.linalg.norm(B.double().numpy(), axis=0))
    assert np.max(np.abs(got - M) / scale) < 1e-5


# ------------------------------------------------------------------ row-multinomial Ω (NEXT-2, R27)
@pytest.mark.parametrize("n1,n2,m_coef,ties", [(100, 100, 0.3, False), (600, 450, 4.0, False),
                                                (300, 257, 50.0, False), (200, 150, 8.0, True)])
def test_multinomial_omega_bit_exact(n1, n2, m_coef, ties):
    """R27 Ω (saturated prefix ∪ distinct row-multinomial draws) bit-exact,
    q̂ within 1e-12 relative; ties: duplicated B columns give equal β, so
    σ's tie order (column index) decides the draws."""
    d, k = 3000, 128
    A = synth.gaussian_small(d, n1, seed=21, scale_cols=True).to(torch.bfloat16)
    B = synth.gaussian_small(d, n2, seed=22, scale_cols=True).to(torch.bfloat16)
    if ties:
        B[:, 10:20] = B[:, 30:40]
        B[:, 100] = B[:, 5]
    sk, fin = gpu_sketch(A, B, k, 0, seed=3)
    orc = oracle_sketch(A, B, k, 0, seed=3)
    m = m_coef * max(n1, n2) * 5 * math.log(max(n1, n2))
    I, J, val, qh = sk.sample_estimate(m, 99, sampler="multinomial")
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    if ties:
        assert len(np.unique(be)) < n2
    Io, Jo, qo = oracle.sample_multinomial(99, m, al, be)
    assert np.array_equal(I.cpu().numpy(), Io) and np.array_equal(J.cpu().numpy(), Jo)
    np.testing.assert_allclose(qh.cpu().numpy(), qo, rtol=2 * NORM_RTOL)
    if m_coef >= 8:
        assert (qo == 1.0).sum() > 0 and (qo < 1.0).sum() > 0     # saturated and drawn pairs
    Mo = oracle.estimate(k, Io, Jo, orc["As"], orc["Bs"], orc["DA"], orc["DB"])
    scale = np.sqrt(orc["a2"][Io] * orc["b2"][Jo])
    assert np.max(np.abs(val.cpu().double().numpy() - Mo) / scale) <= 1e-4


def test_multinomial_pipeline_waltmin():
    """Alg. 1 with the multinomial Ω end to end: the factors agree with the
    oracle run on the same (oracle) Ω to 1e-3 of ||AᵀB||."""
    smp = _smp()
    d, n, r, k = 8192, 256, 5, 256
    VA = synth.lowrank_factors(n, 20, 1, 0, "cpu")
    VB = synth.lowrank_factors(n, 20, 1, 1, "cpu")
    A, B = synth.lowrank_block(0, d, n, 1, VA, VB, device="cpu")
    sk, fin = gpu_sketch(A, B, k, 0, seed=1)
    orc = oracle_sketch(A, B, k, 0, seed=1)
    m = 4 * n * r * math.log(n)
    I, J, val, qh = sk.sample_estimate(m, 1, sampler="multinomial")
    Ug, Vg = sk.waltmin(I, J, val, qh, r, 10, init_iters=30, seed=1)
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    Io, Jo, qo = oracle.sample_multinomial(1, m, al, be)
    Mo = oracle.estimate(k, Io, Jo, orc["As"], orc["Bs"], orc["DA"], orc["DB"])
    Uo, Vo = oracle.waltmin(n, n, r, 10, Io, Jo, Mo, qo, np.sqrt(orc["a2"]), math.sqrt(orc["FA"]),
                            init_iters=30, seed=1)
    M = (A.double().T @ B.double()).numpy()
    assert _uvt_err(Ug.cpu().double().numpy(), Vg.cpu().double().numpy(), Uo, Vo, M) <= 1e-3


# ------------------------------------------------------------------ SVD(ÃᵀB̃) baseline (NEXT-4)
def test_svd_of_sketch_baseline_and_accuracy_claim():
    """The GPU rank-r SVD of ÃᵀB̃ matches numpy's SVD of the oracle's sketch
    product, and on a narrow shared-axis cone SMP-PCA beats it."""
    smp = _smp()
    d, n, r, k = 4000, 80, 3, 256
    A64, B64 = synth.cone_shared_axis(d, n, 0.3, seed=5)
    A, B = A64.float(), B64.float()
    sk, fin = gpu_sketch(A, B, k, smp.PI_GAUSSIAN, seed=3)
    orc = oracle_sketch(A, B, k, 1, seed=3)
    Ms = orc["As"] @ orc["Bs"].T
    u, sv, vt = np.linalg.svd(Ms)
    best = (u[:, :r] * sv[:r]) @ vt[:r]
    M = (A64.T @ B64).numpy()
    Us, Vs = sk.svd_of_sketch(r, seed=3)
    Pg = Us.cpu().double().numpy() @ Vs.cpu().double().numpy().T
    assert np.linalg.norm(Pg - best, 2) / np.linalg.norm(M, 2) <= 1e-3
    m = 6 * n * r * math.log(n)
    I, J, val, qh = sk.sample_estimate(m, 3)
    U, V = sk.waltmin(I, J, val, qh, r, 10, init_iters=30, seed=3)
    nrm = np.linalg.norm(M, 2)
    err = np.linalg.norm(U.cpu().double().numpy() @ V.cpu().double().numpy().T - M, 2) / nrm
    err_svd = np.linalg.norm(Pg - M, 2) / nrm
    assert err <= err_svd, (err, err_svd)


# ------------------------------------------------------------------ FRESH_2T1 partition (Alg. 2 line 3, R11)
@pytest.mark.parametrize("n1,n2,r,T,m_coef", [(150, 120, 3, 3, 20.0), (400, 300, 5, 5, 30.0)])
def test_waltmin_fresh_partition_identical_inputs(n1, n2, r, T, m_coef):
    """FRESH_2T1: Ω split into 2T+1 random subsets (init on Ω_0, V-step t on
    Ω_{2t+1}, U-step on Ω_{2t+2}); GPU vs oracle on identical inputs, and the
    result differs from REUSE_ALL (the partition is really applied)."""
    d, k = 2000, 256
    Z = synth.gaussian_small(d, r, seed=81).double()
    A = (Z @ synth.gaussian_small(r, n1, seed=82).double() + 0.1 * synth.gaussian_small(d, n1, seed=83).double()).to(torch.bfloat16)
    B = (Z @ synth.gaussian_small(r, n2, seed=84).double() + 0.1 * synth.gaussian_small(d, n2, seed=85).double()).to(torch.bfloat16)
    sk, fin = gpu_sketch(A, B, k, 0, seed=1)
    orc = oracle_sketch(A, B, k, 0, seed=1)
    m = m_coef * max(n1, n2) * r * math.log(max(n1, n2))
    al, be = oracle.alpha_beta(orc["a2"], orc["b2"], orc["FA"], orc["FB"])
    Io, Jo, qo = oracle.sample(5, m, al, be)
    Mo = oracle.estimate(k, Io, Jo, orc["As"], orc["Bs"], orc["DA"], orc["DB"]).astype(np.float32)
    Uo, Vo = oracle.waltmin(n1, n2, r, T, Io, Jo, Mo.astype(np.float64), qo, np.sqrt(orc["a2"]),
                            math.sqrt(orc["FA"]), init_iters=30, seed=9, partition=oracle.PART_FRESH_2T1)
    dev = torch.device("cuda")
    args = (torch.tensor(Io, device=dev), torch.tensor(Jo, device=dev), torch.tensor(Mo, device=dev),
            torch.tensor(qo, device=dev), r, T)
    Ug, Vg = sk.waltmin(*args, init_iters=30, seed=9, partition="fresh_2t1")
    M = (A.double().T @ B.double()).numpy()
    Ug, Vg = Ug.cpu().double().numpy(), Vg.cpu().double().numpy()
    assert _uvt_err(Ug, Vg, Uo, Vo, M) <= 1e-3
    Ur, Vr = sk.waltmin(*args, init_iters=30, seed=9)
    assert _uvt_err(Ug, Vg, Ur.cpu().double().numpy(), Vr.cpu().double().numpy(), M) > 1e-6


def test_waltmin_fresh_partition_needs_2t_plus_1_samples():
    smp = _smp()
    A = synth.gaussian_small(256, 20, seed=1).to(torch.bfloat16)
    B = synth.gaussian_small(256, 20, seed=2).to(torch.bfloat16)
    sk, _ = gpu_sketch(A, B, 32, 0)
    dev = torch.device("cuda")
    I = torch.arange(6, dtype=torch.int32, device=dev)
    J = torch.arange(6, dtype=torch.int32, device=dev)
    val = torch.ones(6, device=dev)
    q = torch.ones(6, dtype=torch.float64, device=dev)
    with pytest.raises(smp.SmpError) as e:
        sk.waltmin(I, J, val, q, 2, 3, partition="fresh_2t1")   # 6 < 2·3+1
    assert e.value.status == 3


# ------------------------------------------------------------------ LELA (NEXT-3)
@pytest.mark.parametrize("dtype,d,n1,n2,blocks", [
    ("bf16", 5000, 130, 97, [(0, 5000)]),
    ("f32", 3001, 200, 150, [(1700, 3001), (0, 64), (64, 1700)]),   # ragged chunks, blocks in any order
])
def test_lela_two_pass_parity(dtype, d, n1, n2, blocks):
    """LELA through the C ABI: pass 1 norms (fp64, ~exact), Ω bit-exact with
    the oracle's Eq. 1 sample, pass 2 exact entries (AᵀB)_Ω within 1e-9 of
    ||A_i|| ||B_j||, and WAltMin on them within 1e-3 of ||AᵀB|| (end to end)."""
    smp = _smp()
    r = 5
    Z = synth.gaussian_small(d, r, seed=91).double()
    A = Z @ synth.gaussian_small(r, n1, seed=92).double() + 0.2 * synth.gaussian_small(d, n1, seed=93).double()
    B = Z @ synth.gaussian_small(r, n2, seed=94).double() + 0.2 * synth.gaussian_small(d, n2, seed=95).double()
    A = A.to(torch.bfloat16 if dtype == "bf16" else torch.float32)
    B = B.to(torch.bfloat16 if dtype == "bf16" else torch.float32)
    inp = smp.IN_DENSE_BF16 if dtype == "bf16" else smp.IN_DENSE_F32
    m = 4 * max(n1, n2) * r * math.log(max(n1, n2))
    sk = smp.SMPSketch(d, n1, n2, 1, input=inp)
    Ad, Bd = A.cuda(), B.cuda()
    for r0, r1 in blocks:
        sk.norms_block(r0, Ad[r0:r1], Bd[r0:r1])
    fin = sk.finalize()
    Ah, Bh = _to_np(A), _to_np(B)
    orc = oracle.lela(Ah, Bh, r, m, 10, seed=4, init_iters=30)
    np.testing.assert_allclose(fin["a_norm2"].cpu().numpy(), orc["a2"], rtol=1e-12)
    np.testing.assert_allclose(fin["b_norm2"].cpu().numpy(), orc["b2"], rtol=1e-12)
    I, J, _, qh = sk.sample_estimate(m, 4)
    assert np.array_equal(I.cpu().numpy(), orc["I"]) and np.array_equal(J.cpu().numpy(), orc["J"])
    acc = torch.zeros(I.numel(), dtype=torch.float64, device="cuda")
    for r0, r1 in blocks:
        sk.exact_entries_block(r0, Ad[r0:r1], Bd[r0:r1], I, J, acc)
    scale = np.sqrt(orc["a2"][orc["I"]] * orc["b2"][orc["J"]])
    assert np.max(np.abs(acc.cpu().numpy() - orc["M"]) / scale) <= 1e-9
    U, V = sk.waltmin(I, J, acc.float(), qh, r, 10, init_iters=30, seed=4)
    M = (A.double().T @ B.double()).numpy()
    assert _uvt_err(U.cpu().double().numpy(), V.cpu().double().numpy(), orc["U"], orc["V"], M) <= 1e-3
    # the one-call driver gives the same factors
    res = smp.lela(Ad, Bd, r, m, 10, seed=4, init_iters=30)
    assert torch.equal(res["I"], I) and torch.equal(res["J"], J)
    assert _uvt_err(res["U"].cpu().double().numpy(), res["V"].cpu().double().numpy(), orc["U"], orc["V"], M) <= 1e-3
