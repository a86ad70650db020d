"""GPU parity at BASELINE.json's FULL sizes, in the launch configuration
bench.py times (one SMPSketch over all d rows, the same synthetic inputs),
checked against the CPU oracle on sampled outputs it can compute exactly:

  * sketch columns Ã_i, B̃_j for a sample of columns over the full d
    (columns are independent, so this is exact per column);
  * their column norms;
  * cfg1-cfg4: Ω bit-exact over all n1·n2 pairs from the oracle's own full
    column norms, and M̃ on Ω ∩ (sampled A columns × sampled B columns);
  * cfg1-cfg4: WAltMin (bench's r, T, init_iters) on identical inputs — the
    GPU's Ω, M̃, q̂ fed to oracle.waltmin — with
    ||UVᵀ_gpu − UVᵀ_or||_2 / ||AᵀB||_2 <= 1e-3, ||AᵀB||_2 of the implicit
    product by power iteration (north-star factor tolerance).

Tolerances as in test_gpu_parity.py.
"""
import math

import numpy as np
import pytest
import torch

import bench
import oracle
import synth

from test_gpu_parity import NORM_RTOL, col_rel_err

pytestmark = pytest.mark.gpu

PI = {"rademacher": 0, "gaussian": 1}


def _smp():
    import paper_1610_06656_b200 as smp
    return smp


def _host(X):
    return synth.bf16_bits(X) if X.dtype == torch.bfloat16 else X.numpy()


def _sample_cols(n, count, seed):
    rng = np.random.default_rng(seed)
    pick = set([0, n - 1]) | set(rng.choice(n, count - 2, replace=False).tolist())
    return np.array(sorted(pick), dtype=np.int64)


def _oracle_cols(cfg, X, cols):
    """Oracle sketch (scaled), norms² and D of the sampled columns over all d rows."""
    sub = X[:, torch.as_tensor(cols, device=X.device)].contiguous().cpu()
    sk, n2 = oracle.sketch_rows(PI[cfg["pi"]], cfg["seed"], cfg["k"], _host(sub))
    S, sn, D = oracle.finalize(cfg["k"], sk, n2)
    return S, n2, D


def _oracle_full_norms(X, block=1 << 16):
    n2 = np.zeros(X.shape[1], np.float64)
    for r0 in range(0, X.shape[0], block):
        oracle.colnorms(_host(X[r0:r0 + block].cpu()), n2)
    return n2


def _lowrank_diff_norm(U1, V1, U2, V2):
    """||U1 V1ᵀ − U2 V2ᵀ||_2 from the factors (rank <= 2r, no n1 x n2 matrix)."""
    Qa, Ra = np.linalg.qr(np.hstack([U1, U2]))
    Qb, Rb = np.linalg.qr(np.hstack([V1, -V2]))
    return np.linalg.norm(Ra @ Rb.T, 2)


def _power_norm(matvec, rmatvec, n, iters=40, seed=0):
    """||M||_2 of an implicit M (n columns) by power iteration on MᵀM."""
    v = torch.randn(n, generator=torch.Generator().manual_seed(seed), dtype=torch.float64)
    v /= v.norm()
    lam = 0.0
    for _ in range(iters):
        w = rmatvec(matvec(v))
        lam = float(w.norm())
        v = w / lam
    return math.sqrt(lam)


def _dense_ops(A, B, chunk=1 << 18):
    """x -> AᵀB x and y -> BᵀA y on device-resident row-major A, B (fp32
    accumulation, fp64 vectors; test infrastructure, not the method)."""
    dev = A.device

    def mv(X, Y, x):  # Xᵀ (Y x)
        xd = x.to(dev, torch.float32)
        out = torch.zeros(X.shape[1], dtype=torch.float64, device=dev)
        for r0 in range(0, X.shape[0], chunk):
            t = Y[r0:r0 + chunk].float() @ xd
            out += (X[r0:r0 + chunk].float().T @ t).double()
        return out.cpu()
    return (lambda x: mv(A, B, x)), (lambda y: mv(B, A, y))


def _check_waltmin_identical(sk, cfg, I, J, val, qh, a2, FA, normM, tag):
    """GPU WAltMin vs oracle WAltMin on the GPU's own Ω, M̃, q̂ (bench's r, T,
    init_iters = 30, seed)."""
    r, T, n1, n2 = cfg["r"], cfg["T"], cfg["n1"], cfg["n2"]
    Ug, Vg = sk.waltmin(I, J, val, qh, r, T, init_iters=30, seed=cfg["seed"])
    Uo, Vo = oracle.waltmin(n1, n2, r, T, I.cpu().numpy(), J.cpu().numpy(),
                            val.cpu().double().numpy(), qh.cpu().numpy(), np.sqrt(a2), math.sqrt(FA),
                            init_iters=30, seed=cfg["seed"])
    err = _lowrank_diff_norm(Ug.cpu().double().numpy(), Vg.cpu().double().numpy(), Uo, Vo) / normM
    assert err <= 1e-3, f"{tag}: factor parity {err:.3e}"
    return err


def _free(*xs):
    for x in xs:
        del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("cfgname,ns,full_omega", [("cfg1", 16, True), ("cfg4", 12, True),
                                                     ("cfg2", 8, True)])
def test_dense_full_size(cfgname, ns, full_omega):
    smp = _smp()
    cfg = synth.CONFIGS[cfgname]
    d, n1, n2, k = cfg["d"], cfg["n1"], cfg["n2"], cfg["k"]
    a_is_b = cfg.get("a_is_b", False)
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(cfgname, cfg, 0, d, dev)
    inp = smp.IN_DENSE_BF16 if A.dtype == torch.bfloat16 else smp.IN_DENSE_F32
    sk = smp.SMPSketch(d, n1, n2, k, pi=PI[cfg["pi"]], seed=cfg["seed"], a_is_b=a_is_b, input=inp,
                       device=dev)
    sk.block(0, A, None if a_is_b else B)
    fin = sk.finalize()

    ca = _sample_cols(n1, ns, 1)
    As, a2s, DA = _oracle_cols(cfg, A, ca)
    ea = col_rel_err(fin["A_sk"][torch.as_tensor(ca, device=dev)], As)
    assert ea.max() <= 1e-5, f"{cfgname}: A sketch max col rel err {ea.max():.3e}"
    np.testing.assert_allclose(fin["a_norm2"].cpu().numpy()[ca], a2s, rtol=NORM_RTOL)
    if not a_is_b:
        cb = _sample_cols(n2, ns, 2)
        Bs, b2s, DB = _oracle_cols(cfg, B, cb)
        eb = col_rel_err(fin["B_sk"][torch.as_tensor(cb, device=dev)], Bs)
        assert eb.max() <= 1e-5, f"{cfgname}: B sketch max col rel err {eb.max():.3e}"
        np.testing.assert_allclose(fin["b_norm2"].cpu().numpy()[cb], b2s, rtol=NORM_RTOL)

    if full_omega:
        a2 = _oracle_full_norms(A)
        b2 = a2 if a_is_b else _oracle_full_norms(B)
        if a_is_b:
            cb, Bs, DB = ca, As, DA
        np.testing.assert_allclose(fin["a_norm2"].cpu().numpy(), a2, rtol=NORM_RTOL)
        np.testing.assert_allclose(fin["b_norm2"].cpu().numpy(), b2, rtol=NORM_RTOL)
        m = synth.m_of(cfg)
        I, J, val, qh = sk.sample_estimate(m, cfg["seed"])
        al, be = oracle.alpha_beta(a2, b2, oracle.pairwise_sum(a2), oracle.pairwise_sum(b2))
        Io, Jo, qo = oracle.sample(cfg["seed"], m, al, be)
        assert np.array_equal(I.cpu().numpy(), Io) and np.array_equal(J.cpu().numpy(), Jo), \
            f"Omega differs: {I.numel()} vs {len(Io)} samples"
        # M̃ on Ω ∩ (ca × cb), from the oracle's sketches of those columns
        Ih, Jh = I.cpu().numpy(), J.cpu().numpy()
        pa = {c: i for i, c in enumerate(ca)}
        pb = {c: i for i, c in enumerate(cb)}
        sel = np.array([s for s in range(len(Ih)) if Ih[s] in pa and Jh[s] in pb], dtype=np.int64)
        if len(sel):
            li = np.array([pa[c] for c in Ih[sel]], np.int32)
            lj = np.array([pb[c] for c in Jh[sel]], np.int32)
            Mo = oracle.estimate(k, li, lj, As, Bs, DA, DB)
            scale = np.sqrt(a2[Ih[sel]] * b2[Jh[sel]])
            err = np.abs(val.cpu().double().numpy()[sel] - Mo) / scale
            assert err.max() <= 1e-4, err.max()
        Bx = A if a_is_b else B
        mv, rmv = _dense_ops(A, Bx)
        normM = _power_norm(mv, rmv, n2)
        _check_waltmin_identical(sk, cfg, I, J, val, qh, a2, oracle.pairwise_sum(a2), normM, cfgname)
    sk.close()
    _free(A, B)


def test_csr_full_size_cfg3():
    """cfg3 (8e6 x (10^4 + 8000) CSR, Gaussian k = 512) at full size: sampled
    columns' sketches, exact norms of every column, Ω bit-exact."""
    smp = _smp()
    cfg = synth.CONFIGS["cfg3"]
    d, n1, n2, k = cfg["d"], cfg["n1"], cfg["n2"], cfg["k"]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs_csr(cfg, 0, d, dev)
    sk = smp.SMPSketch(d, n1, n2, k, pi=PI[cfg["pi"]], seed=cfg["seed"], input=smp.IN_CSR_F32,
                       device=dev)
    sk.block_csr(0, d, *A, *B)
    fin = sk.finalize()

    def restricted(X, cols):
        rp, col, val = X
        lut = torch.full((int(col.max()) + 1,), -1, dtype=torch.int32, device=dev)
        lut[torch.as_tensor(cols, device=dev)] = torch.arange(len(cols), dtype=torch.int32, device=dev)
        nc = lut[col.long()]
        keep = nc >= 0
        rows = torch.repeat_interleave(torch.arange(d, device=dev), rp[1:] - rp[:-1])
        cnt = torch.bincount(rows[keep], minlength=d)
        rp2 = torch.zeros(d + 1, dtype=torch.int64, device=dev)
        rp2[1:] = torch.cumsum(cnt, 0)
        return rp2.cpu().numpy(), nc[keep].cpu().numpy(), val[keep].cpu().numpy()

    for X, n, key, seed in ((A, n1, "A", 3), (B, n2, "B", 4)):
        rng = np.random.default_rng(seed)
        cols = np.array(sorted(set([50, n - 1] + rng.choice(np.arange(100, n), 8, replace=False).tolist())))
        rp2, c2, v2 = restricted(X, cols)
        skc, n2c = oracle.sketch_csr(PI[cfg["pi"]], cfg["seed"], k, len(cols), rp2, c2, v2)
        S, _, _ = oracle.finalize(k, skc, n2c)
        e = col_rel_err(fin[f"{key}_sk"][torch.as_tensor(cols, device=dev)], S)
        assert e.max() <= 1e-5, f"cfg3 {key} sketch max col rel err {e.max():.3e}"
        assert np.array_equal(fin[f"{key.lower()}_norm2"].cpu().numpy()[cols], n2c)

    # exact norms of every column (k = 1 oracle pass: Σ v² in row order), streamed
    def full_norms(X, n):
        rp, col, val = X
        nrm = np.zeros(n, np.float64)
        sk1 = np.zeros((n, 1), np.float64)
        step = 1 << 20
        for r0 in range(0, d, step):
            r1 = min(d, r0 + step)
            e0, e1 = int(rp[r0]), int(rp[r1])
            oracle.sketch_csr(PI[cfg["pi"]], cfg["seed"], 1, n, rp[r0:r1 + 1].cpu().numpy(),
                              col[e0:e1].cpu().numpy(), val[e0:e1].cpu().numpy(), row0=r0,
                              sk=sk1, norm2=nrm)
        return nrm

    a2 = full_norms(A, n1)
    b2 = full_norms(B, n2)
    assert np.array_equal(fin["a_norm2"].cpu().numpy(), a2)
    assert np.array_equal(fin["b_norm2"].cpu().numpy(), b2)
    m = synth.m_of(cfg)
    I, J, val, qh = sk.sample_estimate(m, cfg["seed"])
    al, be = oracle.alpha_beta(a2, b2, oracle.pairwise_sum(a2), oracle.pairwise_sum(b2))
    Io, Jo, qo = oracle.sample(cfg["seed"], m, al, be)
    assert np.array_equal(I.cpu().numpy(), Io) and np.array_equal(J.cpu().numpy(), Jo)
    # WAltMin on identical inputs; ||AᵀB||_2 by power iteration with CSR SpMVs
    def csr_t(X, n):
        rp, col, val = X
        return torch.sparse_csr_tensor(rp, col.long(), val.double(), size=(d, n))
    SA, SB = csr_t(A, n1), csr_t(B, n2)

    SAc = SA.to_sparse_coo().t().coalesce()
    SBc = SB.to_sparse_coo().t().coalesce()

    def mv(x):
        return torch.mv(SAc, torch.mv(SB, x.to(dev))).cpu()

    def rmv(y):
        return torch.mv(SBc, torch.mv(SA, y.to(dev))).cpu()
    normM = _power_norm(mv, rmv, n2)
    _check_waltmin_identical(sk, cfg, I, J, val, qh, a2, oracle.pairwise_sum(a2), normM, "cfg3")
    sk.close()
    _free(A, B)
