"""NEXT-3 on the GPU at reduced size: the paper's Table 1 synthetic instance
(reading R28: A = B = G·D, G i.i.d. N(0,1), D_ii = 1/i) with
n = d = 2000, r = 5, T = 10, m = 4 n r ln n, Gaussian Π — SMP-PCA and LELA
through the C ABI against the oracle on identical inputs, and the paper's
ordering of the three errors (optimal <= LELA <= SMP-PCA)."""
import math

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu

N, R, T, SEED = 2000, 5, 10, 3


def _gd(n):
    rng = np.random.default_rng(1)
    G = rng.standard_normal((n, n)).astype(np.float32)
    return (G * (1.0 / np.arange(1, n + 1, dtype=np.float32))).astype(np.float32)


@pytest.fixture(scope="module")
def instance():
    A = _gd(N)
    M = A.astype(np.float64).T @ A.astype(np.float64)
    s = np.linalg.svd(M, compute_uv=False)
    return A, M, s


def _err(M, s0, U, V):
    return float(np.linalg.norm(M - U @ V.T, 2) / s0)


@pytest.mark.parametrize("k", [256, 512])
def test_table1_reduced_smp_pca_and_lela(instance, k):
    import paper_1610_06656_b200 as smp
    A, M, s = instance
    m = 4 * N * R * math.log(N)
    Ad = torch.from_numpy(A).cuda()
    res = smp.smp_pca(Ad, None, k=k, r=R, m=m, T=T, pi=smp.PI_GAUSSIAN, seed=SEED, init_iters=30, a_is_b=True)
    orc = oracle.smp_pca(A, A, k, R, m, T, pi_kind=oracle.PI_GAUSSIAN, seed=SEED, init_iters=30, a_is_b=True)
    # Ω and its indices bit-exact; factors on identical arithmetic within the north-star 1e-3
    assert np.array_equal(res["I"].cpu().numpy(), orc["I"]) and np.array_equal(res["J"].cpu().numpy(), orc["J"])
    Ug, Vg = res["U"].cpu().double().numpy(), res["V"].cpu().double().numpy()
    par = np.linalg.norm(Ug @ Vg.T - orc["U"] @ orc["V"].T, 2) / s[0]
    assert par <= 1e-3, par

    lg = smp.lela(Ad, None, R, m, T, seed=SEED, init_iters=30, a_is_b=True)
    lo = oracle.lela(A, A, R, m, T, seed=SEED, init_iters=30)
    assert np.array_equal(lg["I"].cpu().numpy(), lo["I"])
    Ul, Vl = lg["U"].cpu().double().numpy(), lg["V"].cpu().double().numpy()
    assert np.linalg.norm(Ul @ Vl.T - lo["U"] @ lo["V"].T, 2) / s[0] <= 1e-3

    opt = s[R] / s[0]                   # optimal rank-r error sigma_{r+1}/sigma_1
    e_smp = _err(M, s[0], Ug, Vg)
    e_lela = _err(M, s[0], Ul, Vl)
    # Optimal 0.0271 <= LELA 0.0274 <= SMP-PCA 0.0280 (here 0.0276 / 0.0276 / ~0.034)
    assert opt <= e_lela * (1 + 1e-6) and e_lela <= e_smp, (opt, e_lela, e_smp)
    assert e_lela <= 1.01 * opt and e_smp <= 1.3 * opt, (opt, e_lela, e_smp)
