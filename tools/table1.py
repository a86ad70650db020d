"""NEXT-3: the paper's Table 1 synthetic instance at full scale on
one B200 — A = B = G D with G i.i.d. N(0,1) and D_ii = 1/i, d = n = 100,000
(reading R28: "A and B as GD" with the same G — its optimal
rank-5 error σ6/σ1 ≈ 1/36 matches the printed 0.0271, while independent G's
give 0.055 at this size and 0.24 at n = 1500, where the oracle itself fails),
r = 5, T = 10, m = 4 n r ln n,
sketch size k = 2,000 — through the library's C ABI (fp32 inputs: K1F; the
Ω sampler and Π are selectable), and the spectral error of the result
against ‖AᵀB‖₂ next to the optimal rank-r error σ_{r+1}/σ_1, both estimated
by block power iteration on the implicit product (AᵀB is never formed; the
evaluation uses torch GEMMs on the resident A, B — it is not part of the
method).  Printed numbers: Optimal 0.0271, LELA 0.0274,
SMP-PCA 0.0280.  LELA (the two-pass comparison) runs through the same
C ABI: pass 1 smp_norms_block, Ω by Eq. 1 (Bernoulli), pass 2
smp_exact_entries_block, WAltMin.

    python tools/table1.py [n] [k] [multinomial|bernoulli] [gaussian|srht|rademacher] [lela|nolela]
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1610_06656_b200 import IN_DENSE_F32, PI_GAUSSIAN, PI_RADEMACHER, PI_SRHT, SMPSketch  # noqa: E402


def gd(d, n, seed, dev, block=8192):
    """A = G D (fp32), generated block by block on the device."""
    g = torch.Generator(device=dev).manual_seed(seed)
    Dg = 1.0 / torch.arange(1, n + 1, device=dev, dtype=torch.float32)
    X = torch.empty(d, n, device=dev, dtype=torch.float32)
    for r0 in range(0, d, block):
        r1 = min(d, r0 + block)
        X[r0:r1] = torch.randn(r1 - r0, n, generator=g, device=dev) * Dg
    return X


def top_singular(A, B, p=8, iters=30, seed=0):
    """Top-p singular values of AᵀB by block subspace iteration (fp32 GEMMs)."""
    n = A.shape[1]
    g = torch.Generator(device=A.device).manual_seed(seed)
    Y = torch.randn(n, p, generator=g, device=A.device)
    for _ in range(iters):
        Z, _ = torch.linalg.qr(A.T @ (B @ Y))
        Y, R = torch.linalg.qr(B.T @ (A @ Z))
    return torch.linalg.svdvals(R.double())


def err_norm(A, B, U, V, iters=40, seed=1):
    """‖AᵀB − UVᵀ‖₂ by power iteration on the implicit residual."""
    n = A.shape[1]
    g = torch.Generator(device=A.device).manual_seed(seed)
    x = torch.randn(n, 1, generator=g, device=A.device)
    x /= x.norm()
    s = 0.0
    for _ in range(iters):
        y = A.T @ (B @ x) - U @ (V.T @ x)
        z = B.T @ (A @ y) - V @ (U.T @ y)
        s = float(z.norm()) ** 0.5
        x = z / z.norm()
    return s


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    k = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    sampler = sys.argv[3] if len(sys.argv) > 3 else "multinomial"
    pi_name = sys.argv[4] if len(sys.argv) > 4 else "gaussian"
    pi = {"gaussian": PI_GAUSSIAN, "srht": PI_SRHT, "rademacher": PI_RADEMACHER}[pi_name]
    run_lela = (sys.argv[5] if len(sys.argv) > 5 else "lela") == "lela"
    d, r, T = n, 5, 10
    m = 4 * n * r * math.log(n)
    dev = torch.device("cuda", 0)
    A = gd(d, n, 1, dev)
    B = A
    torch.cuda.synchronize()
    t0 = time.time()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    sk = SMPSketch(d, n, n, k, pi=pi, seed=7, a_is_b=True, input=IN_DENSE_F32, device=dev)
    e[0].record()
    sk.block(0, A)
    sk.finalize()
    e[1].record()
    I, J, val, qh = sk.sample_estimate(m, 7, sampler=sampler)
    e[2].record()
    U, V = sk.waltmin(I, J, val, qh, r, T, init_iters=30, seed=7)
    e[3].record()
    torch.cuda.synchronize()
    wall = time.time() - t0
    # warm re-run of Step 3 alone (the first call also grows the memory pool)
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0.record()
    sk.waltmin(I, J, val, qh, r, T, init_iters=30, seed=7)
    w1.record()
    torch.cuda.synchronize()
    sk.close()
    lela = None
    if run_lela:
        # LELA: two passes over A, same sampler and WAltMin
        le = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        sl = SMPSketch(d, n, n, 1, pi=PI_RADEMACHER, seed=7, a_is_b=True, input=IN_DENSE_F32, device=dev)
        le[0].record()
        sl.norms_block(0, A)
        sl.finalize()
        le[1].record()
        Il, Jl, _, ql = sl.sample_estimate(m, 7)
        le[2].record()
        acc = torch.zeros(Il.numel(), dtype=torch.float64, device=dev)
        sl.exact_entries_block(0, A, None, Il, Jl, acc)
        le[3].record()
        Ul, Vl = sl.waltmin(Il, Jl, acc.float(), ql, r, T, init_iters=30, seed=7)
        le[4].record()
        torch.cuda.synchronize()
        sl.close()
        lela = dict(omega=int(Il.numel()), ms={"pass1_norms": le[0].elapsed_time(le[1]),
                                               "omega": le[1].elapsed_time(le[2]),
                                               "pass2_exact_entries": le[2].elapsed_time(le[3]),
                                               "waltmin": le[3].elapsed_time(le[4])})
    s = top_singular(A, B)
    nrm = float(s[0])
    opt = float(s[r]) / nrm
    err = err_norm(A, B, U, V) / nrm
    if lela is not None:
        lela["error"] = err_norm(A, B, Ul, Vl) / nrm
    out = dict(d=d, n=n, k=k, r=r, T=T, m=m, omega=int(I.numel()), sampler=sampler, pi=pi_name,
               optimal=opt, smp_pca=err, lela=lela,
               paper={"optimal": 0.0271, "lela": 0.0274, "smp_pca": 0.0280},
               ms={"sketch+finalize": e[0].elapsed_time(e[1]), "omega+mtilde": e[1].elapsed_time(e[2]),
                   "waltmin": e[2].elapsed_time(e[3]), "waltmin_warm": w0.elapsed_time(w1)}, wall_s=wall)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
