"""SMP-PCA vs SVD(ÃᵀB̃) on the paper's cone family (Figs.
2b/4b), everything on the GPU through the C ABI.

    python tools/cone_sweep.py [d] [n] [k] [r]

For each cone angle θ: A, B = shared-axis cones (synth.cone_shared_axis),
SMP-PCA's rank-r factors and the rank-r SVD of the sketch product ÃᵀB̃ (same
sketch), and their spectral errors relative to ||AᵀB||₂.  The paper's claim:
SMP-PCA is more accurate, increasingly so as θ → 0.
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1610_06656_b200 import IN_DENSE_F32, PI_GAUSSIAN, SMPSketch  # noqa: E402


def run(d=20000, n=200, k=256, r=5, thetas=(0.1, 0.3, 0.6, 1.0, 1.5), seed=3):
    dev = torch.device("cuda", 0)
    rows = []
    for th in thetas:
        A64, B64 = synth.cone_shared_axis(d, n, th, seed=seed)
        M = (A64.T @ B64).to(dev)
        nrm = torch.linalg.matrix_norm(M, 2)
        A, B = A64.float().to(dev), B64.float().to(dev)
        sk = SMPSketch(d, n, n, k, pi=PI_GAUSSIAN, seed=seed, input=IN_DENSE_F32, device=dev)
        sk.block(0, A, B)
        sk.finalize()
        m = 6 * n * r * math.log(n)
        I, J, val, qh = sk.sample_estimate(m, seed)
        U, V = sk.waltmin(I, J, val, qh, r, 10, init_iters=30, seed=seed)
        Us, Vs = sk.svd_of_sketch(r, seed=seed)
        sk.close()
        err = float(torch.linalg.matrix_norm(U.double() @ V.double().T - M, 2) / nrm)
        err_svd = float(torch.linalg.matrix_norm(Us.double() @ Vs.double().T - M, 2) / nrm)
        s = torch.linalg.svdvals(M)
        opt = float(s[r] / nrm)
        rows.append(dict(theta=th, smp_pca=err, svd_sketch=err_svd, ratio=err_svd / max(err, 1e-300),
                         optimal=opt, omega=int(I.numel())))
        print(json.dumps(rows[-1]), flush=True)
    return rows


if __name__ == "__main__":
    args = [int(a) for a in sys.argv[1:]]
    run(*args)
