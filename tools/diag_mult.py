"""Diagnostic: WAltMin on the same multinomial Ω (oracle-generated) on the GPU
and in the oracle, Table-1-like data (A = B = G D), n = d given."""
import math, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import oracle
from paper_1610_06656_b200 import IN_DENSE_F32, PI_GAUSSIAN, SMPSketch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
k, r = 300, 5
rng = np.random.default_rng(1)
A = rng.standard_normal((n, n)) * (1 / np.arange(1, n + 1))
M = A.T @ A
s = np.linalg.svd(M, compute_uv=False)
m = 4 * n * r * math.log(n)
sk, a2 = oracle.sketch_rows(oracle.PI_GAUSSIAN, 3, k, A)
As, _, DA = oracle.finalize(k, sk, a2)
FA = oracle.pairwise_sum(a2)
al, be = oracle.alpha_beta(a2, a2, FA, FA)
dev = torch.device("cuda")
g = SMPSketch(n, n, n, k, pi=PI_GAUSSIAN, seed=3, a_is_b=True, input=IN_DENSE_F32, device=dev)
g.block(0, torch.tensor(A, dtype=torch.float32, device=dev))
g.finalize()
for name, (I, J, q) in (("bern", oracle.sample(3, m, al, be)), ("mult", oracle.sample_multinomial(3, m, al, be))):
    Mt = oracle.estimate(k, I, J, As, As, DA, DA)
    t = time.time()
    Uo, Vo = oracle.waltmin(n, n, r, 10, I, J, Mt, q, np.sqrt(a2), math.sqrt(FA), init_iters=30, seed=3)
    to = time.time() - t
    Ug, Vg = g.waltmin(torch.tensor(I, device=dev), torch.tensor(J, device=dev),
                       torch.tensor(Mt.astype(np.float32), device=dev), torch.tensor(q, device=dev), r, 10,
                       init_iters=30, seed=3)
    Pg = Ug.cpu().double().numpy() @ Vg.cpu().double().numpy().T
    Po = Uo @ Vo.T
    print(name, len(I), "oracle err %.4f" % (np.linalg.norm(Po - M, 2) / s[0]),
          "gpu err %.4f" % (np.linalg.norm(Pg - M, 2) / s[0]),
          "gpu-vs-oracle %.2e" % (np.linalg.norm(Pg - Po, 2) / s[0]), "opt %.4f" % (s[r] / s[0]),
          "oracle %.0fs" % to, flush=True)
