"""Diagnostic: one small Gaussian bf16 sketch through K1's PANEL path."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import synth, oracle
from paper_1610_06656_b200 import SMPSketch, IN_DENSE_BF16
d, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
A = synth.gaussian_small(d, n, seed=1).to(torch.bfloat16)
sk = SMPSketch(d, n, n, k, pi=1, seed=3, a_is_b=True, input=IN_DENSE_BF16)
sk.block(0, A.cuda())
torch.cuda.synchronize()
print("K1 done", flush=True)
fin = sk.finalize()
s, n2 = oracle.sketch_rows(1, 3, k, synth.bf16_bits(A))
S, _, _ = oracle.finalize(k, s, n2)
g = fin["A_sk"].cpu().double().numpy()
print("max col rel err", (np.linalg.norm(g - S, axis=1) / np.linalg.norm(S, axis=1)).max())
