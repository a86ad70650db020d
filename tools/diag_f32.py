"""Diagnostic: fp32-input sketch error vs the oracle for cfg4-like data at
reduced d (chunk boundaries of the 3-plane split), Gaussian vs Rademacher."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import synth, oracle
from paper_1610_06656_b200 import SMPSketch, IN_DENSE_F32
from test_gpu_parity import col_rel_err

cfg = synth.CONFIGS["cfg4"]
n = cfg["n1"]
W, sig, D = synth.pca_params(n, cfg["seed"], device="cuda")
for d in [43690, 131072, 262144]:
    A = synth.pca_block(0, d, n, cfg["seed"], W, sig, D, device="cuda")
    for pi in (0, 1):
        for k in (256, 512):
            sk = SMPSketch(d, n, n, k, pi=pi, seed=4, a_is_b=True, input=IN_DENSE_F32)
            sk.block(0, A)
            fin = sk.finalize()
            cols = np.array([0, 7, 100, 2047])
            sub = A[:, torch.as_tensor(cols, device="cuda")].contiguous().cpu().numpy()
            s, n2 = oracle.sketch_rows(pi, 4, k, sub)
            S, _, _ = oracle.finalize(k, s, n2)
            e = col_rel_err(fin["A_sk"][torch.as_tensor(cols, device="cuda")], S)
            print(f"d={d} pi={pi} k={k}: col rel err {e}", flush=True)
            sk.close()
