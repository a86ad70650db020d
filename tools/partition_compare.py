"""Alg. 2 line 3 readings side by side (R11): REUSE_ALL (all of Ω
in every phase, the deployed ALS) vs FRESH_2T1 (2T+1 disjoint random
subsets), and the Bernoulli vs row-multinomial Ω (R27), on a bench
workload through the C ABI.  Reports ||AᵀB − ÛV̂ᵀ||_2 / ||AᵀB||_2 and the
optimal rank-r error σ_{r+1}/σ_1 (AᵀB formed in fp32 on the GPU; n ≤ 4096).

    python tools/partition_compare.py [cfg1|cfg2] [m_coef ...]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1610_06656_b200 import IN_DENSE_BF16, SMPSketch  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    coefs = [float(x) for x in sys.argv[2:]] or [4.0, 12.0]
    cfg = dict(synth.CONFIGS[name])
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    M = torch.zeros(cfg["n1"], cfg["n2"], dtype=torch.float32, device=dev)
    for r0 in range(0, cfg["d"], 1 << 18):
        M += A[r0:r0 + (1 << 18)].float().T @ B[r0:r0 + (1 << 18)].float()
    s = torch.linalg.svdvals(M.double())
    r, T = cfg["r"], cfg["T"]
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   input=IN_DENSE_BF16, device=dev)
    sk.block(0, A, B)
    sk.finalize()
    out = {"workload": name, "r": r, "T": T, "optimal": float(s[r] / s[0]), "runs": []}
    n = max(cfg["n1"], cfg["n2"])
    for c in coefs:
        m = c * n * r * math.log(n)
        for sampler in ("bernoulli", "multinomial"):
            I, J, val, qh = sk.sample_estimate(m, cfg["seed"], sampler=sampler)
            for part in ("reuse_all", "fresh_2t1"):
                U, V = sk.waltmin(I, J, val, qh, r, T, init_iters=30, seed=cfg["seed"], partition=part)
                err = float(torch.linalg.matrix_norm((U.double() @ V.double().T) - M.double(), 2) / s[0])
                out["runs"].append({"m_coef": c, "m": m, "omega": int(I.numel()), "sampler": sampler,
                                    "partition": part, "error": err})
                print(json.dumps(out["runs"][-1]), flush=True)
    print(json.dumps(out), flush=True)
    sk.close()


if __name__ == "__main__":
    main()
