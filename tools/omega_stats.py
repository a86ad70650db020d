"""Ω row / column sample-count distribution of a config (WAltMin load-balance diagnostic).

    python tools/omega_stats.py [cfg3]
"""
import sys, os, math, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, synth
from paper_1610_06656_b200 import SMPSketch, IN_CSR_F32
cfg = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg3"]; dev = torch.device("cuda", 0)
A, B = bench.make_inputs_csr(cfg, 0, cfg["d"], dev)
sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"], input=IN_CSR_F32, device=dev)
sk.block_csr(0, cfg["d"], *A, *B); sk.finalize()
m = synth.m_of(cfg)
I, J, val, qh = sk.sample_estimate(m, cfg["seed"])
for name, idx, n in (("rows", I, cfg["n1"]), ("cols", J, cfg["n2"])):
    c = torch.bincount(idx.long(), minlength=n).double()
    s, _ = torch.sort(c, descending=True)
    tot = c.sum().item()
    W = 128 * 8
    avg = tot / W
    thr = max(1024, 4 * avg)
    heavy = c[c > thr]
    print(name, "n", n, "tot", tot, "mean", c.mean().item(), "max", s[0].item(), "top10", s[:10].tolist(),
          "heavy>", thr, "count", heavy.numel(), "heavy samples", heavy.sum().item(), "frac", heavy.sum().item() / tot,
          "zero rows", int((c == 0).sum()))
