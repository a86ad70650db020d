"""Time Ω + M̃ (smp_sample_estimate_ex) for both samplers on a dense config.

    python tools/prof_omega.py [cfg1] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1610_06656_b200 import IN_DENSE_BF16, IN_DENSE_F32, SMPSketch  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    inp = IN_DENSE_BF16 if A.dtype == torch.bfloat16 else IN_DENSE_F32
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   a_is_b=cfg.get("a_is_b", False), input=inp, device=dev)
    sk.block(0, A, B)
    sk.finalize()
    m = synth.m_of(cfg)
    for sampler in ("bernoulli", "multinomial"):
        I, *_ = sk.sample_estimate(m, cfg["seed"], sampler=sampler)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            I, *_ = sk.sample_estimate(m, cfg["seed"], sampler=sampler, cap=I.numel() + 1024)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} n1={cfg['n1']} n2={cfg['n2']} m={m:.0f} {sampler}: |Omega|={I.numel()} "
              f"{e0.elapsed_time(e1) / reps:.3f} ms (incl. M~ and host syncs)")
    sk.close()


if __name__ == "__main__":
    main()
