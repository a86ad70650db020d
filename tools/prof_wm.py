"""Time smp_waltmin alone (CUDA events) on a dense config's Ω / M̃, for a few
(init_iters, T) settings; diagnostic for the persistent WAltMin kernel.

    python tools/prof_wm.py [cfg1] [reps]
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
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    settings = [(1, 1), (30, 1), (1, 10), (30, 10)]
    if len(sys.argv) > 3:
        settings = [tuple(int(x) for x in sys.argv[3].split(","))]
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    inp = IN_DENSE_BF16 if A.dtype == torch.bfloat16 else IN_DENSE_F32
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   a_is_b=cfg.get("a_is_b", False), input=inp, device=dev)
    sk.reset()
    sk.block(0, A, B)
    sk.finalize()
    I, J, val, qh = sk.sample_estimate(synth.m_of(cfg), cfg["seed"])
    del A, B
    for key, X, n in (("rows", I, cfg["n1"]), ("cols", J, cfg["n2"])):
        c = torch.bincount(X.long(), minlength=n)
        print(f"{name} {key}: n={n} max={int(c.max())} mean={float(c.float().mean()):.1f} "
              + " ".join(f">{t}:{int((c > t).sum())}" for t in (128, 256, 512, 1024)))
    for iters, T in settings:
        sk.waltmin(I, J, val, qh, cfg["r"], T, init_iters=iters, seed=cfg["seed"])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            sk.waltmin(I, J, val, qh, cfg["r"], T, init_iters=iters, seed=cfg["seed"])
        e1.record()
        torch.cuda.synchronize()
        print(f"{name} |Omega|={I.numel()} r={cfg['r']} init_iters={iters} T={T}: "
              f"{e0.elapsed_time(e1) / reps:.3f} ms")
    sk.close()


if __name__ == "__main__":
    main()
