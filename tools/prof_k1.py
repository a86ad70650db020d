"""Minimal driver for profiling K1 (sketch_tc_kernel) under ncu on one GPU:
runs the one-pass sketch of a dense config a few times (no WAltMin).

    python tools/prof_k1.py [cfg1] [reps]
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
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    inp = IN_DENSE_BF16 if A.dtype == torch.bfloat16 else IN_DENSE_F32
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   a_is_b=cfg.get("a_is_b", False), input=inp, device=dev)
    # warm-up (module load, TMA descriptor path, allocations) outside the timing
    sk.reset()
    sk.block(0, A, B)
    torch.cuda.synchronize()
    sk.set_timing(True)
    for _ in range(reps):
        sk.reset()
        sk.block(0, A, B)
        try:
            sk.finalize()
        except Exception as e:  # debug variants produce invalid sketches
            if not os.environ.get("SMP_K1_DEBUG"):
                raise
            _ = e
    ms, n = sk.kernel_timing()
    print(f"{name}: K1 {ms / max(n, 1):.4f} ms/launch over {n} launches")
    sk.close()


if __name__ == "__main__":
    main()
