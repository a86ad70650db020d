"""K1F ablation on one GPU (cfg4, fp32 input): time the fused fp32 sketch kernel
with parts switched off (SMP_K1F_DEBUG bits: 1 = no norms, 4 = no MMA, 32 = no
third-plane MMA, 64 = no conversion).  Diagnostics only (the sketches of modes
!= 0 are wrong by construction).

    python tools/k1f_ablation.py [reps] [modes, e.g. 0,4,64]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1610_06656_b200 import IN_DENSE_F32, SMPSketch  # noqa: E402


def main():
    name = "cfg4"
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   a_is_b=cfg.get("a_is_b", False), input=IN_DENSE_F32, device=dev)
    modes = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1, 32, 4, 64, 68, 69, 0]
    lib = os.path.basename(os.environ.get("SMP_LIB", "libsmp.so"))
    names = ((1, "no-norms"), (4, "no-MMA"), (32, "no-plane2-MMA"), (64, "no-convert"), (128, "no-Pi-TMA"),
             (256, "no-X-TMA"), (512, "TMA-producer-solo"))
    for mode in modes:
        os.environ["SMP_K1F_DEBUG"] = str(mode)
        sk.reset()
        sk.block(0, A, B)
        torch.cuda.synchronize()
        sk.set_timing(True)
        sk.kernel_timing()
        clk = bench.ClockSampler(0)
        clk.start()
        time.sleep(0.3)
        for _ in range(reps):
            sk.reset()
            sk.block(0, A, B)
        ms, n = sk.kernel_timing()
        c = clk.stop()
        sk.set_timing(False)
        parts = [p for b, p in names if mode & b]
        print(f"{lib} {name} mode {mode} ({'+'.join(parts) or 'full'}): {ms / max(n, 1):.4f} ms/launch "
              f"over {n} launches, sm {c and c['sm_mhz']} MHz {c and c['reasons']}", flush=True)
    os.environ.pop("SMP_K1F_DEBUG")
    sk.close()


if __name__ == "__main__":
    main()
