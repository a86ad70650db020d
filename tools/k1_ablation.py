"""K1 ablation on one GPU: time the dense sketch kernel with parts of its work
switched off (SMP_K1_DEBUG bits: 1 = no norms, 2 = constant Π instead of the
Philox generator, 4 = no MMA), each mode run for ~reps launches back to back.
Diagnostics only (the sketches of modes != 0 are wrong by construction).

    python tools/k1_ablation.py [cfg1|cfg2] [reps] [modes, e.g. 0,5,1]

SMP_LIB=paper_1610_06656_b200/libsmp_<variant>.so selects a tuning build.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1610_06656_b200 import IN_DENSE_BF16, SMPSketch  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   input=IN_DENSE_BF16, device=dev)
    modes = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 1, 2, 3, 4, 5, 6, 7, 0]
    lib = os.path.basename(os.environ.get("SMP_LIB", "libsmp.so"))
    for mode in modes:
        os.environ["SMP_K1_DEBUG"] = str(mode)
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
        parts = [p for b, p in ((1, "no-norms"), (2, "const-Pi"), (4, "no-MMA")) if mode & b]
        print(f"{lib} {name} mode {mode} ({'+'.join(parts) or 'full'}): {ms / max(n, 1):.4f} ms/launch "
              f"over {n} launches, sm {c and c['sm_mhz']} MHz {c and c['reasons']}", flush=True)
    os.environ.pop("SMP_K1_DEBUG")
    sk.close()


if __name__ == "__main__":
    main()
