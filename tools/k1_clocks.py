"""K1 under sustained load with nvidia-smi clock / power sampling (diagnostic).

    SMP_K1_DEBUG=<mask> python tools/k1_clocks.py [cfg1] [seconds]

Prints K1 ms/launch (CUDA events on the launching stream) and the median SM
clock, power and active throttle reasons seen while it ran.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1610_06656_b200 import IN_DENSE_BF16, IN_DENSE_F32, SMPSketch  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
    secs = float(sys.argv[2]) if len(sys.argv) > 2 else 3.0
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    inp = IN_DENSE_BF16 if A.dtype == torch.bfloat16 else IN_DENSE_F32
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   a_is_b=cfg.get("a_is_b", False), input=inp, device=dev)
    if os.environ.get("CUBLAS"):
        # reference point: cuBLAS bf16 GEMM of the same shape with a stored Π
        P = torch.ones(cfg["k"], cfg["d"], dtype=torch.bfloat16, device=dev)
        for _ in range(3):
            torch.mm(P, A)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clk = bench.ClockSampler(0)
        clk.start()
        e0.record()
        reps = 0
        t0 = time.time()
        while time.time() - t0 < secs:
            for _ in range(20):
                torch.mm(P, A)
                reps += 1
            torch.cuda.synchronize()
        e1.record()
        torch.cuda.synchronize()
        print(f"cuBLAS {cfg['k']}x{cfg['d']} @ {cfg['d']}x{cfg['n1']} bf16: "
              f"{e0.elapsed_time(e1) / reps:.4f} ms; clocks {clk.stop()}")
        return
    sk.reset()
    sk.block(0, A, B)
    torch.cuda.synchronize()
    clk = bench.ClockSampler(0)
    power = []
    clk.start()
    sk.set_timing(True)
    t0 = time.time()
    reps = 0
    while time.time() - t0 < secs:
        for _ in range(20):
            sk.reset()
            sk.block(0, A, B)
            reps += 1
        torch.cuda.synchronize()
    ms, n = sk.kernel_timing()
    c = clk.stop()
    for ln in clk.lines:
        f = [x.strip() for x in ln.split(",")]
        try:
            power.append(float(f[3]))
        except (ValueError, IndexError):
            pass
    power.sort()
    print(f"{name} debug={os.environ.get('SMP_K1_DEBUG', '0')}: K1 {ms / max(n, 1):.4f} ms/launch "
          f"over {n} launches; clocks {c}; power median {power[len(power) // 2] if power else None} W")
    sk.close()


if __name__ == "__main__":
    main()
