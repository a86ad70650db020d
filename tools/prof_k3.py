"""Minimal driver for profiling the CSR sketch (K3 head + tail) on cfg3 under
ncu on one GPU: one smp_sketch_block_csr over all rows, twice.

    python tools/prof_k3.py [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1610_06656_b200 import IN_CSR_F32, SMPSketch  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    cfg = synth.CONFIGS["cfg3"]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs_csr(cfg, 0, cfg["d"], dev)
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   input=IN_CSR_F32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(reps):
        sk.reset()
        e0.record()
        sk.block_csr(0, cfg["d"], *A, *B)
        e1.record()
        torch.cuda.synchronize()
        print(f"cfg3 CSR sketch pass {i}: {e0.elapsed_time(e1):.2f} ms")
    sk.close()


if __name__ == "__main__":
    main()
