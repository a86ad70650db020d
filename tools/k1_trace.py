"""Per-K-block pipeline timeline of one K1 CTA pair (tuning build with
-DSMP_K1_TRACE=<pair index>); SMP_LIB must point at the trace build.

    python -m paper_1610_06656_b200.build -DSMP_K1_TRACE=40 --out=libsmp_k1tr.so --only=sketch_tc.cu
    SMP_LIB=.../libsmp_k1tr.so python tools/k1_trace.py [cfg1|cfg2]

Events (clock64 of the CTA's own SM): 0 TMA issue, 1 relay: X landed, 2 generator
(set of this K-block, quad 0): start, 3 generator: bits built (before the wait
for the TMEM stage), 7 generator: TMEM stage free, 4 relay: Π stage written,
5 leader: both CTAs ready, 6 leader: MMAs + commits issued.
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_1610_06656_b200 import IN_DENSE_BF16, SMPSketch  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
    cfg = synth.CONFIGS[name]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs(name, cfg, 0, cfg["d"], dev)
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   input=IN_DENSE_BF16, device=dev)
    for _ in range(2):
        sk.reset()
        sk.block(0, A, B)
    torch.cuda.synchronize()
    lib = ctypes.CDLL(os.environ["SMP_LIB"])
    buf = np.zeros((2, 8, 512), dtype=np.uint64)
    rc = lib.smp_debug_k1_trace(buf.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0, rc
    t = buf.astype(np.int64)
    names = ["TMA issue", "relay: X landed", "gen: start", "gen: bits built", "relay: Pi written",
             "leader: ready", "leader: issued", "gen: TMEM stage free"]
    order = (0, 1, 2, 3, 7, 4, 5, 6)
    lo, hi = 200, 440
    for rank in (0, 1):
        print(f"== {name} CTA rank {rank}: mean period per K-block (cycles) over it {lo}..{hi}")
        for e in order:
            if t[rank, e, lo] == 0:
                continue
            print(f"  {names[e]:22s} period {(t[rank, e, hi] - t[rank, e, lo]) / (hi - lo):8.1f}")
        base = t[rank, 1]
        print("  mean offsets relative to 'relay: X landed' of the same K-block:")
        for e in order:
            if t[rank, e, lo] == 0:
                continue
            print(f"  {names[e]:22s} {(t[rank, e, lo:hi] - base[lo:hi]).mean():9.1f}")
        print("  rows (it: " + ", ".join(names[e] for e in order) + ") relative to X landed[lo]:")
        for it in range(lo, lo + 12):
            print("   ", it, [int(t[rank, e, it] - base[lo]) if t[rank, e, it] else None for e in order])
    sk.close()


if __name__ == "__main__":
    main()
