"""Per-K-block pipeline timeline of one K1F CTA pair (tuning build with
-DSMP_F32_TRACE=<pair index>): prints the clock64 deltas between the pipeline
events of the steady state.  SMP_LIB must point at the trace build.

    python -m paper_1610_06656_b200.build -DSMP_F32_TRACE=100 --out=libsmp_ftr.so --only=sketch_tc_f32.cu
    SMP_LIB=.../libsmp_ftr.so python tools/k1f_trace.py
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
from paper_1610_06656_b200 import IN_DENSE_F32, SMPSketch  # noqa: E402


def main():
    cfg = synth.CONFIGS["cfg4"]
    dev = torch.device("cuda", 0)
    A, B = bench.make_inputs("cfg4", cfg, 0, cfg["d"], dev)
    sk = SMPSketch(cfg["d"], cfg["n1"], cfg["n2"], cfg["k"], pi=bench.pi_code(cfg), seed=cfg["seed"],
                   a_is_b=cfg.get("a_is_b", False), input=IN_DENSE_F32, device=dev)
    for _ in range(2):
        sk.reset()
        sk.block(0, A, B)
    torch.cuda.synchronize()
    lib = ctypes.CDLL(os.environ["SMP_LIB"])
    buf = np.zeros((2, 8, 512), dtype=np.uint64)
    rc = lib.smp_debug_k1f_trace(buf.ctypes.data_as(ctypes.c_void_p))
    assert rc == 0, rc
    t = buf.astype(np.int64)
    names = ["TMA issue", "conv: xfull seen", "conv: pempty seen", "conv w8 done", "relay: pfull seen",
             "leader: ready seen", "leader: commits issued", "conv w23 done"]
    lo, hi = 100, 200
    for rank in (0, 1):
        print(f"== CTA rank {rank}: mean period per K-block (cycles) over it {lo}..{hi}")
        for e in range(8):
            if t[rank, e, lo] == 0:
                continue
            per = (t[rank, e, hi] - t[rank, e, lo]) / (hi - lo)
            print(f"  {names[e]:26s} period {per:8.1f}")
        base = t[rank, 1]
        print("  mean offsets relative to 'conv: xfull seen' of the same K-block:")
        for e in range(8):
            if t[rank, e, lo] == 0:
                continue
            off = (t[rank, e, lo:hi] - base[lo:hi]).mean()
            print(f"  {names[e]:26s} {off:9.1f}")
        # lookahead: TMA issue of it+NSTG relative to xfull seen of it
        print("  sample rows (it: TMA issue, xfull, pempty, conv done, relay, ready, commit) relative to xfull[lo]:")
        for it in range(lo, lo + 8):
            print("   ", it, [int(t[rank, e, it] - base[lo]) if t[rank, e, it] else None for e in (0, 1, 2, 3, 7, 4, 5, 6)])
    sk.close()


if __name__ == "__main__":
    main()
