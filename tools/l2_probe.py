"""Measure the L2 -> SM gather throughput that bounds K3d (DESIGN.md §7 K3):
whole 1 KB rows at hashed indices of an L2-resident panel, the best over grid
sizes and loads in flight.  Writes one JSON line (also to
profiles/round2/l2_probe.json when --save).

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC tools/l2_probe.cu -o tools/libl2probe.so
    python tools/l2_probe.py [--save]
"""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "libl2probe.so")


def main():
    if not os.path.exists(SO):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", os.path.join(HERE, "l2_probe.cu"), "-o", SO])
    lib = ctypes.CDLL(SO)
    lib.l2_probe_run.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_uint32, ctypes.c_void_p, ctypes.c_void_p]
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    out = torch.zeros(4, dtype=torch.int32, device=dev)
    res = []
    for mb in (8, 32, 64):
        nrows = mb * 1024
        panel = torch.randint(0, 2**31 - 1, (nrows * 256,), dtype=torch.int32, device=dev)
        for bps in (3, 4, 8):
            for u in (2, 4, 8):
                blocks = 148 * bps
                rpw = 2048
                args = (panel.data_ptr(), nrows, blocks, rpw, u, 0, out.data_ptr(), st.cuda_stream)
                for _ in range(3):
                    lib.l2_probe_run(*args)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                reps = 10
                torch.cuda.synchronize()
                e0.record(st)
                for r in range(reps):
                    lib.l2_probe_run(panel.data_ptr(), nrows, blocks, rpw, u, r + 1, out.data_ptr(), st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
                nbytes = blocks * 8 * rpw * 1024
                res.append({"panel_mb": mb, "blocks": blocks, "u": u, "ms": ms, "tb_s": nbytes / ms / 1e9})
                print(json.dumps(res[-1]), flush=True)
    best = max(res, key=lambda r: r["tb_s"])
    line = {"what": "L2->SM gather of 1 KB rows at hashed indices (K3d's pattern, no arithmetic)",
            "best_tb_s": best["tb_s"], "best": best,
            "best_32mb_tb_s": max(r["tb_s"] for r in res if r["panel_mb"] == 32),
            "gpu": torch.cuda.get_device_name(0)}
    print(json.dumps(line))
    if "--save" in sys.argv:
        os.makedirs(os.path.join(os.path.dirname(HERE), "gpurun_out"), exist_ok=True)
        with open(os.path.join(os.path.dirname(HERE), "gpurun_out", "l2_probe.json"), "w") as f:
            f.write(json.dumps({"runs": res, **line}, indent=1))


if __name__ == "__main__":
    main()
