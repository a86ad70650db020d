#!/usr/bin/env python
"""Benchmark of the SMP-PCA hot path on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1] [--impl smp|reference]

One STEP = one pass of the whole hot path over the
configuration's synthetic input resident in HBM: the one-pass sketch with
fused norms (K1/K2), the cross-GPU combine (one NCCL all-reduce when N > 1),
finalize (K4), Ω + M̃ (K5/K6) and WAltMin (K7-K9).

  value        = BASELINE metric part 1: bytes of A and B / time of the
                 one-pass sketch+norms stage (first row block -> finalize
                 complete, incl. the all-reduce), GB/s, max over ranks.
  smp_pca_sec  = BASELINE metric part 2: whole Alg. 1 time per step.
  ms_per_step  = whole step (Alg. 1) in ms.
  e2e          = the same GB/s through the C ABI with HOST buffers (pinned),
                 H2D copies inside the timed region, plus the whole e2e step.
  roofline     = the dominant kernel K1 (sketch_tc_kernel), timed with CUDA
                 events on its launching stream (smp_set_timing).

--impl reference runs the CPU oracle (oracle/) as it stands on a bounded
sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "A,B GB/s through one-pass sketch+norms (roofline %); end-to-end SMP-PCA sec"
L2_BYTES = 126 * 2**20


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=float(d["hbm_gbs"]), tc=float(d["bf16_tflops"]),
                    tc_sust=float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), src="measured")
    return dict(hbm=6650.0, tc=1590.0, tc_sust=1400.0, src="fallback")


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx), "samples": len(sm),
                "reasons": sorted(reasons)}


# --------------------------------------------------------------------- data
def shard_rows(d, world, rank, align=synth.GEN_BLOCK):
    """Row shard of rank: equal generator-block-aligned ranges."""
    nblk = (d + align - 1) // align
    b0 = nblk * rank // world
    b1 = nblk * (rank + 1) // world
    return min(d, b0 * align), min(d, b1 * align)


def make_inputs(cfgname, cfg, r0, r1, device):
    n1, n2 = cfg["n1"], cfg["n2"]
    if cfgname == "cfg1":
        VA = synth.lowrank_factors(n1, 20, cfg["seed"], 0, device)
        VB = synth.lowrank_factors(n2, 20, cfg["seed"], 1, device)
        return synth.lowrank_block(r0, r1 - r0, n1, cfg["seed"], VA, VB, device=device)
    if cfgname == "cfg2":
        return synth.cone_block(r0, r1 - r0, n1, cfg["seed"], 30.0, device=device)
    if cfgname == "cfg0":
        A, B = synth.cone_tiny(cfg["d"], n1, seed=cfg["seed"])
        return A[r0:r1].to(device), B[r0:r1].to(device)
    if cfgname == "cfg4":
        W, sig, D = synth.pca_params(n1, cfg["seed"], device=device)
        return synth.pca_block(r0, r1 - r0, n1, cfg["seed"], W, sig, D, device=device), None
    raise ValueError(f"{cfgname}: dense bench configs are cfg0, cfg1, cfg2, cfg4")


def csr_tail_nnz(A, B, n1, n2, rows, density=None):
    """Nonzeros K3d (the SIMT tail) processes: those NOT in a tensor-core head
    column (a column with >= ceil(density·counted rows) nonzeros in the
    library's row sample, with a value of at most 4 significant bits) — the
    library's head rule (K3), recounted here for the K3d roofline."""
    if density is None:
        density = float(os.environ.get("SMP_CSR_HEAD_DENSITY", "0.02"))
    if density <= 0:
        return A[1].numel() + B[1].numel()
    seg, segs = 4096, 64          # the library counts 64 evenly spaced 4096-row segments
    sample = rows > seg * segs
    thr = max(1, math.ceil(density * (seg * segs if sample else rows)))
    tail = 0
    for (rp, col, val), n in ((A, n1), (B, n2)):
        if sample:
            stride = rows // segs
            cs = torch.cat([col[int(rp[s * stride]):int(rp[s * stride + seg])] for s in range(segs)])
        else:
            cs = col
        head_col = torch.bincount(cs.long(), minlength=n) >= thr
        bits = val.view(torch.int32)
        four = ((bits & 0x7F800000) != 0x7F800000) & ((bits & 0x000FFFFF) == 0)
        tail += int((~(head_col[col.long()] & four)).sum())
    return tail


def make_inputs_csr(cfg, r0, r1, device):
    """cfg3 rows [r0, r1) of A and B in CSR (R18); rowptr relative to the block."""
    A = synth.csr_block(r0, r1 - r0, cfg["n1"], cfg["nnz_a"], cfg["seed"], 0, device=device)
    B = synth.csr_block(r0, r1 - r0, cfg["n2"], cfg["nnz_b"], cfg["seed"], 1, device=device)
    return A, B


def csr_bytes(X):
    rp, col, val = X
    return rp.numel() * rp.element_size() + col.numel() * 4 + val.numel() * 4


def dtype_name(cfg):
    return {"bf16": "bf16", "f32": "f32", "csr": "f32"}[cfg["dtype"]]


def pi_code(cfg):
    """Π kind as the C ABI takes it (SMP_PI_*)."""
    return {"rademacher": 0, "gaussian": 1, "srht": 3}[cfg["pi"]]


def oracle_pi(cfg):
    """Π kind code of the oracle (SRHT carries its Hadamard order)."""
    if cfg["pi"] == "srht":
        import oracle
        return oracle.pi_srht(cfg["d"])
    return pi_code(cfg)


# --------------------------------------------------------------------- oracle arms
def oracle_sample_rate(cfgname, cfg, target_s):
    """Time the CPU oracle's one-pass sketch+norms (oracle/, as it stands) on
    the first rows of the workload, CPU-generated block by block with the same
    generators (generation not timed), until about target_s seconds of oracle
    work; returns (GB/s, info)."""
    import oracle
    n1, n2, k, d = cfg["n1"], cfg["n2"], cfg["k"], cfg["d"]
    a_is_b = cfg.get("a_is_b", False)
    csr = cfg["dtype"] == "csr"

    def host(X):
        return synth.bf16_bits(X) if X.dtype == torch.bfloat16 else X.numpy()

    def gen(r0, r1):
        if csr:
            return make_inputs_csr(cfg, r0, r1, "cpu")
        return make_inputs(cfgname, cfg, r0, r1, "cpu")

    def run(A, B, r0):
        t0 = time.perf_counter()
        if csr:
            for X, n in ((A, n1), (B, n2)):
                oracle.sketch_csr(oracle_pi(cfg), cfg["seed"], k, n, X[0].numpy(), X[1].numpy(),
                                  X[2].numpy(), row0=r0)
            nbytes = csr_bytes(A) + csr_bytes(B)
        else:
            oracle.sketch_rows(oracle_pi(cfg), cfg["seed"], k, host(A), row0=r0)
            if not a_is_b:
                oracle.sketch_rows(oracle_pi(cfg), cfg["seed"], k, host(B), row0=r0)
            nbytes = A.numel() * A.element_size() + (0 if a_is_b else B.numel() * B.element_size())
        return time.perf_counter() - t0, nbytes

    probe = 256
    A, B = gen(0, probe)
    t, _ = run(A, B, 0)                       # warm-up + rate probe (not counted)
    rows_target = int(min(d, max(probe, probe * target_s / max(t, 1e-6))))
    step = synth.GEN_BLOCK if not csr else 8192
    secs, nbytes, rows = 0.0, 0, 0
    while rows < rows_target and secs < 2 * target_s:
        r1 = min(rows_target, (rows // step + 1) * step)
        A, B = gen(rows, r1)
        ts, nb = run(A, B, rows)
        secs += ts
        nbytes += nb
        rows = r1
    info = {"rows": rows, "seconds": secs, "bytes": nbytes, "cores": oracle.num_threads(),
            "sample": f"oracle one-pass sketch+norms (fp64, C/OpenMP) of the first {rows} of {d} "
                      f"rows of A{'' if a_is_b else ' and B'} ({n1}{'' if a_is_b else '+' + str(n2)} "
                      f"columns, k={k}{', CSR' if csr else ''}); {secs:.1f} s"}
    return nbytes / secs / 1e9, info


def config_dict(cfgname, cfg, args, world, extra=None):
    """The workload description both arms print (identical keys and values)."""
    d, n1, n2, k = cfg["d"], cfg["n1"], cfg["n2"], cfg["k"]
    a_is_b = cfg.get("a_is_b", False)
    csr = cfg["dtype"] == "csr"
    es = {"bf16": 2, "f32": 4}.get(cfg["dtype"], 0)
    out = {"workload": cfgname, "d": d, "n1": n1, "n2": n2, "k": k, "pi": cfg["pi"], "r": cfg["r"],
           "T": cfg["T"], "m": synth.m_of(cfg), "sampler": args.sampler, "partition": args.partition,
           "init_iters": args.init_iters, "a_is_b": a_is_b,
           "parallelism": f"row-shard x{world} + one NCCL all-reduce" if world > 1 else "1 GPU",
           "l2": ("CSR inputs (11.6 GB)" if csr else "inputs (%.1f GB)" % (d * (n1 + (0 if a_is_b else n2)) * es / 1e9))
           + " larger than the 126 MB L2; no flush",
           "value_scope": "A+B bytes / (sketch_block .. finalize) time; ms_per_step = whole Alg. 1"}
    if csr:
        out["input"] = "CSR int64 rowptr / int32 col / fp32 val"
    if extra:
        out.update(extra)
    return out


def oracle_rest_seconds(fin, cfg, m, args):
    """Time the oracle's steps after the pass (finalize, Ω, M̃, WAltMin) on the
    workload's full n-sized data — the finalized GPU sketch and norms as its
    input data (values are not compared here) — for metric part 2's CPU
    counterpart.  Returns (seconds, |Ω|)."""
    import oracle
    k = cfg["k"]
    t0 = time.perf_counter()
    skA = fin["A_sk"].double().cpu().numpy() * math.sqrt(k)
    skB = fin["B_sk"].double().cpu().numpy() * math.sqrt(k)
    a2 = fin["a_norm2"].cpu().numpy().copy()
    b2 = fin["b_norm2"].cpu().numpy().copy()
    t0 = time.perf_counter()
    As, _, DA = oracle.finalize(k, skA, a2)
    Bs, _, DB = oracle.finalize(k, skB, b2)
    FA, FB = oracle.pairwise_sum(a2), oracle.pairwise_sum(b2)
    al, be = oracle.alpha_beta(a2, b2, FA, FB)
    if args.sampler == "multinomial":
        I, J, q = oracle.sample_multinomial(cfg["seed"], m, al, be)
    else:
        I, J, q = oracle.sample(cfg["seed"], m, al, be)
    Mt = oracle.estimate(k, I, J, As, Bs, DA, DB)
    oracle.waltmin(len(a2), len(b2), cfg["r"], cfg["T"], I, J, Mt, q, np.sqrt(a2), math.sqrt(FA),
                   init_iters=args.init_iters, seed=cfg["seed"],
                   partition=1 if args.partition == "fresh_2t1" else 0)
    return time.perf_counter() - t0, len(I)


def run_reference(args, cfgname, cfg, world, rank):
    if rank != 0:
        return
    per_step = []
    info = None
    # size each step to ~ (3 min) / (K + W) of CPU work
    budget = max(2.0, min(20.0, 150.0 / (args.steps + args.warmup)))
    for s in range(args.warmup + args.steps):
        rate, info = oracle_sample_rate(cfgname, cfg, budget)
        if s >= args.warmup:
            per_step.append(info["seconds"])
    value = info["bytes"] / statistics.mean(per_step) / 1e9
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * statistics.mean(per_step), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(cfgname, cfg, args, world),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": info["cores"], "kind": "oracle",
                         "sample": info["sample"] + f"; {info['rows']} rows per step"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out), flush=True)


# --------------------------------------------------------------------- main arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2",
                    help="workload (default cfg2: the largest single-GPU config of BASELINE.json)")
    ap.add_argument("--impl", default="smp", choices=["smp", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--init-iters", type=int, default=30)
    ap.add_argument("--sampler", default="bernoulli", choices=["bernoulli", "multinomial"],
                    help="Ω sampler: Alg. 1's Bernoulli sweep or the appendix's row-multinomial (NEXT-2)")
    ap.add_argument("--pi", default=None, choices=["rademacher", "gaussian", "srht"],
                    help="override the config's Π (e.g. srht, the paper's Spark sketch; NEXT-1)")
    ap.add_argument("--partition", default="reuse_all", choices=["reuse_all", "fresh_2t1"],
                    help="Alg. 2 line 3 reading (DESIGN.md R11)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfgname = args.config
    cfg = dict(synth.CONFIGS[cfgname])
    if args.pi:
        cfg["pi"] = args.pi

    if args.impl == "reference":
        run_reference(args, cfgname, cfg, world, rank)
        return

    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1610_06656_b200 import SMPSketch, IN_DENSE_BF16, IN_DENSE_F32

    from paper_1610_06656_b200 import IN_CSR_F32

    d, n1, n2, k = cfg["d"], cfg["n1"], cfg["n2"], cfg["k"]
    a_is_b = cfg.get("a_is_b", False)
    csr = cfg["dtype"] == "csr"
    r0, r1 = shard_rows(d, world, rank)
    if csr:
        A, B = make_inputs_csr(cfg, r0, r1, dev)
        inp = IN_CSR_F32
        my_bytes = csr_bytes(A) + csr_bytes(B)
        nnz = A[1].numel() + B[1].numel()
        tail_nnz = csr_tail_nnz(A, B, cfg["n1"], cfg["n2"], r1 - r0)
        t = torch.tensor([float(my_bytes), float(nnz)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t)
        total_bytes, total_nnz = float(t[0]), float(t[1])
    else:
        A, B = make_inputs(cfgname, cfg, r0, r1, dev)
        inp = IN_DENSE_BF16 if A.dtype == torch.bfloat16 else IN_DENSE_F32
        es = A.element_size()
        total_bytes = d * (n1 + (0 if a_is_b else n2)) * es
    m = synth.m_of(cfg)
    r, T = cfg["r"], cfg["T"]
    stream = torch.cuda.current_stream(dev)
    sk = SMPSketch(d, n1, n2, k, pi=pi_code(cfg), seed=cfg["seed"], a_is_b=a_is_b, input=inp,
                   row_begin=r0, row_end=r1, stream=stream, device=dev)

    from paper_1610_06656_b200 import dist as smp_dist

    def combine():
        if world > 1:   # ONE all-reduce of the fp64 exchange buffer
            smp_dist.combine(sk)

    csr_pipe = {}

    def csr_host_blocks(host):
        """e2e CSR path: the pinned host CSR streamed in row chunks (multiples
        of the 2^15-row Π panel), H2D of chunk c+1 on a copy stream overlapped
        with smp_sketch_block_csr of chunk c (double-buffered device chunks)."""
        (arp, acol, aval), (brp, bcol, bval) = host
        rows = r1 - r0
        nch = 8
        ch = -(-rows // nch)
        ch = -(-ch // 32768) * 32768
        bounds = [(c0, min(rows, c0 + ch)) for c0 in range(0, rows, ch)]
        if not csr_pipe:
            csr_pipe["copy"] = torch.cuda.Stream(dev)
            ea = max(int(arp[c1]) - int(arp[c0]) for c0, c1 in bounds)
            eb = max(int(brp[c1]) - int(brp[c0]) for c0, c1 in bounds)
            csr_pipe["buf"] = [[torch.empty(ch + 1, dtype=torch.int64, device=dev),
                                torch.empty(ea, dtype=torch.int32, device=dev),
                                torch.empty(ea, dtype=torch.float32, device=dev),
                                torch.empty(ch + 1, dtype=torch.int64, device=dev),
                                torch.empty(eb, dtype=torch.int32, device=dev),
                                torch.empty(eb, dtype=torch.float32, device=dev)] for _ in range(2)]
        cs, buf = csr_pipe["copy"], csr_pipe["buf"]
        ready = [torch.cuda.Event() for _ in bounds]
        free = [torch.cuda.Event() for _ in bounds]

        def copy(i):
            c0, c1 = bounds[i]
            b = buf[i & 1]
            with torch.cuda.stream(cs):
                if i >= 2:
                    cs.wait_event(free[i - 2])
                out = []
                for (rp, col, val), (drp, dcol, dval) in (((arp, acol, aval), b[0:3]), ((brp, bcol, bval), b[3:6])):
                    e0, e1 = int(rp[c0]), int(rp[c1])
                    drp[:c1 - c0 + 1].copy_(rp[c0:c1 + 1], non_blocking=True)
                    dcol[:e1 - e0].copy_(col[e0:e1], non_blocking=True)
                    dval[:e1 - e0].copy_(val[e0:e1], non_blocking=True)
                    out += [drp[:c1 - c0 + 1], dcol[:e1 - e0], dval[:e1 - e0]]
                ready[i].record(cs)
            return out

        nxt = copy(0)
        for i, (c0, c1) in enumerate(bounds):
            cur = nxt
            if i + 1 < len(bounds):
                nxt = copy(i + 1)
            stream.wait_event(ready[i])
            sk.block_csr(r0 + c0, c1 - c0, *cur)
            free[i].record(stream)

    def step(evs, host=None):
        sk.reset()
        evs[0].record(stream)
        if csr:
            if host is None:
                sk.block_csr(r0, r1 - r0, *A, *B)
            else:  # H2D of the pinned CSR arrays inside the timed region, chunk-pipelined
                csr_host_blocks(host)
        elif host is None:
            sk.block(r0, A, B)
        else:
            sk.block_host(r0, host[0], host[1])
        combine()
        sk.finalize()
        evs[1].record(stream)
        I, J, val, qh = sk.sample_estimate(m, cfg["seed"], sampler=args.sampler)
        if len(evs) > 3:
            evs[3].record(stream)
        U, V = sk.waltmin(I, J, val, qh, r, T, init_iters=args.init_iters, seed=cfg["seed"],
                          partition=args.partition)
        if host is not None:
            Uh, Vh = U.cpu(), V.cpu()  # D2H of the result
        evs[2].record(stream)
        return int(I.numel()), U, V

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize(dev)

    # clock sampler runs over the warm-up and the timed region (nvidia-smi
    # needs ~0.3 s to start; the timed region alone can be shorter)
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.5)
    # warm-up
    for _ in range(args.warmup):
        step([torch.cuda.Event(enable_timing=True) for _ in range(3)])
    # timed region (inputs 4.3+ GB >> 126 MB L2: no flush needed)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    sk.set_timing(True)
    sk.kernel_timing()
    launches0 = sk.kernel_launches
    barrier()
    nomega = 0
    for s in range(args.steps):
        nomega, _, _ = step(evs[s])
    barrier()
    launches = sk.kernel_launches - launches0
    k1_ms, k1_n = sk.kernel_timing()
    sk.set_timing(False)
    clk = clocks.stop()
    t_sketch = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    t_step = sum(e[0].elapsed_time(e[2]) for e in evs) / args.steps
    t_omega = sum(e[1].elapsed_time(e[3]) for e in evs) / args.steps   # Ω draw + M̃ (lines 3-4)
    t_wm = sum(e[3].elapsed_time(e[2]) for e in evs) / args.steps      # WAltMin (line 5)
    if world > 1:
        t = torch.tensor([t_sketch, t_step, k1_ms / max(k1_n, 1)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_sketch, t_step, k1_avg = t.tolist()
    else:
        k1_avg = k1_ms / max(k1_n, 1)

    value = total_bytes / (t_sketch * 1e-3) / 1e9

    pk = peaks()

    def l2_view(tb_s):
        """K3d against the measured L2 -> SM gather rate of its own access
        pattern (tools/l2_probe.py: 1 KB rows at hashed indices of a 32 MB
        L2-resident panel, no arithmetic; profiles/round2/l2_probe.json)."""
        f = os.path.join(ROOT, "profiles", "round2", "l2_probe.json")
        if not os.path.exists(f):
            return None
        peak = json.load(open(f))["best_32mb_tb_s"]
        return {"achieved": tb_s, "peak": peak, "unit": "TB/s", "frac": tb_s / peak,
                "peak_source": "measured L2 gather probe, 32 MB panel (profiles/round2/l2_probe.json)"}

    if csr:
        # the sparse sketch as a whole (K3: tensor-core head through K1 + the
        # SIMT tail K3a-d), timed as the sketch stage: 2k FLOP per nonzero
        # against the SIMT fp32 peak derived from the unit counts (148 SMs x
        # 128 FP32 lanes x 2 FLOP x max SM clock, K3).  The
        # tail kernel K3d alone is reported beside it.
        sm_max = 1965.0 if not clk else clk["sm_max_mhz"]
        alu_peak = 148 * 128 * 2 * sm_max * 1e6 / 1e12
        flops_step = 2.0 * k * nnz * 1.0
        ach_stage = flops_step / (t_sketch * 1e-3) / 1e12
        k3_ms_step = k1_ms / max(args.steps, 1)
        # dominant kernel: K3d (csr_accumulate_kernel), one launch per Π panel,
        # timed with CUDA events on its stream; algorithmic work = 2k FLOP per
        # tail nonzero (FHFMA.BF16 on the SIMT pipe), its π rows (kp bf16 per
        # nonzero) gathered from the L2-resident panel
        k3_launch_ms = k1_ms / max(k1_n, 1)
        launches_per_step = max(k1_n // max(args.steps, 1), 1)
        tail_launch = tail_nnz / launches_per_step
        flops_launch = 2.0 * k * tail_launch
        ach = flops_launch / (k3_launch_ms * 1e-3) / 1e12
        kp_pad = 256 * (1 if k <= 256 else 2 if k <= 512 else 4 if k <= 1024 else 8 if k <= 2048 else 16)
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "k1_traffic.json")
        if os.path.exists(tfile) and world == 1:   # ncu capture of the N=1 launch shape
            traffic = json.load(open(tfile)).get(cfgname)
        roof = {"bound": "alu", "achieved": ach, "peak": alu_peak, "unit": "TFLOP/s",
                "frac": ach / alu_peak, "traffic": traffic,
                "kernel": "csr_accumulate_kernel (K3d, SIMT tail)",
                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x %.0f MHz" % sm_max,
                "k3d_ms_per_launch": k3_launch_ms,
                "k3d_share_of_stage": k3_ms_step / t_sketch,
                "algorithmic_per_launch": {"flops": flops_launch, "tail_nnz": tail_launch,
                                           "l2_pi_gather_bytes": tail_launch * kp_pad * 2},
                "l2_pi_gather_tb_s": tail_launch * kp_pad * 2 / (k3_launch_ms * 1e-3) / 1e12,
                "l2_view": l2_view(tail_launch * kp_pad * 2 / (k3_launch_ms * 1e-3) / 1e12),
                "stage_view": {"achieved": ach_stage, "peak": alu_peak, "frac": ach_stage / alu_peak,
                               "unit": "TFLOP/s", "nnz": nnz, "tail_nnz": tail_nnz,
                               "timed": "sketch stage (CUDA events): head K1 + Π panels + sort + K3d"}}
        roofline_time = max(total_bytes / (pk["hbm"] * 1e9), 2.0 * k * total_nnz / (pk["tc"] * 1e12))
    else:
        # roofline of K1 (per launch = one matrix over this rank's rows),
        # from the ALGORITHMIC work of the method: 2k FLOP and
        # one read of the input element (2 B bf16, 4 B fp32) per element.  The
        # bf16 planes K1F executes for fp32 inputs (R21) are reported beside
        # it as "executed", not counted as useful work.
        rows = r1 - r0
        es_in = A.element_size()
        planes = 3 if inp == IN_DENSE_F32 else (2 if cfg["pi"] == "gaussian" else 1)
        launches_per_step = max(k1_n // max(args.steps, 1), 1)
        ncols_total = (n1 + (0 if a_is_b else n2))
        flops_launch = 2.0 * k * rows * ncols_total / launches_per_step
        bytes_launch = rows * ncols_total * es_in / launches_per_step
        t_hbm = bytes_launch / (pk["hbm"] * 1e9)
        t_tc = flops_launch / (pk["tc"] * 1e12)
        traffic = None
        tfile = os.path.join(ROOT, "profiles", "k1_traffic.json")
        if os.path.exists(tfile) and world == 1:   # ncu capture of the N=1 launch shape
            traffic = json.load(open(tfile)).get(cfgname)
        kname = "sketch_tc_f32_kernel (K1F)" if inp == IN_DENSE_F32 else "sketch_tc_kernel (K1)"
        if t_tc >= t_hbm:
            ach = flops_launch / (k1_avg * 1e-3) / 1e12
            roof = {"bound": "tensor", "achieved": ach, "peak": pk["tc"], "unit": "TFLOP/s",
                    "frac": ach / pk["tc"], "traffic": traffic, "kernel": kname,
                    "peak_source": pk["src"] + " burst bf16 dense (MEASURED_PEAKS.json)"}
            alt_ach = bytes_launch / (k1_avg * 1e-3) / 1e9
            roof["hbm_view"] = {"achieved": alt_ach, "peak": pk["hbm"], "unit": "GB/s",
                                "frac": alt_ach / pk["hbm"]}
        else:
            ach = bytes_launch / (k1_avg * 1e-3) / 1e9
            roof = {"bound": "hbm", "achieved": ach, "peak": pk["hbm"], "unit": "GB/s",
                    "frac": ach / pk["hbm"], "traffic": traffic, "kernel": kname,
                    "peak_source": pk["src"] + " HBM copy bandwidth (MEASURED_PEAKS.json)"}
            alt = flops_launch / (k1_avg * 1e-3) / 1e12
            roof["tensor_view"] = {"achieved": alt, "peak": pk["tc"], "unit": "TFLOP/s",
                                   "frac": alt / pk["tc"]}
        roof["sustained_view"] = {"peak": pk["tc_sust"], "unit": "TFLOP/s",
                                  "frac": flops_launch / (k1_avg * 1e-3) / 1e12 / pk["tc_sust"]}
        if planes > 1:
            exe = flops_launch * planes / (k1_avg * 1e-3) / 1e12
            roof["executed"] = {"planes": planes, "achieved": exe, "unit": "TFLOP/s", "frac": exe / pk["tc"],
                                "note": "bf16 plane-split tensor work actually issued (R21); not useful work"}
        roof["k1_ms_per_launch"] = k1_avg
        roof["algorithmic_per_launch"] = {"flops": flops_launch, "bytes": bytes_launch}
        roofline_time = max(total_bytes / (pk["hbm"] * 1e9),
                            2.0 * k * d * ncols_total / (pk["tc"] * 1e12))

    # e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        def pinned(X):
            h = torch.empty(X.shape, dtype=X.dtype, pin_memory=True)
            h.copy_(X)
            return h
        if csr:
            Ah = [pinned(x) for x in A]
            Bh = [pinned(x) for x in B]
        else:
            Ah = pinned(A)
            Bh = None if B is None else pinned(B)
        step([torch.cuda.Event(enable_timing=True) for _ in range(3)], host=(Ah, Bh))
        ee = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.e2e_steps)]
        barrier()
        for s in range(args.e2e_steps):
            step(ee[s], host=(Ah, Bh))
        barrier()
        te_sk = sum(e[0].elapsed_time(e[1]) for e in ee) / args.e2e_steps
        te_all = sum(e[0].elapsed_time(e[2]) for e in ee) / args.e2e_steps
        if world > 1:
            t = torch.tensor([te_sk, te_all], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te_sk, te_all = t.tolist()
        h2d = (my_bytes if csr else int(A.numel() * es + (0 if B is None else B.numel() * es)))
        e2e = {"value": total_bytes / (te_sk * 1e-3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int((n1 + n2) * r * 4),
               "smp_pca_sec": te_all * 1e-3, "steps": args.e2e_steps,
               "path": ("pinned CSR arrays -> device in 8 row chunks on a copy stream, overlapped with "
                        "smp_sketch_block_csr of the previous chunk" if csr else
                        "smp_sketch_block_host (library-staged pinned H2D, double-buffered)")
                       + " + finalize + sample_estimate + waltmin + D2H(U,V)"}
        del Ah, Bh

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, info = oracle_sample_rate(cfgname, cfg, 20.0)
        cpu = {"value": rate, "unit": "GB/s", "cores": info["cores"], "kind": "oracle",
               "sample": info["sample"]}
        if not csr:
            # metric part 2 on the CPU: the pass extrapolated from the sampled
            # rate, the n-sized steps (finalize, Ω, M̃, WAltMin) run in full
            sk.reset()
            sk.block(r0, A, B)
            fin = sk.finalize()
            rest, nom = oracle_rest_seconds(fin, cfg, m, args)
            cpu["smp_pca_sec"] = total_bytes / (rate * 1e9) + rest
            cpu["smp_pca_sec_parts"] = {"pass_extrapolated_s": total_bytes / (rate * 1e9),
                                        "finalize_omega_mtilde_waltmin_s": rest, "omega": nom}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype_name(cfg), "data": "synthetic",
            "config": config_dict(cfgname, cfg, args, world),
            "omega": nomega,
            **({"nnz": int(total_nnz)} if csr else {}),
            "smp_pca_sec": t_step * 1e-3,
            "sketch_ms": t_sketch,
            "omega_mtilde_ms": t_omega,
            "waltmin_ms": t_wm,
            "roofline_pct_of_stage": 100.0 * roofline_time / (t_sketch * 1e-3),
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(out), flush=True)
    sk.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
