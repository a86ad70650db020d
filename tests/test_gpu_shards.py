"""Row sharding on ONE GPU: G handles, each
restricted to its row range [row_begin, row_end) = shard_rows(d, G, g), sketch
their own rows; their packed partials (smp_sketch_partials) are summed on the
device — what the single NCCL all-reduce computes across GPUs — and one handle
finalizes.  The result must equal the single-handle pass (sketch within 1e-5
per column, norms within 1e-12, Ω bit-exact) and the oracle.  This runs the
library's multi-GPU data path (row-ranged handles, partial buffers, combine,
finalize) without a second GPU; the collective itself is covered by the gloo
test (test_dist_cpu.py)."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_1610_06656_b200.dist import shard_rows
from test_gpu_parity import NORM_RTOL, col_rel_err

pytestmark = pytest.mark.gpu


def _smp():
    import paper_1610_06656_b200 as smp
    return smp


@pytest.mark.parametrize("G,via", [(2, "partials"), (4, "partials"), (8, "partials"), (2, "exchange"),
                                   (8, "exchange")])
def test_row_sharded_handles_sum_to_single_pass(G, via):
    smp = _smp()
    d, n, k = 8 * synth.GEN_BLOCK, 256, 256
    dev = torch.device("cuda", 0)
    VA = synth.lowrank_factors(n, 20, 1, 0, dev)
    VB = synth.lowrank_factors(n, 20, 1, 1, dev)
    A, B = synth.lowrank_block(0, d, n, 1, VA, VB, device=dev)
    # single pass
    one = smp.SMPSketch(d, n, n, k, pi=smp.PI_RADEMACHER, seed=7, device=dev)
    one.block(0, A, B)
    f1 = one.finalize()
    # G row-ranged handles, blocks delivered out of order inside each shard
    hs = []
    for g in range(G):
        r0, r1 = shard_rows(d, G, g)
        h = smp.SMPSketch(d, n, n, k, pi=smp.PI_RADEMACHER, seed=7, row_begin=r0, row_end=r1, device=dev)
        mid = (r0 + r1) // 2
        h.block(mid, A[mid:r1], B[mid:r1])
        h.block(r0, A[r0:mid], B[r0:mid])
        out = r1 if r1 < d else 0                  # a row outside [r0, r1)
        with pytest.raises(smp.SmpError):          # rows outside the handle's range are rejected
            h.block(out, A[out:out + 64], B[out:out + 64])
        hs.append(h)
    if via == "partials":
        sk0, nr0 = hs[0].partials()
        for h in hs[1:]:
            sk, nr = h.partials()
            sk0 += sk
            nr0 += nr
    else:
        # the single fp64 exchange buffer that dist.combine all-reduces
        bufs = [h.pack_partials() for h in hs]
        torch.cuda.synchronize()
        acc = bufs[0]
        for b in bufs[1:]:
            acc += b
        hs[0].unpack_partials()
    fG = hs[0].finalize()
    e = col_rel_err(fG["A_sk"], f1["A_sk"].cpu().double().numpy())
    assert e.max() <= 1e-5, e.max()
    e = col_rel_err(fG["B_sk"], f1["B_sk"].cpu().double().numpy())
    assert e.max() <= 1e-5, e.max()
    np.testing.assert_allclose(fG["a_norm2"].cpu().numpy(), f1["a_norm2"].cpu().numpy(), rtol=1e-12)
    np.testing.assert_allclose(fG["b_norm2"].cpu().numpy(), f1["b_norm2"].cpu().numpy(), rtol=1e-12)
    # oracle on a few columns over all d rows
    cols = np.array([0, 17, 100, 255])
    sub = A[:, torch.as_tensor(cols, device=dev)].contiguous()
    skc, n2c = oracle.sketch_rows(0, 7, k, synth.bf16_bits(sub))
    S, _, _ = oracle.finalize(k, skc, n2c)
    assert col_rel_err(fG["A_sk"][torch.as_tensor(cols, device=dev)], S).max() <= 1e-5
    np.testing.assert_allclose(fG["a_norm2"].cpu().numpy()[cols], n2c, rtol=NORM_RTOL)
    # Ω from the combined handle == Ω from the single pass (bit-exact)
    m = 4 * n * 5 * math.log(n)
    I1, J1, v1, q1 = one.sample_estimate(m, 3)
    IG, JG, vG, qG = hs[0].sample_estimate(m, 3)
    assert torch.equal(I1, IG) and torch.equal(J1, JG)
    scale = torch.sqrt(f1["a_norm2"][I1.long()] * f1["b_norm2"][J1.long()])
    assert float(((v1.double() - vG.double()).abs() / scale).max()) <= 1e-4
    for h in hs:
        h.close()
    one.close()


def _nccl_combine_worker(port, out):
    import os
    import torch.distributed as dist
    from paper_1610_06656_b200 import dist as smp_dist
    smp = _smp()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    d, n, k = 2 * synth.GEN_BLOCK, 300, 256
    A = synth.gaussian_small(d, n, seed=21, scale_cols=True).to(torch.bfloat16).to(dev)
    B = synth.gaussian_small(d, n, seed=22).to(torch.bfloat16).to(dev)
    res = []
    for comb in (False, True):
        h = smp.SMPSketch(d, n, n, k, pi=smp.PI_RADEMACHER, seed=5, device=dev)
        h.block(0, A, B)
        if comb:
            # the N > 1 bench's combine on a 1-rank NCCL group: pack -> all-reduce -> unpack
            orig = dist.get_world_size
            dist.get_world_size = lambda group=None: 2   # take the collective branch
            try:
                smp_dist.combine(h)
            finally:
                dist.get_world_size = orig
        f = h.finalize()
        res.append([f[x].cpu() for x in ("A_sk", "B_sk", "a_norm2", "b_norm2")])
        h.close()
    out.put(all(torch.equal(x, y) for x, y in zip(*res)))
    dist.destroy_process_group()


def test_nccl_single_allreduce_combine_is_exact():
    """dist.combine = smp_sketch_pack_partials -> ONE NCCL all-reduce of the
    fp64 exchange buffer -> smp_sketch_unpack_partials, run on a 1-rank NCCL
    group: the round trip (fp32 widened to fp64, summed over one rank,
    rounded back) must leave the finalized sketch and norms bit-identical."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_combine_worker, args=(port, q))
    p.start()
    ok = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert ok


def _nccl_worker(port, out):
    import os
    import torch.distributed as dist
    from paper_1610_06656_b200.dist import _coalesced_allreduce
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    a = torch.arange(10, dtype=torch.float32, device="cuda")
    b = torch.arange(4, dtype=torch.float64, device="cuda") * 0.5
    _coalesced_allreduce([a, b])           # the calls bench.py's combine makes
    c = torch.ones(3, dtype=torch.float32, device="cuda")
    _coalesced_allreduce([a, c, b])        # two fp32 buffers: the coalesced NCCL group
    torch.cuda.synchronize()
    out.put((a.cpu().numpy().tolist(), b.cpu().numpy().tolist()))
    dist.destroy_process_group()


def test_nccl_coalesced_allreduce_runs():
    """The NCCL branch of the combine (one all-reduce per dtype; same-dtype
    buffers in one coalesced group) on a 1-rank NCCL group: the API path the
    N > 1 bench takes executes on this GPU and leaves the buffers intact (sum
    over 1 rank).  Round 2 found here that NCCL's coalescing manager rejects
    an fp32 + fp64 group."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(port, q))
    p.start()
    a, b = q.get(timeout=120)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert a == list(range(10)) and b == [0.0, 0.5, 1.0, 1.5]
