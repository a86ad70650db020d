"""Multi-rank host logic on CPU (gloo, world size 2): row shards cover the
rows exactly once, and one all-reduce of per-shard partial sketches and norms
equals the single-process pass (S:146 merge contract)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1610_06656_b200.dist import allreduce_partials, shard_rows


def test_shard_rows_partition():
    for d in [1, 1000, 65536, 65537, 1 << 20, 4_194_304, 2_000_000]:
        for world in [1, 2, 3, 4, 8]:
            rs = [shard_rows(d, world, r, align=65536) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == d
            for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
                assert a1 == b0
            assert all(r0 % 65536 == 0 for r0, _ in rs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, k, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = shard_rows(X.shape[0], world, rank, align=64)
    sk, n2 = oracle.sketch_rows(0, 3, k, X[r0:r1], row0=r0)
    t_sk = torch.from_numpy(sk.astype(np.float32).ravel().copy())
    t_n2 = torch.from_numpy(n2.copy())
    allreduce_partials([t_sk, t_n2])
    if rank == 0:
        out.put((t_sk.numpy().copy(), t_n2.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_two_rank_combine_equals_whole():
    rng = np.random.default_rng(0)
    d, n, k = 640, 24, 32
    X = rng.standard_normal((d, n))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    sk, n2 = q.get(timeout=100)
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    whole, wn = oracle.sketch_rows(0, 3, k, X)
    np.testing.assert_allclose(sk.reshape(n, k), whole, rtol=1e-5, atol=1e-4)
    np.testing.assert_allclose(n2, wn, rtol=1e-12)


class _StubSketch:
    """Stands in for SMPSketch on CPU: exposes packed partials like
    smp_sketch_partials (fp32 sketch sums, fp64 norms²)."""

    def __init__(self, sk, nrm):
        self.sk, self.nrm = sk, nrm

    def partials(self):
        return self.sk, self.nrm

    def pack_partials(self):            # smp_sketch_pack_partials: [sk widened | nrm] in fp64
        self.buf = torch.cat([self.sk.double(), self.nrm])
        return self.buf

    def unpack_partials(self):          # smp_sketch_unpack_partials: sk rounded to fp32 once
        n = self.sk.numel()
        self.sk.copy_(self.buf[:n].float())
        self.nrm.copy_(self.buf[n:])


def _combine_worker(rank, world, port, X, k, out):
    from paper_1610_06656_b200.dist import combine
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r0, r1 = shard_rows(X.shape[0], world, rank, align=64)
    sk, n2 = oracle.sketch_rows(0, 3, k, X[r0:r1], row0=r0)
    stub = _StubSketch(torch.from_numpy(sk.astype(np.float32).ravel().copy()), torch.from_numpy(n2.copy()))
    combine(stub)                       # the call bench.py makes between the pass and finalize
    out.put((rank, stub.sk.numpy().copy(), stub.nrm.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_gloo_combine_api_all_ranks_equal_whole():
    """dist.combine (bench's combine step) leaves the full sums on EVERY rank
    (replicated finalize / Ω / WAltMin need them everywhere)."""
    rng = np.random.default_rng(1)
    d, n, k = 704, 20, 16
    X = rng.standard_normal((d, n))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_combine_worker, args=(r, 2, port, X, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=100) for _ in range(2)]
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    whole, wn = oracle.sketch_rows(0, 3, k, X)
    for _, sk, n2 in res:
        np.testing.assert_allclose(sk.reshape(n, k), whole, rtol=1e-5, atol=1e-4)
        np.testing.assert_allclose(n2, wn, rtol=1e-12)
