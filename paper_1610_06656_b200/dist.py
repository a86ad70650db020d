"""Row sharding across GPUs and the single combine step.

ΠA = Σ_g Π[:, rows_g] A[rows_g, :] and ||A_i||² = Σ_g ||A_i^(g)||² are sums
over row blocks (the Spark treeAggregate of P:145), so each rank sketches its
own rows and the packed partials are combined by ONE all-reduce (NCCL over
NVLink on B200; gloo works for the CPU tests).  Everything after the combine
(finalize, Ω, M̃, WAltMin) is replicated: the hashes make Ω identical on every
rank without further communication.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

GEN_BLOCK = 65536


def shard_rows(d: int, world: int, rank: int, align: int = GEN_BLOCK):
    """[r0, r1) of rank: equal, `align`-aligned row ranges (the input
    generators are keyed by 65,536-row blocks, so shards see identical data)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    nblk = (d + align - 1) // align
    b0 = nblk * rank // world
    b1 = nblk * (rank + 1) // world
    return min(d, b0 * align), min(d, b1 * align)


def _coalesced_allreduce(tensors, group=None):
    """The collective itself.  Buffers of one dtype are coalesced into one
    NCCL group call; the fp32 sketch and the fp64 norms differ in dtype (which
    NCCL's coalescing rejects), so one all-reduce per dtype is issued
    asynchronously back to back and waited on together."""
    by_dtype = {}
    for t in tensors:
        by_dtype.setdefault(t.dtype, []).append(t)
    works = []
    for group_tensors in by_dtype.values():
        if len(group_tensors) > 1 and dist.get_backend(group) == "nccl":
            with dist._coalescing_manager(group=group, async_ops=False):
                for t in group_tensors:
                    dist.all_reduce(t, group=group)
        else:
            for t in group_tensors:
                works.append(dist.all_reduce(t, group=group, async_op=True))
    for w in works:
        w.wait()
    return tensors


def allreduce_partials(tensors, group=None):
    """Sum the partial sketch (fp32) and norm (fp64) buffers across ranks in
    place (one collective per dtype, see _coalesced_allreduce)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return tensors
    return _coalesced_allreduce(tensors, group)


def combine(sketch, group=None):
    """Combine an SMPSketch's row-shard partials with ONE all-reduce (before
    finalize): the library packs [fp32 sketch sums widened to fp64 | fp64
    norms²] into one exchange buffer on its stream (smp_sketch_pack_partials),
    NCCL sums it in place, and the library writes it back
    (smp_sketch_unpack_partials; the sketch rounded to fp32 once).  The fp64
    sum of <= 8 widened fp32 partials is exact in practice, so the result does
    not depend on NCCL's reduction order."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return sketch.partials()
    buf = sketch.pack_partials()
    if buf.is_cuda:
        # the collective on the handle's stream: after the pack, before the unpack
        with torch.cuda.stream(sketch.stream):
            dist.all_reduce(buf, group=group)
    else:
        dist.all_reduce(buf, group=group)
    sketch.unpack_partials()
    return sketch.partials()
