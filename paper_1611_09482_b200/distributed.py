"""Multi-GPU plumbing: shard independent streams over ranks, gather at the end.

The reference runs independent generation sessions in parallel with no
communication (``fast.py:101-102``, ``SPEC.md:307-308``). On a box of B200s
the streams of one generate call are split contiguously over the ranks
(one process per GPU, ``torch.distributed`` over NCCL): rank k owns global
streams [offset_k, offset_k + count_k). Sampling noise is keyed by the global
stream id (``Sampler.stream_offset``), so the generated sequences do not
depend on the number of GPUs. No collective runs per step; the only one is
the final gather of the generated class sequences (uint8/int32 over
NVLink).
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    offset: int  # global id of this rank's first stream
    count: int  # streams on this rank


def shard_streams(total: int, world: int, rank: int) -> Shard:
    """Contiguous split of `total` streams; the first `total % world` ranks get one more."""
    if total < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError("need total >= 1, world >= 1 and 0 <= rank < world")
    base, extra = divmod(total, world)
    count = base + (1 if rank < extra else 0)
    offset = rank * base + min(rank, extra)
    return Shard(rank, world, offset, count)


def gather_sequences(local, shard: Shard, total: int, group=None):
    """Gather each rank's (steps, count) class tensor into (steps, total) on every rank.

    Uses all_gather_into_tensor when every rank holds the same count (NCCL's
    fast path), else a padded all_gather. Works for NCCL (CUDA tensors) and gloo
    (CPU tensors).
    """
    import torch
    import torch.distributed as dist

    if shard.world == 1:
        return local
    steps = local.shape[0]
    counts = [shard_streams(total, shard.world, r).count for r in range(shard.world)]
    cmax = max(counts)
    if all(c == cmax for c in counts) and dist.get_backend(group) == "nccl":
        # rank-major flat buffer: [world][steps][count]
        flat = torch.empty((shard.world, steps, cmax), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(flat, local.contiguous(), group=group)
        parts = list(flat.unbind(0))
    else:
        padded = torch.zeros((steps, cmax), dtype=local.dtype, device=local.device)
        padded[:, : local.shape[1]] = local
        parts = [torch.empty_like(padded) for _ in range(shard.world)]
        dist.all_gather(parts, padded, group=group)
        parts = [p[:, :c] for p, c in zip(parts, counts)]
    return torch.cat(parts, dim=1)
