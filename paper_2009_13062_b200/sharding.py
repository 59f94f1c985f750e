"""Instance sharding across GPUs.

Merged instances are independent (slice m depends only on
x_m and W_m), so N instances split into contiguous per-rank shards, each rank
merges and runs its own shard, and nothing crosses GPUs on the hot path.
Outputs are gathered once, after the timed region, with one collective.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(num_instances: int, world: int, rank: int) -> range:
    """Contiguous, balanced instance ids of ``rank`` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    base, extra = divmod(num_instances, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def gather_instance_outputs(per_instance: list[torch.Tensor], num_instances: int,
                            group=None) -> list[torch.Tensor] | None:
    """Gather every rank's per-instance outputs (same shape per instance) to
    rank 0 in global instance order; other ranks get None. One
    all_gather over padded flat buffers (NCCL on GPU, gloo on CPU)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = shard_range(num_instances, world, rank)
    if len(per_instance) != len(mine):
        raise ValueError(f"rank {rank} holds {len(per_instance)} outputs, shard is {len(mine)}")
    ref = per_instance[0]
    width = max(len(shard_range(num_instances, world, r)) for r in range(world))
    flat = torch.zeros((width,) + tuple(ref.shape), dtype=ref.dtype, device=ref.device)
    for i, t in enumerate(per_instance):
        flat[i].copy_(t)
    bufs = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(bufs, flat, group=group)
    if rank != 0:
        return None
    out = []
    for r in range(world):
        out.extend(bufs[r][i] for i in range(len(shard_range(num_instances, world, r))))
    return out
