"""View sharding across GPUs (one process per GPU, torch.distributed for plumbing).

The reference has no multi-device code; views of a scene are
independent, so a batch of cameras is split into contiguous shards, one per
rank, with the scene replicated on every GPU. There is no data-path collective:
the only communication is the barrier / max-over-ranks timing and an optional
final gather of the rendered images to rank 0 (NCCL over NVLink on the GPU box,
gloo in the CPU tests).
"""
from __future__ import annotations


def shard_views(n_views: int, world: int, rank: int) -> range:
    """Contiguous, balanced shard of view indices for `rank` (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(n_views, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over all ranks."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_images(images, n_views: int, dist=None):
    """Collects every rank's rendered views ([k, H, W, C] tensor, in shard order)
    on rank 0 as one [n_views, H, W, C] tensor (None on other ranks)."""
    import torch
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return images
    world, rank = dist.get_world_size(), dist.get_rank()
    counts = [len(shard_views(n_views, world, r)) for r in range(world)]
    kmax = max(counts)
    padded = torch.zeros((kmax,) + tuple(images.shape[1:]), dtype=images.dtype, device=images.device)
    padded[: images.shape[0]] = images
    bufs = [torch.empty_like(padded) for _ in range(world)] if rank == 0 else None
    dist.gather(padded, gather_list=bufs, dst=0)
    if rank != 0:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)
