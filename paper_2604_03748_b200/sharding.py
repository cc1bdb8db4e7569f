"""Frame sharding across GPUs.

Frames are independent (the density is "streamed directly into
the guiding map generation" frame by frame; Algorithm 1 is per ray, L394), so
the batch is partitioned by frame with no data-path collective: rank r of P
marches the frames f with f mod P == r (cyclic, which balances slowly varying
per-frame cost such as a rotating camera or a growing plume).  Jitter is keyed
by the GLOBAL frame id (C4), so every shard's output is bit-identical
to the same frames of an unsharded run.

The only collective is the optional result gather to rank 0 (NCCL over
NVLink on GPUs; gloo works for the CPU tests): every rank contributes a tensor
of identical shape [F_per_rank, ...] (shards are padded to equal length) and
rank 0 receives them in rank order and undoes the cyclic interleave.
"""
from __future__ import annotations

from typing import List, Sequence


def shard_frames(n_frames: int, world: int, rank: int) -> List[int]:
    """Global frame ids of `rank` under cyclic sharding."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    return list(range(rank, n_frames, world))


def shard_len(n_frames: int, world: int) -> int:
    """Padded per-rank shard length (the gather needs equal shapes)."""
    return (n_frames + world - 1) // world


def unshard_order(n_frames: int, world: int) -> List[int]:
    """Index into the rank-major concatenation [rank][slot] for each global frame."""
    L = shard_len(n_frames, world)
    return [(f % world) * L + f // world for f in range(n_frames)]


def gather_frames(local, n_frames: int, group=None):
    """Gather per-rank outputs to rank 0 and restore global frame order.

    local: tensor [L, ...] with L = shard_len(n_frames, world) (pad rows beyond
    the rank's real frames are ignored).  Returns the [n_frames, ...] tensor on
    rank 0 and None elsewhere.  Uses torch.distributed.gather (NCCL: grouped
    send/recv; gloo on CPU)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    L = shard_len(n_frames, world)
    if local.shape[0] != L:
        raise ValueError(f"local shard must have {L} rows, got {local.shape[0]}")
    bufs = [torch.empty_like(local) for _ in range(world)] if rank == 0 else None
    dist.gather(local.contiguous(), bufs, dst=0, group=group)
    if rank != 0:
        return None
    cat = torch.cat(bufs, dim=0)
    idx = torch.tensor(unshard_order(n_frames, world), device=cat.device)
    return cat.index_select(0, idx)


def pad_shard(t, n_frames: int, world: int, rank: int):
    """Pad a rank's [n_real, ...] output to shard_len rows (zeros)."""
    import torch
    L = shard_len(n_frames, world)
    if t.shape[0] == L:
        return t
    pad = torch.zeros((L - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    return torch.cat([t, pad], dim=0)
