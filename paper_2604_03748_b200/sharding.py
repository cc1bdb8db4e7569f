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

ChunkedGather overlaps that gather with the march (SURVEY §8(e) "Overlap"):
each rank's padded shard [L, ...] is marched in chunks of c frames; as soon as
chunk k is done on the compute stream it is sent to rank 0 on a communication
stream (point-to-point sends, one receive per peer on rank 0, grouped so NCCL
runs them concurrently) while chunk k+1 marches.  Rank 0 receives peer r's
chunk straight into its rank-major result buffer out[r, k*c:(k+1)*c] and marches
its own frames into out[0], so nothing is copied twice; unshard_order maps a
global frame to its row of out.view(P*L, ...).
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


def chunk_bounds(L: int, chunk: int) -> List[tuple]:
    """[start, end) rows of each chunk of a padded shard of L rows (the last may be short)."""
    if chunk < 1:
        raise ValueError("chunk must be >= 1")
    return [(a, min(a + chunk, L)) for a in range(0, L, chunk)]


class ChunkedGather:
    """Chunked result gather to rank 0, overlapped with the march (module docstring).

    bufs: the per-rank shard buffers, one tensor per output kind (e.g. rgbt [L,H,W,4] and
    depth [L,H,W]); on rank 0 these are out[0] views of the rank-major result tensors
    `outs` ([P, L, ...] each), on the other ranks plain [L, ...] tensors.  After chunk k
    rows a:b of every buf are final on the compute stream, call send_chunk(a, b); at the
    end call finish().  NCCL: device tensors, the sends/receives run on `comm_stream`
    (which first waits for the compute stream), so they overlap the next chunk's march.
    gloo (CPU tests, ranks sharing one GPU): tensors are staged through host memory and
    the exchange is synchronous."""

    def __init__(self, bufs, outs=None, group=None, comm_stream=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.bufs = list(bufs)
        self.outs = None if outs is None else list(outs)
        if self.rank == 0 and self.outs is None:
            raise ValueError("rank 0 needs the rank-major result tensors")
        self.nccl = dist.get_backend(group) == "nccl"
        self.comm = comm_stream
        self.works = []

    def send_chunk(self, a: int, b: int):
        import torch
        dist = self.dist
        if self.world == 1:
            return
        if self.nccl:
            ev = torch.cuda.Event()
            ev.record()                                   # the chunk's march on the compute stream
            self.comm.wait_event(ev)
            with torch.cuda.stream(self.comm):
                ops = []
                for t, o in zip(self.bufs, self.outs or [None] * len(self.bufs)):
                    if self.rank == 0:
                        for r in range(1, self.world):
                            ops.append(dist.P2POp(dist.irecv, o[r, a:b], r, self.group))
                    else:
                        ops.append(dist.P2POp(dist.isend, t[a:b], 0, self.group))
                self.works += dist.batch_isend_irecv(ops)
            return
        # gloo: host staging, synchronous
        for i, t in enumerate(self.bufs):
            if self.rank == 0:
                for r in range(1, self.world):
                    h = torch.empty(t[a:b].shape, dtype=t.dtype)
                    dist.recv(h, src=r, group=self.group)
                    self.outs[i][r, a:b].copy_(h)
            else:
                dist.send(t[a:b].detach().cpu().contiguous(), dst=0, group=self.group)

    def finish(self):
        """Make the current stream wait for every outstanding send/receive."""
        import torch
        if self.nccl and self.works:
            with torch.cuda.stream(self.comm):
                for w in self.works:
                    w.wait()
            torch.cuda.current_stream().wait_stream(self.comm)
        self.works = []
