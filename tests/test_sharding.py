"""Multi-process (world_size 2, gloo, CPU) tests of the frame sharding and the
result gather: shards are disjoint and cover every frame, and
gathering per-rank outputs to rank 0 restores the global frame order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_03748_b200 import sharding


def test_shard_cover_and_order():
    for F in (1, 7, 60, 240, 1024):
        for P in (1, 2, 3, 4, 8):
            shards = [sharding.shard_frames(F, P, r) for r in range(P)]
            flat = sorted(f for s in shards for f in s)
            assert flat == list(range(F))
            L = sharding.shard_len(F, P)
            assert all(len(s) <= L for s in shards)
            order = sharding.unshard_order(F, P)
            # order maps each global frame to its (rank, slot) in the rank-major concatenation
            for f, k in enumerate(order):
                r, slot = divmod(k, L)
                assert shards[r][slot] == f
    with pytest.raises(ValueError):
        sharding.shard_frames(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, F, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = sharding.shard_frames(F, world, rank)
    # a stand-in "guiding map" per frame whose content encodes the global frame id
    local = torch.stack([torch.full((3, 5, 4), float(f)) for f in mine]) if mine else torch.zeros((0, 3, 5, 4))
    local = sharding.pad_shard(local, F, world, rank)
    full = sharding.gather_frames(local, F)
    if rank == 0:
        torch.save(full, out_path)
    else:
        assert full is None
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("F", [8, 7, 1])
def test_gather_world2_gloo(tmp_path, F):
    out = str(tmp_path / "full.pt")
    mp.spawn(_worker, args=(2, _free_port(), F, out), nprocs=2, join=True)
    full = torch.load(out)
    assert full.shape == (F, 3, 5, 4)
    for f in range(F):
        assert torch.all(full[f] == float(f))


def test_bench_rank_workloads_partition_frames():
    """bench.py's weak-scaling workload: each rank marches distinct global frame ids
    (rank + world*k), so N ranks together cover N*F_rank distinct frames."""
    import importlib.util
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    sys.modules["bench_mod"] = bench
    spec.loader.exec_module(bench)
    world = 4
    ids = []
    for r in range(world):
        w = bench.rank_workload("C2", r, world, 6)
        assert w.n_frames == 6
        ids += list(w.frame_ids)
        assert w.frame_ids == sharding.shard_frames(6 * world, world, r)
    assert sorted(ids) == list(range(24))


def _chunk_worker(rank, world, port, F, chunk, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = sharding.shard_len(F, world)
    mine = sharding.shard_frames(F, world, rank)
    if rank == 0:
        outs = [torch.full((world, L, 3, 5, 4), -1.0), torch.full((world, L, 3, 5), -1.0)]
        bufs = [outs[0][0], outs[1][0]]
    else:
        outs = None
        bufs = [torch.full((L, 3, 5, 4), -1.0), torch.full((L, 3, 5), -1.0)]
    g = sharding.ChunkedGather(bufs, outs)
    for a, b in sharding.chunk_bounds(L, chunk):
        for i in range(a, min(b, len(mine))):          # the stand-in "march" of the chunk's real frames
            bufs[0][i] = float(mine[i])
            bufs[1][i] = 1000.0 + mine[i]
        g.send_chunk(a, b)
    g.finish()
    if rank == 0:
        order = torch.tensor(sharding.unshard_order(F, world))
        torch.save((outs[0].reshape(world * L, 3, 5, 4)[order], outs[1].reshape(world * L, 3, 5)[order]), out_path)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,F,chunk", [(2, 8, 3), (2, 7, 2), (2, 9, 16), (2, 2, 1), (3, 10, 2), (4, 9, 1)])
def test_chunked_gather_gloo(tmp_path, world, F, chunk):
    """ChunkedGather (the bench's overlapped result gather): chunk by chunk, rank 0 receives
    every peer's rows straight into the rank-major result; unshard_order restores frame order
    (world sizes 2-4, ragged F, chunks smaller and larger than the shard)."""
    out = str(tmp_path / "full.pt")
    mp.spawn(_chunk_worker, args=(world, _free_port(), F, chunk, out), nprocs=world, join=True)
    rgbt, depth = torch.load(out)
    assert rgbt.shape == (F, 3, 5, 4) and depth.shape == (F, 3, 5)
    for f in range(F):
        assert torch.all(rgbt[f] == float(f)) and torch.all(depth[f] == 1000.0 + f)


def test_chunk_bounds():
    assert sharding.chunk_bounds(10, 4) == [(0, 4), (4, 8), (8, 10)]
    assert sharding.chunk_bounds(3, 8) == [(0, 3)]
    with pytest.raises(ValueError):
        sharding.chunk_bounds(3, 0)
