"""Multi-rank frame sharding on the GPU: two or four ranks that share cuda:0 (gloo
process group: the 1-GPU test box cannot host NCCL ranks) march their cyclic shards of a
C2 batch through the C ABI, chunk by chunk, and gather every chunk to rank 0
(sharding.ChunkedGather, host-staged under gloo).  The gathered maps must equal a
single-rank run of the same frames bit for bit (jitter is keyed by the global frame id and
the march uses no atomics).  The ranks' kernels never wait on one another."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FRAMES = list(range(0, 60, 6))          # 10 C2 frames


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, chunk, out_path):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import nsl_inputs as I
    import paper_2604_03748_b200 as nsl
    from paper_2604_03748_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    full = I.make_workload("C2", frames=FRAMES)
    F = full.n_frames
    L = sharding.shard_len(F, world)
    mine = sharding.shard_frames(F, world, rank)
    w = full.subset(mine)
    H, W = w.height, w.width
    if rank == 0:
        outs = [torch.zeros((world, L, H, W, 4), device="cuda"), torch.zeros((world, L, H, W), device="cuda")]
        bufs = [outs[0][0], outs[1][0]]
    else:
        outs = None
        bufs = [torch.zeros((L, H, W, 4), device="cuda"), torch.zeros((L, H, W), device="cuda")]
    vols = nsl.upload_workload_volumes(w, 3)
    g = sharding.ChunkedGather(bufs, outs)
    for a, b in sharding.chunk_bounds(L, chunk):
        e = min(b, len(mine))
        if a < e:
            sub = w.subset(list(range(a, e)))
            plan = nsl.Plan(vols, sub.frame_vol, sub.cameras, sub.lights, sub.light_mode, sub.medium, sub.march,
                            sub.frame_ids)
            plan.execute(bufs[0][a:e], bufs[1][a:e])
        torch.cuda.synchronize()
        g.send_chunk(a, b)
    g.finish()
    if rank == 0:
        order = torch.tensor(sharding.unshard_order(F, world), device="cuda")
        rg = outs[0].reshape(world * L, H, W, 4).index_select(0, order)
        dp = outs[1].reshape(world * L, H, W).index_select(0, order)
        np.savez(out_path, rgbt=rg.cpu().numpy(), depth=dp.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,chunk", [(2, 2), (2, 16), (4, 1)])
def test_ranks_gathered_equal_single_rank(tmp_path, world, chunk):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    import nsl_inputs as I
    import paper_2604_03748_b200 as nsl
    out = str(tmp_path / "gathered.npz")
    mp.get_context("spawn")
    mp.spawn(_worker, args=(world, _free_port(), chunk, out), nprocs=world, join=True)
    got = np.load(out)
    w = I.make_workload("C2", frames=FRAMES)
    rgbt, depth, _ = nsl.run_workload(w, layout=3)
    torch.cuda.synchronize()
    assert np.array_equal(got["rgbt"].view(np.uint32), rgbt.cpu().numpy().view(np.uint32))
    assert np.array_equal(got["depth"].view(np.uint32), depth.cpu().numpy().view(np.uint32))


def test_bench_self_launches_two_ranks_strong_scaling():
    """`bench.py --gpus 2` outside torchrun re-launches itself as two ranks; the strong-scaling
    step (fixed batch split over the ranks, chunked gather to rank 0 inside the timed region)
    prints one JSON line with n_gpus = 2."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                        "--scaling", "strong", "--config", "C2", "--frames", "12", "--chunk", "4",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["frames_total"] == 12 and d["gather_bytes_to_rank0_per_step"] == 6 * 512 * 512 * 20


def test_bench_self_launches_two_ranks_weak_default():
    """The default (weak-scaling) bench path under two self-launched ranks: one JSON line,
    n_gpus = 2, frames_total = 2 x frames_per_rank, max-over-ranks timing."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA GPU")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--backend", "gloo",
                        "--frames", "6", "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-e2e",
                        "--no-sampler-ceiling"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["frames_total"] == 12 and d["config"]["frames_per_rank"] == 6
