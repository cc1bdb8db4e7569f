#!/usr/bin/env python
"""Benchmark of the B200 guiding-map ray march (Algorithm 1) — see DESIGN.md §7.

One *step* = one pass of the whole hot path over one batch: the volume
layout (row a1, from the device-resident raw grid) plus the batched march of
all frames of BASELINE.json configs[1] (C2: chimney plume 128^3, 60 frames of
512x512, rotating camera, guide lights), rows a2-a9: 4 kernel launches per
step (layout, occupancy, frame setup, march) from device-resident inputs via a
prepared plan (nsl_plan_execute).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config C2]

Multi-GPU (torchrun, one process per GPU; `--gpus N` outside torchrun re-launches
itself as N ranks): frames are independent, so by default each rank marches its
own 60 frames (global frame ids rank + N*k, weak scaling) with no data-path
collective; time = max over ranks of the device-timed loop.  `--scaling strong`
splits the config's fixed batch (C4: 240, C5: 1024 frames) cyclically over the
ranks and `--gather` gathers every step's guiding maps to rank 0 inside the
timed step (chunked, overlapped with the march).  Rank 0
prints ONE JSON line.
"""
import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "guiding-map rays/s and march samples/s; ms/frame at 512² over 128³; frames/s @1/2/4/8 GPU"
CONFIG_TEXT = {
    "C1": "C1: puff 64^3, 1 frame 128x128, guide lights",
    "C2": "C2: chimney plume 128^3, 60 frames x 512x512, rotating camera, guide lights",
    "C3": "C3: obstacle-carved plume 256^3, 60 frames x 1024x1024, moving light",
    "C4": "C4: animated plume 256^3 (distinct volume per frame), 1024x1024, guide lights",
    "C5": "C5: plume 512^3, 2048x2048 frames, guide lights",
    "P482": "P482: the paper's timed workload (PAPER.md:482): plume 400^3, one 512x512 frame per step "
            "(a fresh volume layout every step, as when the simulation streams density in), guide lights",
}
# frames on each config's camera path, and the frames one step marches by default
N_PATH = {"C1": 1, "C2": 60, "C3": 60, "C4": 240, "C5": 1024, "P482": 60}
N_STEP = dict(N_PATH, P482=1)
# the paper's only number for this path: ~2 ms per 512^2 frame over 400^3 (an
# unnamed 16,384-core 24 GB GPU, RTX-4090 class) = 131 M rays/s
PAPER_P482 = {"ms_per_frame": 2.0, "rays_per_s": 512 * 512 / 2e-3, "source": "PAPER.md:482 (§5 Performance)",
              "hardware": "a GPU with 16,384 cores and 24 GB (RTX-4090 class, inferred)"}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="nsl", choices=["nsl", "reference"])
    p.add_argument("--config", default="C2", choices=sorted(CONFIG_TEXT),
                   help="C1-C5: BASELINE.json's configs (C2 = the headline); P482: the paper's own timed workload")
    p.add_argument("--frames", type=int, default=0, help="frames per rank (default: the config's)")
    p.add_argument("--layout", default="auto", choices=["linear_f32", "quad_f32", "corner_f16", "oct_f32",
                                                        "brick_oct_f32", "tex3d_f32", "morton_oct_f32", "auto"],
                   help="auto (default): the library's size-based choice (nsl_layout_resolve)")
    p.add_argument("--light-model", default="march", choices=["march", "tv"],
                   help="march: canonical C8 (the headline); tv: NEXT-4 transmittance volume (DESIGN.md §12)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--gather", action="store_true",
                   help="N>1: gather every step's guiding maps to rank 0 inside the timed step (chunked, overlapped)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-sampler-ceiling", action="store_true",
                   help="skip the sampler microbenchmark after the timed region (ncu launch lists)")
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target oracle sample time")
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: every rank its own F frames (default); strong: the config's fixed batch "
                        "(C4: 240, C5: 1024 frames) split cyclically over the ranks")
    p.add_argument("--chunk", type=int, default=0,
                   help="sharded runs: frames per chunk (a gathered chunk's send overlaps the next chunk's march)")
    p.add_argument("--graph", action="store_true",
                   help="time replays of the step captured as a CUDA graph (volume rebuild + plan execute)")
    p.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                   help="process group backend (gloo: functional runs of ranks sharing one GPU, host-staged gather)")
    return p.parse_args()


# ------------------------------------------------------------------ clocks during the timed region
class ClockSampler:
    REASONS = {"gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
               "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

    def __init__(self, index):
        self.index, self.samples, self.reasons, self.max_mhz = index, [], set(), None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # no NVML: report nothing rather than guess
            self.error = str(e)
            return self

        def loop():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for k, bit in self.REASONS.items():
                        if r & bit and k != "gpu_idle":
                            self.reasons.add(k)
                except Exception:
                    pass
                time.sleep(0.005)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "n_samples": len(self.samples)}


# ------------------------------------------------------------------ workload
def rank_workload(cfg, rank, world, frames_per_rank):
    """Weak scaling: rank r marches frames_per_rank frames with global ids r + world*k."""
    import nsl_inputs as I
    base = I.make_workload(cfg, frames=[0])
    n_cfg = N_PATH[cfg]
    F = frames_per_rank or N_STEP[cfg]
    gids = [rank + world * k for k in range(F)]
    full = I.make_workload(cfg, frames=None) if cfg in ("C1", "C2", "C3", "P482") else None
    if cfg in ("C1", "C2", "C3", "P482"):
        # extend the camera/light path periodically to world*F global frames
        idx = [g % n_cfg for g in gids]
        w = full.subset(idx)
        w.frame_ids = gids
        return w
    return I.make_workload(cfg, frames=[g % n_cfg for g in gids])


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ CPU oracle timing
def time_oracle(cfg, seconds, max_frames=None, stride=1):
    """The oracle, as it stands (single-threaded C), on frames of the workload (every
    `stride`-th pixel) until ~`seconds` of CPU work or `max_frames` frames; returns
    rays/s, samples/s and the sample description."""
    import oracle
    import nsl_inputs as I
    w = I.make_workload(cfg, frames=[0])
    n_cfg = N_PATH[cfg]
    rays = samples = 0
    t_total = 0.0
    frames = []
    fstride = 4                             # frames 0, 4, 8, ... of the camera path
    f = 0
    while (len(frames) < max_frames) if max_frames is not None else (t_total < seconds or not frames):
        wf = I.make_workload(cfg, frames=[f % n_cfg])
        sub = stride * (16 if cfg == "C4" else 64 if cfg == "C5" else 1)
        pix = np.arange(0, wf.width * wf.height, sub) if sub > 1 else None
        wf.volume(0)                        # generation is not oracle work
        t0 = time.perf_counter()
        r = oracle.run_workload_frame(wf, 0, pixels=pix)
        dt = time.perf_counter() - t0
        d = r["debug"].astype(np.int64)
        samples += int(np.where(d[:, 0] > 0, d[:, 3] - d[:, 0] + 1, 0).sum() + d[:, 5].sum())
        rays += len(r["pixels"])
        t_total += dt
        frames.append(f % n_cfg)
        f += fstride
    desc = (f"oracle (plain C, fp64, 1 thread) on {len(frames)} frame(s) {frames[:6]}{'...' if len(frames) > 6 else ''}"
            f" of {cfg}" + (f" (every {sub}th pixel)" if sub > 1 else " (all pixels)"))
    return {"rays_per_s": rays / t_total, "samples_per_s": samples / t_total, "seconds": t_total,
            "sample": desc, "rays": rays}


def host_cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------ reference arm (the oracle)
def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    # each step = one frame of the workload, pixel-subsampled so that the whole
    # (K + W)-step run stays within ~90 s of single-core oracle work
    stride = max(1, math.ceil((args.steps + args.warmup) * 0.25 / 90.0))
    for _ in range(args.warmup):
        time_oracle(cfg, 0.0, max_frames=1, stride=stride)
    res = time_oracle(cfg, 0.0, max_frames=max(1, args.steps), stride=stride)
    v = res["rays_per_s"]
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "rays/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * res["seconds"] / max(1, args.steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[cfg], "reference": "CPU oracle (no upstream code exists)",
                       "step": "one frame of the workload per step"},
            "samples_per_s": res["samples_per_s"],
            "cpu_baseline": {"value": v, "unit": "rays/s", "cores": 1, "kind": "oracle", "sample": res["sample"],
                             "cpu": host_cpu_name()},
            "e2e": {"value": v, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def sampler_ceiling(layout, counts, march_s):
    import torch
    import nsl_inputs as I
    import paper_2604_03748_b200 as nsl
    n = 16
    rng = np.random.default_rng(7)
    dens = torch.from_numpy((0.5 + 0.1 * rng.random((n, n, n))).astype(np.float32)).cuda()
    vol = nsl.Volume(I.Grid(n, n, n, (0.0, 0.0, 0.0), 1.0 / n), dens, layout)
    sink = torch.empty(148 * 16 * 4 * 128, dtype=torch.float32, device="cuda")
    nsl.bench_l1_gather(vol, sink)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        samples = nsl.bench_l1_gather(vol, sink)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    peak = samples / statistics.median(ts)
    gathers = counts["gathers"] / march_s
    tested = (counts["tested_primary"] + counts["tested_light"]) / march_s
    return {"samples_per_s": peak, "source": "nsl_bench_l1_gather, 16^3 fully occupied grid, same layout",
            "executed_gathers_per_s": gathers, "frac_gathers": gathers / peak,
            "tested_samples_per_s": tested, "frac_tested": tested / peak}



def l1_patterns(w, nsl):
    """Lane element offsets [16, 32] for the hardware L1/TEX ceiling (nsl_bench_l1_peak), all in
    the OCT layout of w's grid (one 32-B element per trilinear sample):
      footprint: the march's warp footprint -- the 8 x 4 pixels at the image centre of frame 0,
        every lane at the same ray parameter, patterns 0-7 at 8 consecutive primary steps
        through the volume centre, 8-15 at light steps 1..8 of the guide set's first side light
        (else the only light) from the middle sample (the roofline's peak: the larger, stricter
        denominator);
      footprint_jitter: the same with each lane at its own C4 jitter (t = delta_lane + n h),
        i.e. the march's actual gathers: ~19-22 distinct 128-B lines per warp load;
      coalesced: 32 consecutive elements per pattern (8 distinct 128-B lines per load);
      broadcast: one element for every lane."""
    g = w.grid
    fc = nsl.debug_frame_constants(g, w.cameras[0], w.lights[0], w.light_mode, w.medium, w.march)
    sy, sz = g.nx + 1, (g.nx + 1) * (g.ny + 1)
    W, H = w.width, w.height
    lane = np.arange(32)
    px = (W // 2 - 4) + lane % 8
    py = (H // 2 - 2) + lane // 8
    B, Ex, Ey, Dg = (np.asarray(fc[k], np.float64) for k in ("B", "Ex", "Ey", "Dg"))
    O = B[None, :] + px[:, None] * Ex[None, :] + py[:, None] * Ey[None, :]
    centre = np.array([g.nx, g.ny, g.nz], np.float64) / 2.0 + 0.5
    hidx = w.march.step / g.voxel_width                                   # h in index units
    dlen = np.linalg.norm(Dg)
    tc = float(np.dot(centre - O[0], Dg) / dlen ** 2)                     # ray parameter at the centre
    h = w.march.step
    tc = h * round(tc / h)
    import torch
    hh = torch.empty(W * H, dtype=torch.int32, device="cuda")
    dd = torch.empty(W * H, dtype=torch.float32, device="cuda")
    nsl.debug_jitter(w.march, w.frame_ids[0], hh, dd)                     # C4 delta of every pixel
    delta = dd.cpu().numpy().astype(np.float64)[py * W + px]
    li = 1 if len(fc["Lg"]) > 1 else 0                                    # a side light, else the only light
    L = np.asarray(fc["Lg"][li], np.float64) * h                          # one light step (index units)
    lim = np.array([g.nx, g.ny, g.nz], np.float64)

    def offsets(dl):
        pos = [O + (tc + (k - 4) * h + dl)[:, None] * Dg[None, :] for k in range(8)]
        pos += [pos[4] + j * L[None, :] for j in range(1, 9)]
        e = []
        for u in pos:
            c = np.clip(np.floor(u), 0, lim).astype(np.int64)
            e.append(c[:, 0] + c[:, 1] * sy + c[:, 2] * sz)
        e = np.stack(e)
        return e - e.min()

    coal = np.arange(16)[:, None] * 32 + lane[None, :]
    bcast = np.zeros((16, 32), np.int64)
    return {"footprint": offsets(np.zeros(32)), "footprint_jitter": offsets(delta), "coalesced": coal,
            "broadcast": bcast}


def l1_hw_ceiling(w, nsl, patterns=("footprint",), stride=0, span=1, reps=256, waves=8, iters=7):
    """Measured lane bytes/s of nsl_bench_l1_peak per lane pattern (CUDA events, median)."""
    import torch
    pats = l1_patterns(w, nsl)
    out = {}
    for name in patterns:
        off = torch.from_numpy(pats[name].astype(np.int32)).cuda()
        max_off = int(pats[name].max())
        buf = torch.ones((span + max_off + 1) * 8, dtype=torch.float32, device="cuda")
        sink = torch.empty(148 * 8 * 256 * waves, dtype=torch.float32, device="cuda")
        nbytes = nsl.bench_l1_peak(buf, off, stride, span, waves, reps, sink)
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nsl.bench_l1_peak(buf, off, stride, span, waves, reps, sink)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        t = statistics.median(ts)
        lines = [len(set((pats[name][k] * 32 // 128).tolist())) for k in range(16)]
        out[name] = {"lane_gbs": nbytes / t / 1e9, "launch_ms": t * 1e3, "bytes": nbytes,
                     "lines_per_load": float(np.mean(lines))}
    return out


def launches_per_step(w, args, nsl, layout) -> int:
    """Kernels of one timed step: the volume build per distinct volume (nsl_volume_build_launches:
    occ_reset + oct_build + occ_finalize, or volume_build + occ_finalize), then frame_setup,
    tile_cull and march_kernel; the TV light model adds tv_setup and, per frame group
    (NSL_TV_BUDGET_MB, the library's host bound), tv_sweep + tile_cull + march_kernel."""
    n = nsl.volume_build_launches(w.grid, layout) * len(w.volume_specs) + 1
    if args.light_model != "tv":
        return n + 2
    g = w.grid
    diag = math.sqrt((g.nx + 1) ** 2 + (g.ny + 1) ** 2 + (g.nz + 1) ** 2)
    hl = w.march.light_step if w.march.light_step > 0 else w.march.step
    astr = math.ceil(diag) + 6
    kstr = math.ceil(diag / (hl / g.voxel_width * (1 - 1e-5))) + 6
    slots = 1 if w.light_mode == 1 else len(w.lights[0])
    per_frame = 8 * astr * astr * kstr * slots
    group = max(1, min(w.n_frames, int(float(os.environ.get("NSL_TV_BUDGET_MB", "4096")) * 1048576 // per_frame)))
    group = min(group, 65535 // slots)
    return n + 1 + 3 * math.ceil(w.n_frames / group)


def max_over_ranks(x: float, backend: str) -> float:
    """Max of a host float over all ranks (device tensor for NCCL, host tensor for gloo)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def self_launch(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-run this command as N ranks
    under torch.distributed.run on 127.0.0.1 (one process per GPU) and return its exit code."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ sharded runs (--scaling strong / --gather)
def run_sharded(args, rank, world, local):
    """Frame-sharded step with the result gather to rank 0 inside the timed region (SURVEY
    §8(d): t_P from a barrier to gather completion on rank 0; §8(e): cyclic shards, chunked
    gather overlapped with the march).  strong: the config's fixed batch (C2 60, C3 60, C4 240,
    C5 1024 frames) over the ranks; weak: every rank F frames.  One step: per chunk of the
    rank's padded shard, the layouts of the chunk's volumes (every chunk when frames view
    different volumes -- C4 -- else once per step), the chunk's plan (frame setup, cull,
    march) into its rows of the shard, then the chunk's send to rank 0 on a side stream."""
    import torch
    import torch.distributed as dist
    import nsl_inputs as I
    import paper_2604_03748_b200 as nsl
    from paper_2604_03748_b200 import sharding

    cfg = args.config
    layout = nsl.LAYOUTS[args.layout]
    n_cfg = N_PATH[cfg]
    if args.scaling == "strong":
        F_total = args.frames or N_STEP[cfg]
        mine = sharding.shard_frames(F_total, world, rank)
        full = I.make_workload(cfg, frames=[0]) if cfg in ("C4", "C5") else I.make_workload(cfg)
        w = (I.make_workload(cfg, frames=[g % n_cfg for g in mine]) if cfg in ("C4", "C5")
             else full.subset([g % n_cfg for g in mine]))
        w.frame_ids = list(mine)
    else:
        w = rank_workload(cfg, rank, world, args.frames)
        F_total = w.n_frames * world
    layout = nsl.layout_resolve(w.grid, layout)
    if args.light_model == "tv":
        from dataclasses import replace
        w = replace(w, march=replace(w.march, light_model=1))
    L = sharding.shard_len(F_total, world) if args.scaling == "strong" else w.n_frames
    n_real, H, W = w.n_frames, w.height, w.width
    animated = len(w.volume_specs) > 1
    chunk = args.chunk or (max(1, min(L, 8 if animated else 16)))
    nbl = nsl.volume_build_launches(w.grid, layout)
    bounds = sharding.chunk_bounds(L, chunk)
    stream = torch.cuda.current_stream()

    # inputs resident in HBM: raw densities of the rank's volumes; layout storage for one chunk
    # of per-frame volumes (animated) or the single volume; outputs (rank 0: the rank-major
    # result tensors of all ranks, its own shard = row 0)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=4) as ex:
        host = list(ex.map(w.volume, range(len(w.volume_specs))))
    raw = [torch.from_numpy(v).cuda() for v in host]
    del host
    nslot = chunk if animated else 1
    storage = [torch.empty(nsl.volume_bytes(w.grid, layout), dtype=torch.uint8, device="cuda") for _ in range(nslot)]
    if rank == 0:
        outs = [torch.empty((world, L, H, W, 4), dtype=torch.float32, device="cuda"),
                torch.empty((world, L, H, W), dtype=torch.float32, device="cuda")]
        bufs = [outs[0][0], outs[1][0]]
    else:
        outs = None
        bufs = [torch.empty((L, H, W, 4), dtype=torch.float32, device="cuda"),
                torch.empty((L, H, W), dtype=torch.float32, device="cuda")]
    comm = torch.cuda.Stream() if args.backend == "nccl" else None

    # one plan per chunk (its real frames), built once: frame tables uploaded; the chunk's volume
    # slots (animated) or the single volume are rebuilt in place every step (nsl_volume_rebuild)
    slot_vols = [nsl.Volume(w.grid, raw[0], layout, storage=st) for st in storage] if animated else None
    static_vol = None if animated else [nsl.Volume(w.grid, raw[0], layout, storage=storage[0])]
    plans = []
    for a, b in bounds:
        frames = list(range(a, min(b, n_real)))
        if not frames:
            plans.append(None)
            continue
        sub = w.subset(frames)
        fv = list(range(len(frames))) if animated else [0] * len(frames)
        plans.append(nsl.Plan(slot_vols[:len(frames)] if animated else static_vol, fv, sub.cameras, sub.lights,
                              sub.light_mode, sub.medium, sub.march, sub.frame_ids))
    torch.cuda.synchronize()

    def step():
        g = sharding.ChunkedGather(bufs, outs, comm_stream=comm) if world > 1 else None
        if not animated:
            static_vol[0].rebuild(raw[0])                                    # a1: the volume, once per step
        for (a, b), plan in zip(bounds, plans):
            if plan is not None:
                if animated:                                                 # a1: this chunk's layouts
                    for i, f in enumerate(range(a, min(b, n_real))):
                        slot_vols[i].rebuild(raw[w.frame_vol[f]])
                e = min(b, n_real)
                plan.execute(bufs[0][a:e], bufs[1][a:e])                     # a2-a9
            if g is not None:
                g.send_chunk(a, b)
        if g is not None:
            g.finish()

    step()
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    K = args.steps
    clocks = ClockSampler(local).start()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    times = []
    for _ in range(K):
        flush.zero_()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)                   # after finish(): the last receive on rank 0
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    clk = clocks.stop()
    t_loop = sum(times)
    if world > 1:
        t_loop = max_over_ranks(t_loop, args.backend)
    rays = W * H * F_total * K
    line = {"metric": METRIC, "value": rays / t_loop, "unit": "rays/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_loop / K, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f16" if layout == 2 else "f32",
            "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[cfg], "frames_total": F_total, "frames_per_rank": L,
                       "map": f"{W}x{H}", "grid": f"{w.grid.nx}^3", "layout": nsl.LAYOUT_NAMES[layout] + (" (auto)" if args.layout == "auto" else ""),
                       "light_model": args.light_model, "chunk_frames": chunk,
                       "l2": "flushed (512 MiB write) before each timed step, outside the events",
                       "parallelism": f"frame-sharded x{world} (cyclic), results gathered to rank 0 "
                                      f"inside the step ({args.backend}, chunked, overlapped)"},
            "frames_per_s": F_total * K / t_loop, "ms_per_frame": 1e3 * t_loop / (K * F_total),
            "gather_bytes_to_rank0_per_step": int((world - 1) * L * H * W * 20),
            "gpu_launches": K * sum(nbl * (len(p._vols) if animated else 0) + 3 for p in plans if p is not None)
                            + (K * nbl if not animated else 0),
            "clocks": clk}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return line


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import torch.distributed as dist
    import paper_2604_03748_b200 as nsl

    dev = local % max(1, torch.cuda.device_count())        # ranks may share a GPU (gloo functional runs)
    torch.cuda.set_device(dev)
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    if args.scaling == "strong" or (args.gather and world > 1):
        run_sharded(args, rank, world, dev)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return
    cfg = args.config
    w = rank_workload(cfg, rank, world, args.frames)
    layout = nsl.layout_resolve(w.grid, nsl.LAYOUTS[args.layout])
    if args.light_model == "tv":
        from dataclasses import replace
        w = replace(w, march=replace(w.march, light_model=1))
    F, H, W = w.n_frames, w.height, w.width
    stream = torch.cuda.current_stream()

    # inputs resident in HBM before timing: raw density grids + layout storage + outputs
    raw = [torch.from_numpy(w.volume(i)).cuda() for i in range(len(w.volume_specs))]
    storage = [torch.empty(nsl.volume_bytes(w.grid, layout), dtype=torch.uint8, device="cuda") for _ in raw]
    outputs = nsl.alloc_outputs(F, H, W, debug=False)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    # per-frame inputs (cameras, lights, frame ids, volume storage) marshalled and uploaded once
    vols = [nsl.Volume(w.grid, r, layout, storage=s) for r, s in zip(raw, storage)]
    plan = nsl.make_plan(w, vols)

    def step():
        for v, r in zip(vols, raw):
            v.rebuild(r)                                                                       # a1
        plan.execute(outputs[0], outputs[1])                                                   # a2-a9

    step()
    torch.cuda.synchronize()
    counts = plan.execute_counted(outputs[0], outputs[1])
    torch.cuda.synchronize()

    for _ in range(args.warmup):
        flush.zero_()
        step()
    torch.cuda.synchronize()

    K = args.steps
    graph = None
    if args.graph:                          # the step as one CUDA graph (its PDL edges captured)
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for v, r in zip(vols, raw):
                v.rebuild(r, stream=gs)
            plan.execute(outputs[0], outputs[1], stream=gs)
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    # the timed steps: events only around the whole step, so the frame setup's programmatic
    # dependent launch overlaps the volume build's finalize as it does in production
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    clocks = ClockSampler(dev).start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for i in range(K):
        flush.zero_()                       # L2 flushed between timed iterations (outside the events)
        e0, e2 = ev[i]
        e0.record(stream)
        if graph is not None:
            graph.replay()
        else:
            for v, r in zip(vols, raw):
                v.rebuild(r)                    # a1
            plan.execute(outputs[0], outputs[1])   # a2-a9
        e2.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(c) for a, c in ev]
    t_loop = sum(step_ms) / 1e3
    if world > 1:
        t_loop = max_over_ranks(t_loop, args.backend)
    # the same steps again with an event between the build and the plan: the march's own device
    # time (the roofline's kernel time) and the build's (this event costs the PDL overlap, ~10 us)
    K2 = min(K, 50)
    ev3 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
            torch.cuda.Event(enable_timing=True)) for _ in range(K2)]
    for i in range(K2):
        flush.zero_()
        e0, e1, e2 = ev3[i]
        e0.record(stream)
        for v, r in zip(vols, raw):
            v.rebuild(r)
        e1.record(stream)
        plan.execute(outputs[0], outputs[1])
        e2.record(stream)
    torch.cuda.synchronize()
    march_ms = [b.elapsed_time(c) for a, b, c in ev3]
    layout_ms = [a.elapsed_time(b) for a, b, c in ev3]
    total_rays = W * H * F * world * K
    value = total_rays / t_loop
    ms_step = 1e3 * t_loop / K

    # roofline of the dominant kernel (march_kernel): bound = L1/TEX.  Algorithmic
    # bytes = SURVEY §8(d)'s 32 B (8 fp32 corners) per canonical march sample x the canonical
    # samples of one launch, over the plan's device time (frame setup + cull + march, CUDA events
    # on the launch stream).  Peak = the hardware L1/TEX gather ceiling measured live after the
    # timed region (nsl_bench_l1_peak: ld.global.nc.v8.f32 at this march's own 8 x 4 warp
    # footprint, L1-resident, no sampler arithmetic; profiles/r2_l1_hw_peak.jsonl).  Beside it: the
    # FP32 view in one unit (flops, FMA = 2 on both sides), the gathers actually executed and the
    # sampler's own ceiling.
    peaks = load_peaks()
    march_s = statistics.mean(march_ms) / 1e3
    sm_mhz = clk["sm_max_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    bytes_per_sample = 16 if layout == 2 else 32
    alg_bytes = counts["canonical_samples"] * 32
    l1_achieved = alg_bytes / march_s / 1e9
    try:
        hw = l1_hw_ceiling(w, nsl, patterns=("footprint", "footprint_jitter", "coalesced"))
        # the strictest denominator: the faster of the jitter-free warp footprint and fully coalesced
        # lanes (the footprint's rate depends on its L1 bank pattern: C1/C3 footprints are slower)
        best = max(("footprint", "coalesced"), key=lambda k: hw[k]["lane_gbs"])
        l1_peak = hw[best]["lane_gbs"]
        peak_src = (f"measured: nsl_bench_l1_peak, ld.global.nc.v8.f32, L1-resident, this run; the faster of the "
                    f"march's jitter-free 8x4 warp footprint (frame 0) and coalesced lanes ({best})")
    except Exception as e:                    # never fatal: fall back to the nominal figure, say so
        hw = {"error": str(e)[:200]}
        l1_peak = 148 * 128 * sm_mhz * 1e6 / 1e9
        peak_src = "nominal 148 SMs x 128 B/clk x sm_max_mhz (the measurement failed)"
    flops = 25 * counts["canonical_samples"]        # 25 flops per sample (lerp = 2)
    fp32_peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e9  # GFLOP/s, FMA = 2 flops
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_march_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("config") == cfg and tj.get("layout") == nsl.LAYOUT_NAMES[layout] and tj.get("frames") == F:
                traffic = tj["dram_bytes_per_launch"]
        except Exception:
            traffic = None
    roof = {"bound": "l1tex", "achieved": l1_achieved, "peak": l1_peak, "unit": "GB/s", "frac": l1_achieved / l1_peak,
            "traffic": traffic, "peak_source": peak_src,
            "per_unit": "32 B (8 fp32 corners) per canonical march sample (SURVEY 8(d))",
            "kernel": "march_kernel (+ frame_setup_kernel, tile_cull_kernel: the plan's launch sequence)",
            "kernel_ms": march_s * 1e3, "algorithmic_bytes_per_launch": alg_bytes,
            "canonical_samples_per_launch": counts["canonical_samples"],
            "l1_ceiling": hw,
            "jitter_footprint_view": ({
                "peak_gbs": hw["footprint_jitter"]["lane_gbs"],
                "frac_algorithmic": l1_achieved / hw["footprint_jitter"]["lane_gbs"],
                "frac_executed_gathers": counts["gathers"] * bytes_per_sample / march_s / 1e9
                                         / hw["footprint_jitter"]["lane_gbs"],
                "note": "ceiling of the march's actual jittered lane addresses (C4): the L1 delivers about one "
                        "128-B line per cycle, so ~19 lines per warp gather halve the rate"}
                if "footprint_jitter" in hw else None),
            "fp32_view": {"achieved_gflops": flops / march_s / 1e9, "peak_gflops": fp32_peak,
                          "frac": flops / march_s / 1e9 / fp32_peak,
                          "per_unit": "25 flops per canonical sample (SURVEY 8(d), lerp = 2); peak 148 x 128 "
                                      "lanes x 2 (FMA) x sm_max_mhz"},
            "executed_gathers_per_launch": counts["gathers"],
            "executed_gather_gbs": counts["gathers"] * bytes_per_sample / march_s / 1e9,
            "algorithmic_output_bytes_per_launch": 20 * W * H * F,
            "hbm_peak_gbs": peaks.get("hbm_gbs")}
    # the sampler's own ceiling (SURVEY 8(d) "Denominators"): the march's light-sample loop alone
    # on a fully occupied, L1-resident 16^3 grid of the same layout (nsl_bench_l1_gather), measured
    # here after the timed region; executed gathers and tested samples (occupancy tests, gathered
    # or not) of the march per second against it
    try:
        if not args.no_sampler_ceiling:
            roof["sampler_ceiling"] = sampler_ceiling(layout, counts, march_s)
    except Exception as e:                      # reported, never fatal for the bench line
        roof["sampler_ceiling"] = {"error": str(e)[:200]}

    line = {"metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16" if layout == 2 else "f32", "data": "synthetic",
            "config": {"workload": CONFIG_TEXT[cfg], "frames_per_rank": F, "frames_total": F * world,
                       "map": f"{W}x{H}", "grid": f"{w.grid.nx}^3", "layout": nsl.LAYOUT_NAMES[layout] + (" (auto)" if args.layout == "auto" else ""), "light_model": args.light_model,
                       "l2": "flushed (512 MiB write) between timed steps, outside the events",
                       "step": "CUDA-graph replay" if args.graph else "eager launches (PDL-chained)",
                       "parallelism": f"frame-sharded x{world}, no data-path collective"},
            "samples_per_s": counts["canonical_samples"] * world * K / t_loop,
            "ms_per_frame": ms_step / F, "frames_per_s": F * world * K / t_loop,
            "march_ms_per_step": statistics.mean(march_ms), "layout_ms_per_step": statistics.mean(layout_ms),
            "counts_per_rank_step": counts, "gpu_launches": launches_per_step(w, args, nsl, layout) * K, "clocks": clk,
            "roofline": roof}

    if cfg == "P482":                       # the paper's own workload: its number is context (other GPU)
        line["vs_baseline"] = value / PAPER_P482["rays_per_s"]
        line["paper_context"] = dict(PAPER_P482, note="vs_baseline = rays/s / the paper's 512^2 / 2 ms; a "
                                     "different GPU, density field and (unstated) amount of work per frame")
    # end-to-end through the public host API: pinned host density in, pinned host guiding maps out
    if not args.no_e2e:
        hd = torch.from_numpy(w.volume(0)).pin_memory() if len(raw) == 1 else None
        if hd is not None:
            hr = torch.empty((F, H, W, 4), dtype=torch.float32).pin_memory()
            hdep = torch.empty((F, H, W), dtype=torch.float32).pin_memory()
            for _ in range(max(1, args.warmup)):
                nsl.guiding_map_host(w.grid, hd, layout, w.cameras, w.lights, w.light_mode, w.medium, w.march,
                                     w.frame_ids, hr, hdep)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ke = max(1, min(K, 20))       # ~130 ms of e2e steps: host/PCIe hiccups average out
            es.record(stream)
            for _ in range(ke):
                nsl.guiding_map_host(w.grid, hd, layout, w.cameras, w.lights, w.light_mode, w.medium, w.march,
                                     w.frame_ids, hr, hdep)
            ee.record(stream)
            torch.cuda.synchronize()
            te = es.elapsed_time(ee) / 1e3
            if world > 1:
                te = max_over_ranks(te, args.backend)
            line["e2e"] = {"value": W * H * F * world * ke / te, "unit": "rays/s",
                           "h2d_bytes_per_step": int(hd.numel() * 4 + F * (40 + 24 * w.n_lights + 8)),
                           "d2h_bytes_per_step": int(hr.numel() * 4 + hdep.numel() * 4),
                           "ms_per_step": 1e3 * te / ke, "api": "nsl_guiding_map_host"}
            # the compact download (nsl_guiding_map_host_f16: fp16 maps, 10 B/pixel; not the parity path)
            hr16 = torch.empty((F, H, W, 4), dtype=torch.float16).pin_memory()
            hd16 = torch.empty((F, H, W), dtype=torch.float16).pin_memory()
            nsl.guiding_map_host_f16(w.grid, hd, layout, w.cameras, w.lights, w.light_mode, w.medium, w.march,
                                     w.frame_ids, hr16, hd16)
            torch.cuda.synchronize()
            es.record(stream)
            for _ in range(ke):
                nsl.guiding_map_host_f16(w.grid, hd, layout, w.cameras, w.lights, w.light_mode, w.medium, w.march,
                                         w.frame_ids, hr16, hd16)
            ee.record(stream)
            torch.cuda.synchronize()
            te16 = es.elapsed_time(ee) / 1e3
            if world > 1:
                te16 = max_over_ranks(te16, args.backend)
            line["e2e_f16"] = {"value": W * H * F * world * ke / te16, "unit": "rays/s",
                               "h2d_bytes_per_step": int(hd.numel() * 4 + F * (40 + 24 * w.n_lights + 8)),
                               "d2h_bytes_per_step": int(hr16.numel() * 2 + hd16.numel() * 2),
                               "ms_per_step": 1e3 * te16 / ke, "api": "nsl_guiding_map_host_f16",
                               "note": "fp16 (RNE) download of the fp32 maps; not the 1e-4 parity path"}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        res = time_oracle(cfg, args.cpu_seconds)
        line["cpu_baseline"] = {"value": res["rays_per_s"], "unit": "rays/s", "cores": 1, "kind": "oracle",
                                "sample": res["sample"], "samples_per_s": res["samples_per_s"],
                                "cpu": host_cpu_name(), "seconds": res["seconds"],
                                # whole frames of this workload at the oracle's measured sample rate
                                "extrapolated_ms_per_frame": 1e3 * counts["canonical_samples"] / F
                                                            / res["samples_per_s"],
                                "extrapolation": "canonical march samples per frame (this run's counted launch) / "
                                                 "the oracle's measured samples/s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
