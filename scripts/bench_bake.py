"""Benchmark of the NEXT-1 six-way bake on one GPU: C2 volume
(plume 128^3), 512^2, spp samples per pixel, F frames of the rotating camera.
Prints one JSON line (pixel-samples/s, ms/frame, gathers/s, oracle rate).

    python scripts/bench_bake.py [--frames 4 --spp 16 --steps 5 --warmup 2]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--frames", type=int, default=4)
p.add_argument("--spp", type=int, default=16)
p.add_argument("--steps", type=int, default=5)
p.add_argument("--warmup", type=int, default=2)
p.add_argument("--no-oracle", action="store_true")
a = p.parse_args()

w = I.make_workload("C2", frames=list(range(0, 60, 60 // a.frames))[:a.frames])
b = I.default_bake(128, spp=a.spp)
vols = nsl.upload_workload_volumes(w)
out = torch.empty((w.n_frames, w.height, w.width, 2, 4), dtype=torch.float32, device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
nsl.sixway_bake(vols, w.frame_vol, w.cameras, w.medium, b, w.frame_ids, out, counters=cnt)
torch.cuda.synchronize()
gathers = int(cnt.item())
for _ in range(a.warmup):
    nsl.sixway_bake(vols, w.frame_vol, w.cameras, w.medium, b, w.frame_ids, out)
torch.cuda.synchronize()
times = []
for _ in range(a.steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    nsl.sixway_bake(vols, w.frame_vol, w.cameras, w.medium, b, w.frame_ids, out)
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / 1e3)
t = statistics.median(times)
px_samples = w.n_frames * w.width * w.height * a.spp
line = {"metric": "six-way bake pixel-samples/s (NEXT-1)", "value": px_samples / t, "unit": "pixel-samples/s",
        "ms_per_frame": 1e3 * t / w.n_frames, "frames": w.n_frames, "spp": a.spp, "map": "512x512",
        "grid": "128^3 plume (C2)", "gathers_per_s": gathers / t, "gathers_per_launch": gathers,
        "l1tex_gather_gbs": gathers * 32 / t / 1e9, "steps": a.steps}
# roofline: the bake's lanes (16 sub-pixel-jittered samples of one pixel) gather
# near-coalesced, so its L1/TEX ceiling is the measured coalesced rate of nsl_bench_l1_peak (32-B
# elements, L1-resident); achieved = the executed gathers x 32 B per second (a lower bound on
# the algorithmic bytes: empty-block samples are not counted)
import bench as _bench  # noqa: E402
hw = _bench.l1_hw_ceiling(I.make_workload("C2", frames=[0]), nsl, patterns=("coalesced",))
peak = hw["coalesced"]["lane_gbs"]
line["roofline"] = {"bound": "l1tex", "achieved": gathers * 32 / t / 1e9, "peak": peak, "unit": "GB/s",
                    "frac": gathers * 32 / t / 1e9 / peak, "traffic": None,
                    "per_unit": "32 B per executed trilinear gather (occupied primary or light sample)",
                    "peak_source": "measured: nsl_bench_l1_peak, coalesced 32-B lanes, L1-resident, this run"}
if not a.no_oracle:
    import oracle
    pix = np.arange(0, 512 * 512, 509)
    t0 = time.perf_counter()
    oracle.sixway_bake(w.grid, w.volume(0), w.cameras[0], w.medium, b, frame_id=w.frame_ids[0], pixels=pix)
    dt = time.perf_counter() - t0
    line["cpu_baseline"] = {"value": len(pix) * a.spp / dt, "unit": "pixel-samples/s", "cores": 1, "kind": "oracle",
                            "sample": f"{len(pix)} pixels of frame 0 x {a.spp} spp"}
print(json.dumps(line), flush=True)
