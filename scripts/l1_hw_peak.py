"""Hardware L1/TEX gather ceiling (nsl_bench_l1_peak; DESIGN.md §7 roofline): lane bytes/s of
ld.global.nc.v8.f32 loads with no sampler arithmetic, for the march's warp footprint (frame 0
of the config; without and with the per-lane C4 jitter), fully coalesced lanes and a broadcast, L1-resident (stride 0) and streamed
through L2 (the same lane pattern shifted by `--l2-stride` elements per repetition over a
64 MB span).

    python scripts/l1_hw_peak.py [--config C2] [--reps 256] [--waves 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402

if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="C2")
    p.add_argument("--reps", type=int, default=256)
    p.add_argument("--waves", type=int, default=8)
    p.add_argument("--l2-stride", type=int, default=4099)
    a = p.parse_args()
    w = I.make_workload(a.config, frames=[0])
    import torch
    torch.cuda.set_device(0)
    res = bench.l1_hw_ceiling(w, nsl, patterns=("footprint", "footprint_jitter", "coalesced", "broadcast"), reps=a.reps, waves=a.waves)
    for k, v in res.items():
        print(json.dumps({"pattern": k, "source": "L1 (stride 0)", **v}), flush=True)
    span = (64 << 20) // 32
    res = bench.l1_hw_ceiling(w, nsl, patterns=("footprint", "footprint_jitter", "coalesced"), stride=a.l2_stride, span=span,
                              reps=a.reps, waves=a.waves)
    for k, v in res.items():
        print(json.dumps({"pattern": k, "source": f"L2 (stride {a.l2_stride} x 32 B over 64 MB)", **v}), flush=True)
