"""Sampler ceiling per layout (SURVEY §8(d) "Denominators"): nsl_bench_l1_gather on a fully
occupied n^3 grid (16^3: L1-resident; 32^3 / 64^3: L2-resident), CUDA events around the launch.

    python scripts/l1_gather_peak.py [--sizes 16 32 64] [--reps 64] [--waves 4]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402


def peak(n, layout, reps, waves, iters=10):
    rng = np.random.default_rng(7)
    dens = torch.from_numpy((0.5 + 0.1 * rng.random((n, n, n))).astype(np.float32)).cuda()
    vol = nsl.Volume(I.Grid(n, n, n, (0.0, 0.0, 0.0), 1.0 / n), dens, layout)
    sink = torch.empty(148 * 16 * waves * 128, dtype=torch.float32, device="cuda")
    samples = nsl.bench_l1_gather(vol, sink, waves=waves, reps=reps)
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nsl.bench_l1_gather(vol, sink, waves=waves, reps=reps)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = statistics.median(ts)
    return samples / t, t


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    p.add_argument("--sizes", type=int, nargs="+", default=[16, 32, 64])
    p.add_argument("--reps", type=int, default=64)
    p.add_argument("--waves", type=int, default=4)
    a = p.parse_args()
    for name, lay in nsl.LAYOUTS.items():
        for n in a.sizes:
            sps, t = peak(n, lay, a.reps, a.waves)
            print(json.dumps({"layout": name, "grid": n, "samples_per_s": sps, "launch_ms": t * 1e3,
                              "corner_bytes_per_s": sps * (16 if name == "corner_f16" else 32)}), flush=True)
