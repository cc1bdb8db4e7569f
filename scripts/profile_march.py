"""Minimal driver for ncu: the C2 batch (60 frames 512^2 over 128^3, guide lights),
2 warm-up launches then N profiled launches of march_kernel.
    python scripts/profile_march.py [--layout oct_f32] [--launches 1] [--config C2]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--layout", default="oct_f32")
p.add_argument("--launches", type=int, default=1)
p.add_argument("--config", default="C2")
p.add_argument("--frames", type=int, default=0)
a = p.parse_args()
w = I.make_workload(a.config, frames=list(range(a.frames)) if a.frames else None)
layout = nsl.LAYOUTS[a.layout]
vols = nsl.upload_workload_volumes(w, layout)
outs = nsl.alloc_outputs(w.n_frames, w.height, w.width)
plan = nsl.make_plan(w, vols)
for _ in range(2 + a.launches):
    plan.execute(outs[0], outs[1])
torch.cuda.synchronize()
print("ok", w.name, w.n_frames, a.layout)
