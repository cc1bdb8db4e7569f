"""L1-locality probe for the march: time the plan on C2's 60 distinct frames vs 60 copies
of one frame (co-resident CTAs then share their volume data) vs 1 frame repeated.
    python scripts/locality_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402


def timeit(frames, reps=50):
    w = I.make_workload("C2", frames=frames)
    vols = nsl.upload_workload_volumes(w, 3)
    outs = nsl.alloc_outputs(w.n_frames, w.height, w.width)
    plan = nsl.make_plan(w, vols)
    for _ in range(3):
        plan.execute(outs[0], outs[1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.execute(outs[0], outs[1])
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


print("60 distinct frames      ms", timeit(list(range(60))))
print("60 copies of frame 0    ms", timeit([0] * 60))
print("60 copies of frame 30   ms", timeit([30] * 60))
for f in (0, 15, 30, 45):
    print(f"frame {f:2d} alone x60 (sum of 60 single-frame plans) ms", 60 * timeit([f], reps=20))
