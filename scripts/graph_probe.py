"""Eager vs CUDA-graph replay of the bench step (volume re-build + plan execute) on C2:
device time per step with the L2 flushed between steps (outside the events)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402

w = I.make_workload("C2")
raw = torch.from_numpy(w.volume(0)).cuda()
storage = torch.empty(nsl.volume_bytes(w.grid, 3), dtype=torch.uint8, device="cuda")
vols = [nsl.Volume(w.grid, raw, 3, storage=storage)]
plan = nsl.make_plan(w, vols)
outs = nsl.alloc_outputs(w.n_frames, w.height, w.width)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def step():
    keep = nsl.Volume(w.grid, raw, 3, storage=storage, stream=s)
    plan.execute(outs[0], outs[1], stream=s)
    return keep


def timed(fn, n=100):
    ts = []
    for _ in range(n):
        with torch.cuda.stream(s):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        s.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts), statistics.median(ts)


for _ in range(5):
    step()
torch.cuda.synchronize()
print("eager  ms/step mean %.4f median %.4f" % timed(step))
g = torch.cuda.CUDAGraph()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.graph(g, stream=s):
    k = step()
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
def replay():
    with torch.cuda.stream(s):
        g.replay()


print("graph  ms/step mean %.4f median %.4f" % timed(replay))
