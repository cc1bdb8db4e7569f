"""Animated-volume configs (C4: a fresh 256^3 volume per frame): the step is 60 volume builds
plus 60 frame marches.  Sequential: build everything, then march everything (what bench.py
times).  Pipelined: frames in chunks, chunk c+1's volumes build on a second stream while chunk
c marches (stream events order each chunk's march after its builds) - the HBM-bound builds hide
under the latency-bound marches.  Library: the same schedule inside one C-ABI call,
nsl_guiding_map_animated.  Device time per step, L2 flushed between steps.

    python scripts/bench_pipeline.py [--config C4 --frames 60 --chunk 6 --steps 5]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--config", default="C4")
p.add_argument("--frames", type=int, default=60)
p.add_argument("--chunk", type=int, default=6)
p.add_argument("--steps", type=int, default=5)
p.add_argument("--layout", default="oct_f32")
a = p.parse_args()
layout = nsl.LAYOUTS[a.layout]
w = I.make_workload(a.config, frames=list(range(a.frames)))
F = w.n_frames
raw = [torch.from_numpy(w.volume(i)).cuda() for i in range(len(w.volume_specs))]
storage = [torch.empty(nsl.volume_bytes(w.grid, layout), dtype=torch.uint8, device="cuda") for _ in raw]
outs = nsl.alloc_outputs(F, w.height, w.width)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()

# chunk c: frames [c*chunk, (c+1)*chunk) with their own volumes and plan (outputs are views)
chunks = []
for f0 in range(0, F, a.chunk):
    fr = list(range(f0, min(f0 + a.chunk, F)))
    vids = sorted({w.frame_vol[f] for f in fr})
    sub = w.subset(fr)
    vols = [nsl.Volume(w.grid, raw[v], layout, storage=storage[v], stream=sa) for v in vids]
    plan = nsl.make_plan(sub, vols)
    chunks.append((fr, vids, plan))
torch.cuda.synchronize()
all_vols = list(range(len(raw)))
full_plan = nsl.make_plan(w, [nsl.Volume(w.grid, raw[v], layout, storage=storage[v], stream=sa) for v in all_vols])
torch.cuda.synchronize()


def sequential():
    keep = [nsl.Volume(w.grid, raw[v], layout, storage=storage[v], stream=sa) for v in all_vols]
    full_plan.execute(outs[0], outs[1], stream=sa)
    return keep


def pipelined():
    keep = []
    sb.wait_stream(sa)
    for fr, vids, plan in chunks:
        keep += [nsl.Volume(w.grid, raw[v], layout, storage=storage[v], stream=sb) for v in vids]
        ev = torch.cuda.Event()
        ev.record(sb)
        sa.wait_event(ev)
        plan.execute(outs[0][fr[0]:fr[-1] + 1], outs[1][fr[0]:fr[-1] + 1], stream=sa)
    sa.wait_stream(sb)
    return keep


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(a.steps):
        with torch.cuda.stream(sa):
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(sa)
        fn()
        e1.record(sa)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


dens = [raw[w.frame_vol[f]] for f in range(F)]
stor_f = [storage[w.frame_vol[f]] for f in range(F)]


anim = nsl.Animated(w.grid, dens, layout, stor_f, w.cameras, w.lights, w.light_mode, w.medium, w.march,
                    w.frame_ids, chunk=a.chunk)


def library():
    anim(outs[0], outs[1], stream=sa)


t_seq = timed(sequential)
ref = (outs[0].clone(), outs[1].clone())
t_pipe = timed(pipelined)
same = bool(torch.equal(outs[0], ref[0]) and torch.equal(outs[1], ref[1]))
t_lib = timed(library)
same_lib = bool(torch.equal(outs[0], ref[0]) and torch.equal(outs[1], ref[1]))
print(json.dumps({"config": a.config, "frames": F, "volumes": len(raw), "chunk": a.chunk,
                  "sequential_ms_per_step": t_seq, "pipelined_ms_per_step": t_pipe,
                  "library_ms_per_step": t_lib, "speedup": t_seq / t_pipe, "library_speedup": t_seq / t_lib,
                  "outputs_bitwise_equal": same and same_lib}))
