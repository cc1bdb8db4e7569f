"""Ad-hoc timing of workload variants through the C ABI (CUDA events, warm, L2 not flushed)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import numpy as np, torch
import nsl_inputs as I
import paper_2604_03748_b200 as nsl

def timeit(w, reps=20, layout=1):
    vols = nsl.upload_workload_volumes(w, layout)
    outs = nsl.alloc_outputs(w.n_frames, w.height, w.width)
    plan = nsl.make_plan(w, vols)
    for _ in range(3): plan.execute(outs[0], outs[1])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): plan.execute(outs[0], outs[1])
    e1.record(); torch.cuda.synchronize()
    c = plan.execute_counted(outs[0], outs[1])
    return e0.elapsed_time(e1) / reps, c

base = I.make_workload("C2")
base.volume(0)
cases = {
  "C2": base,
  "C2 zero volume": replace(base, _cache={0: np.zeros_like(base.volume(0))}),
  "C2 front only": replace(base, lights=[r[:1] for r in base.lights], _cache=base._cache),
  "C2 front+top": replace(base, lights=[r[:2] for r in base.lights], _cache=base._cache),
  "C2 no jitter": replace(base, march=replace(base.march, jitter=0), _cache=base._cache),
  "C2 no C9": replace(base, march=replace(base.march, front_identity=0), _cache=base._cache),
  "C2 1 frame": base.subset([0]),
  "C2 10 frames": base.subset(list(range(10))),
  "C2 kappa64": replace(base, medium=replace(base.medium, extinction=64.0), _cache=base._cache),
}
for name, w in cases.items():
    ms, c = timeit(w)
    print(f"{name:18s} {ms:8.4f} ms  per frame {1e3*ms/w.n_frames:7.2f} us  tp={c['tested_primary']:.3e} tl={c['tested_light']:.3e} gath={c['gathers']:.3e} occ={c['occupied_samples']:.3e}", flush=True)
