"""e2e host API (C2, fp32 maps): ms per call vs the number of frame chunks (NSL_HOST_CHUNKS), and
the bare 315 MB D2H of the same maps.   python scripts/e2e_chunks.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import nsl_inputs as I  # noqa: E402
import paper_2604_03748_b200 as nsl  # noqa: E402

w = I.make_workload("C2")
F, H, W = w.n_frames, w.height, w.width
hd = torch.from_numpy(w.volume(0)).pin_memory()
hr = torch.empty((F, H, W, 4)).pin_memory()
hdep = torch.empty((F, H, W)).pin_memory()


def call():
    nsl.guiding_map_host(w.grid, hd, 3, w.cameras, w.lights, w.light_mode, w.medium, w.march, w.frame_ids, hr, hdep)


for ch in (2, 4, 8, 15, 30, 60, 8):
    os.environ["NSL_HOST_CHUNKS"] = str(ch)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        call()
    torch.cuda.synchronize()
    print(f"chunks {ch:3d}: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per call", flush=True)
d = torch.empty((F, H, W, 4), device="cuda")
dd = torch.empty((F, H, W), device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20):
    hr.copy_(d, non_blocking=True)
    hdep.copy_(dd, non_blocking=True)
torch.cuda.synchronize()
print(f"bare D2H of the maps: {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms", flush=True)
