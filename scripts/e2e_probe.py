import torch, time, sys, os
sys.path.insert(0, os.getcwd())
import nsl_inputs as I, paper_2604_03748_b200 as nsl
w = I.make_workload("C2")
F, H, W = w.n_frames, w.height, w.width
hd = torch.from_numpy(w.volume(0)).pin_memory()
hr = torch.empty((F, H, W, 4)).pin_memory()
hdep = torch.empty((F, H, W)).pin_memory()
def call():
    nsl.guiding_map_host(w.grid, hd, 3, w.cameras, w.lights, w.light_mode, w.medium, w.march, w.frame_ids, hr, hdep)
for _ in range(3): call()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): call()
torch.cuda.synchronize()
print("host wall ms per call", (time.perf_counter() - t0) / 10 * 1e3)
# host-side marshalling cost alone: time the python+ctypes prep by timing the call with a tiny workload
w1 = I.make_workload("C2", frames=[0])
hr1 = torch.empty((1, H, W, 4)).pin_memory(); hd1 = torch.empty((1, H, W)).pin_memory()
t0 = time.perf_counter()
for _ in range(20):
    nsl.guiding_map_host(w1.grid, hd, 3, w1.cameras, w1.lights, w1.light_mode, w1.medium, w1.march, w1.frame_ids, hr1, hd1)
print("1-frame call ms", (time.perf_counter() - t0) / 20 * 1e3)
d = torch.empty((F, H, W, 4), device="cuda"); dd = torch.empty((F, H, W), device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(10):
    hr.copy_(d, non_blocking=True); hdep.copy_(dd, non_blocking=True)
torch.cuda.synchronize(); print("D2H only ms", (time.perf_counter() - t0) / 10 * 1e3)
