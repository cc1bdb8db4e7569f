import torch, time
n = 315 * 1024 * 1024 // 4
d = torch.empty(n, device="cuda")
h = torch.empty(n).pin_memory()
for _ in range(3):
    h.copy_(d, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    h.copy_(d, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H GB/s", 5 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
e0.record()
for _ in range(5):
    d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("H2D GB/s", 5 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
# chunked D2H 8 pieces
c = n // 8
e0.record()
for _ in range(5):
    for i in range(8):
        h[i*c:(i+1)*c].copy_(d[i*c:(i+1)*c], non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("D2H chunked GB/s", 5 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9)
