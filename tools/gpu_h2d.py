"""Raw pinned host->device copy rate of the cf4 e2e input (132 MB), for the
e2e floor in DESIGN.md: python tools/gpu_h2d.py"""
import torch, time
n = 132 * 1024 * 1024 // 4
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
for _ in range(3):
    d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(10):
    e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print("h2d 132MB ms", min(ts), "GB/s", 132 * 1.048576e6 / min(ts) / 1e6)
