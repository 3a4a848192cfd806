"""Pinned H2D rate vs the host NUMA node of the pinned buffer (first touch
under a CPU affinity): python tools/gpu_numa.py"""
import os, subprocess, torch
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
print("nodes:", sorted(os.listdir("/sys/devices/system/node")) if os.path.exists("/sys/devices/system/node") else None)
for node in sorted(x for x in os.listdir("/sys/devices/system/node") if x.startswith("node")):
    cpus = open(f"/sys/devices/system/node/{node}/cpulist").read().strip()
    print(node, cpus)
print("affinity", sorted(os.sched_getaffinity(0))[:8], len(os.sched_getaffinity(0)))
n = 132 * 1024 * 1024 // 4
def rate(tag):
    h = torch.empty(n, dtype=torch.int32).pin_memory()
    h.fill_(1)
    d = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(8):
        e0.record(); d.copy_(h, non_blocking=True); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(tag, "h2d GB/s", round(138.4 / min(ts), 1))
rate("default")
allc = sorted(os.sched_getaffinity(0))
for node in sorted(x for x in os.listdir("/sys/devices/system/node") if x.startswith("node")):
    cl = open(f"/sys/devices/system/node/{node}/cpulist").read().strip()
    cpus = set()
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-"); cpus |= set(range(int(a), int(b) + 1))
        elif part: cpus.add(int(part))
    cpus &= set(allc)
    if not cpus: continue
    os.sched_setaffinity(0, cpus)
    rate(f"affinity {node}")
os.sched_setaffinity(0, allc)
