"""Host-share throughput probe: native host histogram on 1..N threads (the DeviceA rate on this box)."""
import os, time, sys
sys.path.insert(0, '.')
import numpy as np
from paper_1303_2171_b200.kernels_regular import host_histogram
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
data = (np.arange(1 << 28, dtype=np.uint64) * 0x9E3779B97F4A7C15 >> np.uint64(56)).astype(np.uint8)
for w in (1, 2, 4, 8, 16, 32, 64):
    if w > len(os.sched_getaffinity(0)) * 2: break
    host_histogram(data, 256, w)
    t = time.perf_counter(); host_histogram(data, 256, w); dt = time.perf_counter() - t
    print(f"workers {w:3d}: {data.size / dt / 1e9:.2f} Gelem/s")
import torch
h = torch.from_numpy(data).pin_memory()
d = torch.empty_like(h, device="cuda")
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize()
print(f"H2D pinned: {data.size / (time.perf_counter() - t) / 1e9:.1f} GB/s")
# host histogram while a 1 GiB H2D DMA streams from another pinned buffer (contention)
import threading
big = torch.empty(1 << 30, dtype=torch.uint8, pin_memory=True)
dbig = torch.empty_like(big, device="cuda")
for w in (8, 15):
    stop = False
    def dma():
        while not stop:
            dbig.copy_(big, non_blocking=True); torch.cuda.synchronize()
    th = threading.Thread(target=dma); th.start(); time.sleep(0.05)
    t = time.perf_counter(); host_histogram(data, 256, w); dt = time.perf_counter() - t
    stop = True; th.join()
    print(f"workers {w:3d} under DMA: {data.size / dt / 1e9:.2f} Gelem/s")
