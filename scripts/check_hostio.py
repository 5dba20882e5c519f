"""Pageable host <-> device path of libhb200 (pinned double buffer + threaded
memcpy): a 1 GiB sort and a 2 GiB-output bilateral through host arrays, timed;
exits cleanly (the worker pool must not hang interpreter shutdown)."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
from paper_1303_2171_b200.kernels_regular import build_bilateral_lut, gpu_bilateral_rows, gpu_sort

keys = (np.arange(1 << 28, dtype=np.uint64) * 0x9E3779B97F4A7C15 >> np.uint64(32)).astype(np.uint32)
for _ in range(2):
    t = time.perf_counter()
    out, _, _ = gpu_sort(keys)
    dt = time.perf_counter() - t
print(f"sort 2^28 u32 host->host: {dt * 1e3:.1f} ms, sorted {bool(np.all(out[1:] >= out[:-1]))}")
img = (np.arange(8192 * 8192, dtype=np.uint64) * 2654435761 % 251).astype(np.uint8).reshape(8192, 8192)
lut = build_bilateral_lut(5, 2.5, 40.0)
for _ in range(2):
    t = time.perf_counter()
    o = gpu_bilateral_rows(img, lut, 0, 8192)
    dt = time.perf_counter() - t
print(f"bilateral 8192^2 host->host (512 MiB f64 out): {dt * 1e3:.1f} ms")
