"""Histogram kernel time vs input size (device-resident u8, 256 bins): fits
t = a + b*n to separate the fixed per-launch cost from the streaming rate."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.kernels_regular import gpu_histogram
from paper_1303_2171_b200.rng import device_splitmix

x = torch.empty(1 << 32, dtype=torch.uint8, device="cuda")
device_splitmix(x, 42, _lib.HB_GEN_LOW8)
out = torch.empty(256, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ns, ts = [], []
for lg in (26, 27, 28, 29, 30, 31, 32):
    n = 1 << lg
    v = x[:n]
    for _ in range(3):
        gpu_histogram(v, 256, out, asynchronous=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        gpu_histogram(v, 256, out, asynchronous=True)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    ns.append(n)
    ts.append(us)
    print(f"n=2^{lg}: {us:9.1f} us  {n / us / 1e3:7.0f} GB/s")
b, a = np.polyfit(np.array(ns, dtype=np.float64), np.array(ts), 1)
print(f"fit: t = {a:.1f} us + n / {1e-3 / b:.0f} GB/s")
