"""Per-step times of hybrid_convolve on a pinned 16384^2 image at a few host shares."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1303_2171_b200.datasets import device_gen_image
from paper_1303_2171_b200.kernels_regular import FilterKernel, Image, convolve_rows, hybrid_convolve
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

side = 16384
host = torch.empty((side, side), dtype=torch.uint8, pin_memory=True)
host.copy_(device_gen_image(side, 42))
img = Image(host.numpy())
fk = FilterKernel.gaussian(7)
p = Platform.build(1.0, 3.0, workers_a=15)
for f in (0.0, 0.056, 0.0, 0.056):
    ts = []
    for _ in range(8):
        t = time.perf_counter()
        r = hybrid_convolve(img, fk, p, WorkShare.manual(f))
        ts.append((time.perf_counter() - t) * 1e3)
        del r
    print(f"share {f}: " + " ".join(f"{x:.1f}" for x in ts))
rows = int(0.056 * side)
out = np.empty((rows, side))
for w in (15, 16):
    ts = []
    for _ in range(4):
        t = time.perf_counter()
        convolve_rows(host.numpy(), fk, 0, rows, w, out=out)
        ts.append((time.perf_counter() - t) * 1e3)
    print(f"host conv {rows} rows, {w} workers: " + " ".join(f"{x:.1f}" for x in ts))
