"""End-to-end histogram through the public API on a pinned 2^30 u8 host
array: time per call at fixed host shares, and the calibrated share."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1303_2171_b200.kernels_regular import HistogramWorkload, hybrid_histogram
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare, calibrate_measured

n = 1 << 30
t = torch.empty(n, dtype=torch.uint8, pin_memory=True)
t.numpy()[...] = np.random.default_rng(1).integers(0, 256, size=n, dtype=np.uint8)
x = t.numpy()
import os
p = Platform.build(1.0, 3.0, workers_a=max(1, (os.cpu_count() or 2) - 1))
for f in (0.0, 0.3, 0.34, 0.38, 0.42):
    hybrid_histogram(x, 256, p, WorkShare.manual(f))
    ts = []
    for _ in range(15):
        a = time.perf_counter()
        hybrid_histogram(x, 256, p, WorkShare.manual(f))
        ts.append(time.perf_counter() - a)
    print(f"share {f:.2f}: median {np.median(ts) * 1e3:6.2f} ms  min {min(ts) * 1e3:6.2f} ms  -> {n / np.median(ts) / 1e9:5.1f} Gelem/s  all " + " ".join(f"{v * 1e3:.1f}" for v in ts))
for _ in range(3):
    sh = calibrate_measured(HistogramWorkload(x, 256), p, max_refinements=6, repeats=2)
    print("calibrated share", round(sh.fraction_a, 4))
