"""The histogram's end-to-end call on a PAGEABLE 2^30 u8 input (bench.HistBench's
data): fixed host shares (median of 8 calls) and calibrate_measured on the
pageable workload itself."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
from paper_1303_2171_b200.kernels_regular import HistogramWorkload, hybrid_histogram
from paper_1303_2171_b200.worksharing import WorkShare, calibrate_measured

wl = bench.HistBench()
wl.setup(0, 1)
torch.cuda.synchronize()
x = wl.x[: wl.CONFIG].cpu().numpy().copy()  # pageable
p = bench.host_platform()
for f in (0.0, 0.2, 0.3, 0.42, 0.5, 0.6, 0.7):
    hybrid_histogram(x, 256, p, WorkShare.manual(f))
    ts = []
    for _ in range(8):
        a = time.perf_counter()
        hybrid_histogram(x, 256, p, WorkShare.manual(f))
        ts.append(time.perf_counter() - a)
    print(f"pageable share {f:.2f}: median {np.median(ts) * 1e3:6.2f} ms -> {x.size / np.median(ts) / 1e9:5.1f} Gelem/s", flush=True)
for _ in range(2):
    sh = calibrate_measured(HistogramWorkload(x, 256), p, max_refinements=6, repeats=2)
    print("calibrated on the pageable input:", round(sh.fraction_a, 4), flush=True)
