"""The bench's histogram e2e leg in its own context (bench.HistBench: device-generated
2^30 u8 input, pinned host copy, host_platform()): the calibrate_measured trace, then
fixed host shares timed back to back (median of 12 calls each)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import bench
from paper_1303_2171_b200.kernels_regular import hybrid_histogram
from paper_1303_2171_b200.worksharing import WorkShare

wl = bench.HistBench()
wl.setup(0, 1)
torch.cuda.synchronize()
for _ in range(2):
    wl.e2e_setup()
    tr = wl.share.probe.refinement_steps if wl.share.probe is not None else ()
    print("calibrated", round(wl.share.fraction_a, 4), "solo a/b ms", round(wl.share.probe.t_device_a * 1e3, 2), round(wl.share.probe.t_device_b * 1e3, 2), "trace", [(round(f, 3), round(t * 1e3, 2)) for f, t in tr], flush=True)
x = wl.host_np
for f in (0.0, 0.2918, 0.34, 0.38, 0.40, 0.42, 0.44, 0.46, 0.50):
    hybrid_histogram(x, 256, wl.platform, WorkShare.manual(f))
    ts = []
    for _ in range(12):
        a = time.perf_counter()
        hybrid_histogram(x, 256, wl.platform, WorkShare.manual(f))
        ts.append(time.perf_counter() - a)
    print(f"share {f:.4f}: median {np.median(ts) * 1e3:6.2f} ms -> {x.size / np.median(ts) / 1e9:5.1f} Gelem/s  "
          + " ".join(f"{v * 1e3:.1f}" for v in ts), flush=True)
