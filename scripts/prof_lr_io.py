"""List ranking through the host-buffer API at 2^28 nodes: pinned int64 /
int32 successors, results dropped each call; mean of 5 calls after 2."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1303_2171_b200.datasets import device_gen_list
from paper_1303_2171_b200.kernels_irregular import gpu_list_rank

n = 1 << 28
succ_d, head = device_gen_list(n, 42)
for dt in (torch.int64, torch.int32):
    h = torch.empty(n, dtype=dt, pin_memory=True)
    h.copy_(succ_d.to(dt))
    x = h.numpy()
    ts = []
    for i in range(7):
        a = time.perf_counter()
        r = gpu_list_rank(x, head)
        ts.append(time.perf_counter() - a)
        del r
    print(f"{str(dt):12s} " + " ".join(f"{t * 1e3:6.1f}" for t in ts) + f"  mean(last 5) {np.mean(ts[2:]) * 1e3:.1f} ms", flush=True)
