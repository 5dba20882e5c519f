"""Histogram step overheads: eager back-to-back hb_hist calls (2 memsets +
pool alloc/free + kernel per call) vs the same calls captured once in a
CUDA graph and replayed, 2^30 u8 (BASELINE configs[1])."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_1303_2171_b200 import _lib
from paper_1303_2171_b200.kernels_regular import gpu_histogram
from paper_1303_2171_b200.rng import device_splitmix

n = 1 << 30
x = torch.empty(n, dtype=torch.uint8, device="cuda")
device_splitmix(x, 42, _lib.HB_GEN_LOW8)
out = torch.empty(256, dtype=torch.int64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 20


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(K):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / K * 1e3


eager = timed(lambda: gpu_histogram(x, 256, out, asynchronous=True))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    gpu_histogram(x, 256, out, asynchronous=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        gpu_histogram(x, 256, out, asynchronous=True)
graph = timed(g.replay)
ok = int(out.sum().item()) == n
print(f"eager {eager:.1f} us/step  graph {graph:.1f} us/step  GB/s eager {n / eager / 1e3:.0f} graph {n / graph / 1e3:.0f}  sum ok {ok}")
