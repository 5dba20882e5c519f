"""Eager back-to-back calls vs one CUDA-graph capture replayed, for the
device-resident steps whose kernels are short (SpMV 1M: ~77 us; histogram
2^30: ~177 us): launch overhead per step and whether the library's
asynchronous calls are capturable."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

from paper_1303_2171_b200.datasets import device_gen_csr
from paper_1303_2171_b200.kernels_irregular import gpu_spmv, spmv_preprocess
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

rows = 1_000_000
m = device_gen_csr(rows, rows, 42, 1.6e-5)
prep = spmv_preprocess(m, Platform.build(1.0, 3.0), WorkShare.manual(0.0))
dm, perm = prep.permuted, prep.perm
x = torch.rand(rows, dtype=torch.float64, device="cuda")
y = torch.empty(rows, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, k=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k * 1e3


step = lambda: gpu_spmv(dm, x, 0, rows, y=y, perm=perm, asynchronous=True)
eager = timed(step)
want = y.clone()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
y.zero_()
graph = timed(g.replay)
same = bool(torch.equal(y.view(torch.int64), want.view(torch.int64)))
print(f"spmv eager {eager:.1f} us  graph {graph:.1f} us  bit-identical {same}")
