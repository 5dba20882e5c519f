"""Where the SpMV end-to-end step (spmv_hybrid on pinned host arrays) spends its time."""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1303_2171_b200.datasets import csr_arrays
from paper_1303_2171_b200.kernels_irregular import CsrMatrix, SpmvPrep, _gpu_rows, _host_range_matvec, spmv_hybrid, spmv_preprocess
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

ptr, col, val = csr_arrays(1_000_000, 1_000_000, 42, 1.6e-5)
m = CsrMatrix(1_000_000, 1_000_000, ptr, col, val)
prep = spmv_preprocess(m, Platform.build(1.0, 3.0), WorkShare.manual(0.0))
def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()
p = prep.permuted
hm = CsrMatrix(p.rows, p.cols, pinned(p.row_ptr), pinned(p.col_idx), pinned(p.values))
x = pinned(np.random.default_rng(0).random(1_000_000))
hp = SpmvPrep(hm, prep.perm, 0, 15)
def t(fn, n=3):
    fn(); b = []
    for _ in range(n):
        s = time.perf_counter(); fn(); b.append(time.perf_counter() - s)
    return min(b) * 1e3
print("spmv_hybrid (all GPU)   %.2f ms" % t(lambda: spmv_hybrid(hp, x)))
print("_gpu_rows all rows      %.2f ms" % t(lambda: _gpu_rows(hm, x, 0, hm.rows)))
print("host rows 15 threads    %.2f ms" % t(lambda: _host_range_matvec(hm, x, 0, hm.rows, 15)))
yp = np.random.default_rng(1).random(1_000_000); perm = np.asarray(prep.perm)
def scatter():
    y = np.empty_like(yp); y[perm] = yp
print("numpy y[perm] = y_perm  %.2f ms" % t(scatter))
