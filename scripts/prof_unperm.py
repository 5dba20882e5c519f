"""Where the host-path SpMV un-permute time goes: all rows with / without
perm, y pinned vs pageable, perm int32 vs int64 (median of 15)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1303_2171_b200.datasets import csr_arrays
from paper_1303_2171_b200.gpu import host_empty
from paper_1303_2171_b200.kernels_irregular import CsrMatrix, gpu_spmv, spmv_preprocess
from paper_1303_2171_b200.platform import Platform
from paper_1303_2171_b200.worksharing import WorkShare

ptr, col, val = csr_arrays(1_000_000, 1_000_000, 42, 1.6e-5)
prep = spmv_preprocess(CsrMatrix(1_000_000, 1_000_000, ptr, col, val), Platform.build(1.0, 3.0), WorkShare.manual(0.0))


def pinned(a):
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


p = prep.permuted
hm = CsrMatrix(p.rows, p.cols, pinned(p.row_ptr), pinned(p.col_idx), pinned(p.values))
x = pinned(np.random.default_rng(0).random(1_000_000))
perm64 = np.asarray(prep.perm).astype(np.int64)
perm32 = perm64.astype(np.int32)


def t(fn, n=15):
    fn()
    b = []
    for _ in range(n):
        s = time.perf_counter()
        fn()
        b.append(time.perf_counter() - s)
    return np.median(b) * 1e3


y_pin = host_empty(p.rows, np.float64)
y_pg = np.zeros(p.rows)
print("no perm (y pinned, returned)  %.2f ms" % t(lambda: gpu_spmv(hm, x, 0, p.rows)))
print("perm64, y pinned              %.2f ms" % t(lambda: gpu_spmv(hm, x, 0, p.rows, y_pin, perm64)))
print("perm64, y pageable            %.2f ms" % t(lambda: gpu_spmv(hm, x, 0, p.rows, y_pg, perm64)))
print("perm32, y pinned              %.2f ms" % t(lambda: gpu_spmv(hm, x, 0, p.rows, y_pin, perm32)))
print("perm64 pinned, y pinned       %.2f ms" % t(lambda: gpu_spmv(hm, x, 0, p.rows, y_pin, pinned(perm64))))
dt = torch.empty(1_000_000, dtype=torch.float64, device="cuda")
ht = torch.empty(1_000_000, dtype=torch.float64, pin_memory=True)


def d2h():
    ht.copy_(dt)
    torch.cuda.synchronize()


print("torch D2H 8 MB -> pinned      %.3f ms" % t(d2h))
