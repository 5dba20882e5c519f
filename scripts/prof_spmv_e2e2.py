"""Finer split of the SpMV end-to-end step: PCIe floor, each side alone,
both sides together, and the host-side un-permute."""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, ".")
import numpy as np
import torch

from paper_1303_2171_b200.datasets import csr_arrays
from paper_1303_2171_b200.kernels_irregular import (CsrMatrix, SpmvPrep, _host_range_matvec, gpu_spmv, spmv_hybrid,
                                                    spmv_preprocess)
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
print("dtypes", p.row_ptr.dtype, p.col_idx.dtype, p.values.dtype, "nnz", int(p.row_ptr[-1]))
hm = CsrMatrix(p.rows, p.cols, pinned(p.row_ptr), pinned(p.col_idx), pinned(p.values))
x = pinned(np.random.default_rng(0).random(1_000_000))
perm = np.asarray(prep.perm)


def t(fn, n=5):
    fn()
    torch.cuda.synchronize()
    b = []
    for _ in range(n):
        s = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        b.append(time.perf_counter() - s)
    return min(b) * 1e3


dc = torch.empty(hm.col_idx.size, dtype=torch.int32, device="cuda")
dv = torch.empty(hm.values.size, dtype=torch.float64, device="cuda")
tc, tv = torch.from_numpy(hm.col_idx), torch.from_numpy(hm.values)
print("H2D col+val (torch)        %.2f ms" % t(lambda: (dc.copy_(tc, non_blocking=True), dv.copy_(tv, non_blocking=True))))
y = np.empty(p.rows)
print("gpu_spmv all rows, perm    %.2f ms" % t(lambda: gpu_spmv(hm, x, 0, p.rows, y, perm)))
print("gpu_spmv all rows, no perm %.2f ms" % t(lambda: gpu_spmv(hm, x, 0, p.rows)))
for f in (0.3, 0.4, 0.5):
    cum = np.asarray(p.row_ptr, dtype=np.int64)
    split = int(np.searchsorted(cum, f * cum[-1]))
    ta = t(lambda: _host_range_matvec(hm, x, 0, split, 15))
    tb = t(lambda: gpu_spmv(hm, x, split, p.rows, y, perm))

    def both():
        with ThreadPoolExecutor(2) as pool:
            fa = pool.submit(_host_range_matvec, hm, x, 0, split, 15)
            fb = pool.submit(gpu_spmv, hm, x, split, p.rows, y, perm)
            fa.result(), fb.result()

    ya = _host_range_matvec(hm, x, 0, split, 15)

    def sc():
        y[perm[:split]] = ya

    hp = SpmvPrep(hm, prep.perm, split, 15)
    print(f"f={f}: host alone {ta:.2f}  gpu alone {tb:.2f}  both {t(both):.2f}  numpy scatter {t(sc):.2f}  "
          f"spmv_hybrid {t(lambda: spmv_hybrid(hp, x)):.2f} ms")
